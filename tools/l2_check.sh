# DRAM bytes and L2 hit rate of the contraction launches in a C2 tree (no cache flush between kernels)
for w in 0 1; do
  if [ $w = 1 ]; then export GT_NO_L2_WINDOW=1; else unset GT_NO_L2_WINDOW; fi
  echo "== GT_NO_L2_WINDOW=$w"
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --cache-control none --clock-control none -k regex:"k_count_mma|k_prep8|k_count_lanes8" -s 18 -c 18 --csv python tools/profile_target.py train 3 2>/dev/null | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki].split('(')[0][-14:]), {})[r[mi]]=r[vi]
for (i,k),m in d.items():
    print(i, k, {kk.split('.')[0][-16:]: vv for kk,vv in m.items()})
"
done
