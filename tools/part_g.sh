# k_partition per-level times for each forced thread-group size G
for g in ${GS:-0 2 4 8 16}; do
  GT_PART_G=$g ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_partition --csv --log-file gpurun_out/part$g.csv python tools/profile_target.py train 1 > /dev/null 2>&1
  python -c "
import csv
rows = [r for r in csv.reader(open('gpurun_out/part$g.csv')) if len(r) > 5]
vi = rows[0].index('Metric Value')
v = [float(r[vi].replace(',', '')) / 1e3 for r in rows[1:]]
print('G=$g', ' '.join(f'{x:.1f}' for x in v), 'sum %.1f' % sum(v))
"
done
