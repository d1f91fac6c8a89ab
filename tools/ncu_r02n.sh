# One ncu --set full capture per hot kernel of the C2 tree (first eager tree, the named level) and the C3 walk.
set -x
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_partition_split --launch-skip 5 -c 1 -o gpurun_out/r02n_part_l6 python tools/probe.py c2eager > /dev/null 2>&1
$NCU -k regex:k_count_fused --launch-skip 6 -c 1 -o gpurun_out/r02n_count_l6 python tools/probe.py c2eager > /dev/null 2>&1
$NCU -k regex:k_count_fused --launch-skip 3 -c 1 -o gpurun_out/r02n_count_l3 python tools/probe.py c2eager > /dev/null 2>&1
$NCU -k regex:k_hc_pre --launch-skip 5 -c 1 -o gpurun_out/r02n_hcpre_l5 python tools/probe.py c2eager > /dev/null 2>&1
$NCU -k regex:k_hc_post_finish --launch-skip 5 -c 1 -o gpurun_out/r02n_hcpost_l5 python tools/probe.py c2eager > /dev/null 2>&1
$NCU -k regex:k_walk --launch-skip 3 -c 1 -o gpurun_out/r02n_walk_c3 python tools/probe.py walk > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
for r in gpurun_out/r02n_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv --print-units base > $b.raw.csv
  ncu -i $r --page details --csv > $b.details.csv
  ncu -i $r --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  rm $r
done
gzip -f gpurun_out/r02n_*.sass.csv
du -sh gpurun_out
