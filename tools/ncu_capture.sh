# One `ncu --set full` capture of one launch, exported as CSV pages (the .ncu-rep
# is too large to bring back from the GPU box):
#   bash tools/ncu_capture.sh OUT KERNEL_REGEX LAUNCH_SKIP PROBE_MODE
# e.g. bash tools/ncu_capture.sh gpurun_out/r02_count_l6 k_count_fused 6 c2eager
# writes OUT.raw.csv.gz (metrics), OUT.sass.csv.gz (per-instruction stalls;
# tools/sass_stalls.py, tools/sass_mix.py, tools/sass_lines.py read it).
out=$1; kern=$2; skip=$3; mode=$4
ncu --set full --clock-control none --import-source on -k regex:$kern --launch-skip $skip -c 1 -o $out \
  python tools/probe.py $mode > /dev/null 2>&1
ncu -i $out.ncu-rep --page raw --csv --print-units base > $out.raw.csv
ncu -i $out.ncu-rep --page source --csv --print-source sass > $out.sass.csv 2>/dev/null
rm -f $out.ncu-rep
gzip -f $out.raw.csv $out.sass.csv
