# k_count_mma per-level times: normal, loads only (GT_MMA_PROBE=1), MMAs only (GT_MMA_PROBE=2)
for p in ${PROBES:-0 1 2}; do
  GT_MMA_PROBE=$p ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_count_mma --csv --log-file gpurun_out/probe$p.csv python tools/profile_target.py train 1 > /dev/null 2>&1
  python - $p <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/probe{sys.argv[1]}.csv")) if len(r) > 5]
vi = rows[0].index("Metric Value")
print("probe", sys.argv[1], " ".join(f"{float(r[vi].replace(',', '')) / 1e3:.1f}" for r in rows[1:]))
PY
done
