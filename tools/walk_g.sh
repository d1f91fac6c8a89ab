# C3 / C5 walk time per forced group size G (0 = chooser)
for g in ${GS:-0 1 2 4 8}; do
  GT_WALK_G=$g timeout 300 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('G=$g', 'C3', round(l['secondary']['value']/1e6,1), 'M/s', 'C5', round(l['scale']['c5_infer']['value']/1e6,1), 'M/s')"
done
