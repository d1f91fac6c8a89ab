# C3 / C5 inference with 128- vs 256-thread walk CTAs
for tpb in 128 256 128 256; do
  GT_WALK_TPB=$tpb timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('tpb $tpb', 'C3', round(l['secondary']['value']/1e6,1), 'M/s', 'C5', round(l['scale']['c5_infer']['value']/1e6,1), 'M/s', 'C2', round(l['value']*1e3,4))"
done
