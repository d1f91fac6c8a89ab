for tpb in 128 256 128 256; do
  GT_PART_TPB=$tpb timeout 300 python bench.py --no-cpu-baseline --no-scale --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('tpb $tpb', 'C2', round(l['value']*1e3,4), 'e2e', round(l['e2e']['value']*1e3,4), 'partition ms', round(l['kernel_ms_per_step']['partition'],4))"
done
