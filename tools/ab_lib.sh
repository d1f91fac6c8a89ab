# A/B: the in-tree library vs tools/_variants/v.so (same box, alternating)
cp paper_2305_00645_b200/libgtree_b200.so /tmp/base.so
for v in base var base var; do
  if [ $v = var ]; then cp tools/_variants/v.so paper_2305_00645_b200/libgtree_b200.so; else cp /tmp/base.so paper_2305_00645_b200/libgtree_b200.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-scale --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); k=l['kernel_ms_per_step']; print('$v', 'C2', round(l['value']*1e3,4), 'e2e', round(l['e2e']['value']*1e3,4), 'lanes', round(k['count_lanes'],4), 'part', round(k['partition'],4))"
done
cp /tmp/base.so paper_2305_00645_b200/libgtree_b200.so
