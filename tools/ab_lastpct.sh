for p in 50 25 15 50 25 15; do
  GT_HOST_LAST_PCT=$p timeout 300 python bench.py --no-cpu-baseline --no-scale --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('last $p %', round(l['value']*1e3,4), 'e2e', round(l['e2e']['value']*1e3,4), l['parity']['e2e_tree_equals_reference'])"
done
