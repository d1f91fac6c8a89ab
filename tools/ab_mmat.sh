for v in 0 1 0 1; do
  if [ $v = 1 ]; then export GT_NO_MMA_T=1; else unset GT_NO_MMA_T; fi
  timeout 300 python bench.py --no-scale --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('no_mmat' if '$v'=='1' else 'mmat', l['value']*1e3, l['e2e']['value']*1e3)"
done
