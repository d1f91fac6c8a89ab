# A/B a library switch read from the environment on the same GPU box:
#   bash tools/ab_env.sh VAR [value ...]      ("-" = unset; default: unset 1, twice)
# prints the C2 device value and e2e (ms) per setting (bench.py, 20 steps).
var=$1; shift
vals=${*:-"- 1 - 1"}
for v in $vals; do
  if [ "$v" = "-" ]; then unset $var; label="$var unset"; else export $var=$v; label="$var=$v"; fi
  timeout 300 python bench.py --no-scale --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | \
    python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$label', round(l['value']*1e3,4), 'e2e', round(l['e2e']['value']*1e3,4), all(l['parity'].values()))"
done
unset $var
