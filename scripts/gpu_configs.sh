# Bench lines for the non-headline BASELINE configs (parity is covered by the tests).
for cfg in alexnet resnet nmt random1k random10k; do
  PS_DEBUG=1 timeout 900 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --py-ref-seconds 0 --extra none "$@" 2>&1 | grep -E "^\[parasim\]|^\{" | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); c=d['config']; print('$cfg', round(d['value']), 'e2e', round(d['e2e']['value']), 'tasks', c['tasks_per_eval'], 'warps/SM', c['resident_warps_per_sm'], 'cap', c['ready_capacity'], 'SC', c['shared_counters'], d['clocks']['reasons'])
    else: print(l.strip()[:300])
"
done
