timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for cfg in nmt inception; do
PS_DEBUG=1 timeout 900 python bench.py --config $cfg --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | grep -v "^ " | tail -3 | python -c "
import sys,json
for line in sys.stdin:
    if line.startswith('{'):
        d=json.loads(line); print('$cfg', round(d['value']), 'fail', d['chain_failures'], 'cap', d['config']['ready_capacity'], 'SC', d['config']['shared_counters'], 'warps', d['config']['resident_warps_per_sm'], 'T', d['config']['tasks_per_eval'])
    else: print(line.strip()[:300])
"
done
