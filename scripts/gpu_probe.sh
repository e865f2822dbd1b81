timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for cfg in inception; do
for mode in full-iteration forward; do
PS_DEBUG=1 timeout 600 python bench.py --config $cfg --mode $mode --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | grep -v "^ " | tail -2 | python -c "
import sys,json
for line in sys.stdin:
    if line.startswith('{'):
        d=json.loads(line); print('$cfg $mode', round(d['value']), 'fail', d['chain_failures'], 'cap', d['config']['ready_capacity'], 'SC', d['config']['shared_counters'], 'warps', d['config']['resident_warps_per_sm'], 'T', d['config']['tasks_per_eval'])
    else: print(line.strip()[:300])
"
done
done
