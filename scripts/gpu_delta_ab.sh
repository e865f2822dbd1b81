# Delta-evaluation overhead breakdown on the bench config (full-iteration):
# off / variant only (no snapshots) / snapshots without resume / full delta.
for m in full-iteration forward; do
timeout 300 python bench.py --no-cpu-baseline --mode $m --no-delta --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m off', round(d['value']))"
for e in 1 2 0; do
PS_DELTA_EXP=$e timeout 300 python bench.py --no-cpu-baseline --mode $m --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m exp $e', round(d['value']), round(d['delta']['reused_fraction'],3))"
done
done
