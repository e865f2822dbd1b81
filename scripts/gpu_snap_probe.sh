# random-10k delta probe: snapshot memory budget and back-set capacity of a snapshot
run() { env "$@" timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --py-ref-seconds 0 --extra random10k 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['configs']['random10k']; print('$*', round(c['value']), 'reused', round(c['delta_reused_fraction'],3), 'fail', c['failures'], flush=True)"; }
run X=1
run PS_SNAP_BUDGET_GB=60
run PS_SNAP_BUDGET_GB=60 PS_SNAP_BACK=8192
run PS_SNAP_BUDGET_GB=60 PS_SNAP_BACK=32768
