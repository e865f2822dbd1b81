timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_level or delta or more_chains" 2>&1 | tail -2
for c in "nmt 4096 300" "random1k 4096 300"; do
  set -- $c
  timeout 300 python scripts/phases.py full-iteration $2 $1 $3 2>&1 | grep "sims=\|snapshots\|loop total"
done
timeout 900 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra nmt,random1k,random10k,resnet 2>/dev/null | tail -1 > /tmp/b.json
python - <<'PY'
import json
d=json.load(open('/tmp/b.json'))
print('headline', round(d['value']))
for k,v in d.get('configs',{}).items(): print(k, round(v['value']), round(v['tasks_per_s']/1e9,2), v['ms_per_step'], v['failures'], v['delta_reused_fraction'])
PY
