timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -x -q -k "two_level or delta or capacity or multi_chunk or overflow or full_size or random10k" 2>&1 | tail -2
timeout 300 python scripts/phases.py full-iteration 4096 nmt 300 2>&1 | grep "sims=\|slow rounds\|refill\|loop total"
timeout 900 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra nmt,random1k 2>/dev/null | tail -1 > /tmp/b.json
python - <<'PY'
import json
d=json.load(open('/tmp/b.json'))
print('headline', round(d['value']))
for k,v in d.get('configs',{}).items(): print(k, round(v['value']), round(v['tasks_per_s']/1e9,2), v['ms_per_step'], v['failures'], v['delta_reused_fraction'])
PY
