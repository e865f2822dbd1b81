timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_level or capacity or multi_chunk or overflow" 2>&1 | tail -2
for c in "random1k 4096 300" "random10k 4096 1500" "nmt 4096 300"; do
  set -- $c
  timeout 300 python scripts/phases.py full-iteration $2 $1 $3 2>&1 | tail -15 | head -4
done
timeout 900 python bench.py --py-ref-seconds 0 --extra nmt,random1k,random10k 2>/dev/null | tail -1 > /tmp/b.json
python - <<'PY'
import json
d=json.load(open('/tmp/b.json'))
print('headline', round(d['value']), 'cpu', d['cpu_baseline'])
for k,v in d.get('configs',{}).items(): print(k, {x:v.get(x) for x in ('value','tasks_per_s','ms_per_step','failures','resident_warps_per_sm','error')}, v.get('roofline',{}).get('frac'))
PY
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-900
