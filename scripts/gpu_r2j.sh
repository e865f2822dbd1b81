timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "more_chains or mcmc or delta or time_boxed or two_level" 2>&1 | tail -3
for w in "" "PS_MCMC_WAVES=1"; do
env $w timeout 900 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra nmt,random1k,random10k 2>/dev/null | tail -1 > /tmp/b.json
python - <<PY
import json
d=json.load(open('/tmp/b.json'))
print('$w headline', round(d['value']), 'e2e', round(d['e2e']['value']))
for k,v in d.get('configs',{}).items(): print(k, round(v['value']), round(v['tasks_per_s']/1e9,2), v['ms_per_step'], v['failures'])
PY
done
