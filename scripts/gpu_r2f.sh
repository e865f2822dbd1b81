mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_level or capacity or multi_chunk or overflow or delta" 2>&1 | tail -4
for c in "random1k 4096 300" "nmt 4096 300" "inception 1024 100"; do
  set -- $c
  timeout 300 python scripts/phases.py full-iteration $2 $1 $3 2>&1 | tail -14
done
for i in 1 2; do for lib in base ""; do
  PARASIM_B200_LIB=paper_1807_05358_b200/_lib/$lib/libparasim_cuda.so timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lib=$lib', round(d['value']), 'e2e', round(d['e2e']['value']), 'full', round(d['full_eval']['value']), d['delta']['reused_fraction'])"
done; done
timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 5 --mode forward 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('forward', round(d['value']), 'e2e', round(d['e2e']['value']), 'full', round(d['full_eval']['value']), d['delta']['reused_fraction'])"
timeout 900 python bench.py --no-cpu-baseline --py-ref-seconds 0 2>gpurun_out/bench_r2f.err | tail -1 > gpurun_out/bench_r2f.json
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_r2f.json'))
print('headline', round(d['value']), 'e2e', round(d['e2e']['value']), 'full', round(d['full_eval']['value']), d['clocks'])
for k,v in d.get('configs',{}).items(): print(k, {x:v.get(x) for x in ('value','tasks_per_s','ms_per_step','tasks_per_eval','failures','resident_warps_per_sm','error')}, v.get('roofline',{}).get('frac'))
PY
