# Delta evaluation: parity tests + bench lines with delta on / off, both modes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "delta or mcmc" 2>&1 | tail -5
for m in full-iteration forward; do
for d in "" "--no-delta"; do
timeout 600 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --mode $m $d --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['mode'], d['delta'], round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
done
