# GPU parity suite + default bench line (no CPU baseline) for a kernel change.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for m in full-iteration forward; do
timeout 600 python bench.py --no-cpu-baseline --mode $m 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['mode'], round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks'])"
done
