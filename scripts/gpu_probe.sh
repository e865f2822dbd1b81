set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
for mode in full-iteration forward; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --mode $mode 2>&1 | tail -1
done
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --budget-ms 0 --proposals 16 2>&1 | tail -1
