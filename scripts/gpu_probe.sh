timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for i in 1 2; do for mode in full-iteration forward; do
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --mode $mode 2>&1 | tail -1 | cut -c1-130
done; done
