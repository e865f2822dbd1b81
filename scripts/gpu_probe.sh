timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --mode forward 2>&1 | tail -1 | cut -c1-200
