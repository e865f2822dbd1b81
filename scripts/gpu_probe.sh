timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
