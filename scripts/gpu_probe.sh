set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -40
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -5
