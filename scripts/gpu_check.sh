# Round-trip check on a B200: GPU parity suite, smoke, default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json; cut -c1-3000 gpurun_out/bench_default.json
