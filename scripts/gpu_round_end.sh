# What the driver runs at round end, plus the reference arm and the API microbench.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>gpurun_out/bench_final.err | tail -1 > gpurun_out/bench_final.json; cut -c1-300 gpurun_out/bench_final.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_reference_final.json; cut -c1-300 gpurun_out/bench_reference_final.json
timeout 600 python scripts/api_delta_bench.py > gpurun_out/api_delta.json 2>&1; tail -1 gpurun_out/api_delta.json
nproc; lscpu | grep "Model name"
