# Round 2: new delta-batch / sharded-search tests, whole GPU suite, bench (both arms), API delta microbench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "delta_batch or api_delta or sharded" 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>gpurun_out/bench_r2a.err | tail -1 > gpurun_out/bench_r2a.json; cut -c1-600 gpurun_out/bench_r2a.json; tail -3 gpurun_out/bench_r2a.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_ref_r2a.json; cut -c1-400 gpurun_out/bench_ref_r2a.json
timeout 600 python scripts/api_delta_bench.py 2>&1 | tail -2
nproc
