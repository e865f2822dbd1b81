# What the driver runs at round end, plus the profile captures for profiles/.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_final6.json; cut -c1-400 gpurun_out/bench_final6.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_reference6.json; cut -c1-300 gpurun_out/bench_reference6.json
bash scripts/gpu_configs.sh 2>&1
bash scripts/gpu_prof.sh final6 > /dev/null 2>&1; ls gpurun_out
