# Round-2 re-entry check: full GPU test suite + bench lines (delta on/off, both modes).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/state_tests.txt; cat gpurun_out/state_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash scripts/gpu_delta.sh 2>&1 | tail -12
