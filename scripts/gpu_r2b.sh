# Round 2: phase breakdowns of the large configs, API delta microbench, new acceptance tests.
mkdir -p gpurun_out
for c in "random1k 4096 300" "random10k 4096 1500" "nmt 4096 300" "inception 1024 100"; do
  set -- $c
  timeout 300 python scripts/phases.py full-iteration $2 $1 $3 2>&1 | tail -14
done
timeout 600 python scripts/api_delta_bench.py 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -k "criterion_4 or criterion_6 or api_delta" 2>&1 | tail -3
