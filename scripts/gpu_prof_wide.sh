# One ncu --set full capture of the wide k_mcmc variant on random-10k (source-level)
mkdir -p gpurun_out
TAG=${1:-wide}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_$TAG \
  python bench.py --config random10k --chains 1184 --steps 1 --warmup 1 --no-cpu-baseline --budget-ms 50 --extra none \
  --py-ref-seconds 0 > gpurun_out/prof_run_$TAG.log 2>&1
tail -3 gpurun_out/prof_run_$TAG.log
ls -la gpurun_out
