set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_v5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --budget-ms 20 > gpurun_out/prof_run.log 2>&1
ls -la gpurun_out
