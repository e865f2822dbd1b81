# One ncu --set full capture of k_mcmc (source-level), plus the launch list of a short bench run.
set -x
mkdir -p gpurun_out
TAG=${1:-cur}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --budget-ms 20 --extra none --py-ref-seconds 0 > gpurun_out/prof_run_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --budget-ms 20 --extra none --py-ref-seconds 0 > gpurun_out/launch_run_$TAG.log 2>&1
ls -la gpurun_out
