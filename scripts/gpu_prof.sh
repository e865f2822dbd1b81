set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 2 2>&1 | tail -3 > gpurun_out/bench_r1.json
cat gpurun_out/bench_r1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --proposals 8 > gpurun_out/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_mcmc python bench.py --steps 1 --warmup 1 --no-cpu-baseline --proposals 4 > gpurun_out/prof_run.log 2>&1
ls -la gpurun_out
