mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json; cat gpurun_out/bench_default.json | cut -c1-3000
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_reference.json; cat gpurun_out/bench_reference.json
for cfg in alexnet resnet nmt random; do
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --budget-ms 20 > gpurun_out/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --budget-ms 20 > gpurun_out/prof_run.log 2>&1
ls -la gpurun_out
