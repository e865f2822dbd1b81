# Round-2 profiles: ncu --set full of k_mcmc (headline, delta on) and of the wide variant (NMT-40),
# plus the launch list of a short default bench run.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_r2_inception python bench.py --steps 1 --warmup 1 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 20 > gpurun_out/prof_r2_inception.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_r2_nmt python bench.py --config nmt --chains 1024 --steps 1 --warmup 1 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 50 > gpurun_out/prof_r2_nmt.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 20 > gpurun_out/launch_run_r2.log 2>&1
ls -la gpurun_out
