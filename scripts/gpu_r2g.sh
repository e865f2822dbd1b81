mkdir -p gpurun_out
for i in 1 2; do for ns in 24 12 8; do
  PS_NSNAP=$ns timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nsnap=$ns', round(d['value']), d['delta']['reused_fraction'])"
  PS_NSNAP=$ns timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 5 --mode forward 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwd nsnap=$ns', round(d['value']), d['delta']['reused_fraction'])"
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_r2b_inception python bench.py --steps 1 --warmup 1 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 20 > gpurun_out/prof_r2b_inception.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o gpurun_out/prof_r2b_random1k python bench.py --config random1k --chains 1184 --steps 1 --warmup 1 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 50 > gpurun_out/prof_r2b_random1k.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 20 > gpurun_out/launch_run_r2b.log 2>&1
ls gpurun_out
