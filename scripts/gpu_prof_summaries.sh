# Round-2 profiles (summarised on the box: the .ncu-rep files are too big to bring back).
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o /tmp/p_inc python bench.py --steps 1 --warmup 1 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 20 > gpurun_out/prof_r2_inception.log 2>&1
python scripts/ncu_summary.py /tmp/p_inc.ncu-rep gpurun_out/r2_k_mcmc_inception_ncu.csv "# round 2, k_mcmc<44> (delta on), Inception-v3 4x4 full-iteration, 1024 chains, 20 ms segment"
ncu -i /tmp/p_inc.ncu-rep --page source --csv > gpurun_out/r2_inception_source.csv 2>/dev/null; gzip -f gpurun_out/r2_inception_source.csv
ncu --set full --clock-control none --import-source on -k regex:k_mcmc -s 1 -c 1 -o /tmp/p_r1k python bench.py --config random1k --chains 1184 --steps 1 --warmup 1 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 50 > gpurun_out/prof_r2_random1k.log 2>&1
python scripts/ncu_summary.py /tmp/p_r1k.ncu-rep gpurun_out/r2_k_mcmc_random1k_ncu.csv "# round 2, k_mcmc wide variant, random DAG 1k ops 4x4 full-iteration, 1184 chains, 50 ms segment"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --py-ref-seconds 0 --extra none --budget-ms 20 > gpurun_out/launch_run_r2.log 2>&1
for m in full-iteration forward; do
timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 5 --mode $m 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', round(d['value']), 'e2e', round(d['e2e']['value']), d['delta']['reused_fraction'])"
done
ls -la gpurun_out
