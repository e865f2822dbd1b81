# Round-end check: driver steps (tests, smoke, both bench arms) + API microbench + ncu summaries.
bash scripts/gpu_round_end.sh
bash scripts/gpu_prof_summaries.sh > /dev/null 2>&1
ls gpurun_out
