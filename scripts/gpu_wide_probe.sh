timeout 600 python scripts/phases.py full-iteration 1184 random10k 2500 2>&1 | tail -40 > gpurun_out/phases_r10k.log
timeout 300 python scripts/phases.py full-iteration 1184 random1k 300 2>&1 | tail -40 > gpurun_out/phases_r1k.log
CFGS=random1k,nmt,random10k bash scripts/ab_wide.sh 2>&1 | tee gpurun_out/ab_pairs.log
