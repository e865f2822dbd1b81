# Per-phase cycle breakdown of the wide configs (debug build: bash scripts/build_variant.sh dbg -DPS_PHASES)
mkdir -p gpurun_out
timeout 600 python scripts/phases.py full-iteration 1184 random10k 2500 2>&1 | tail -20 > gpurun_out/phases_r10k.log
timeout 300 python scripts/phases.py full-iteration 1184 random1k 300 2>&1 | tail -20 > gpurun_out/phases_r1k.log
timeout 300 python scripts/phases.py full-iteration 1184 nmt 300 2>&1 | tail -20 > gpurun_out/phases_nmt.log
cat gpurun_out/phases_*.log
