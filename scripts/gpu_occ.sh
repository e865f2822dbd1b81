# Occupancy experiments on the headline: registers capped at 168 (PS_MAX_THREADS=384 build) with more resident warps.
L=paper_1807_05358_b200/_lib
run() { env "$@" timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('$*', round(d['value']), 'warps', c['resident_warps_per_sm'], 'wpb', c['warps_per_block'], 'SC', c['shared_counters'], 'cap', c['ready_capacity'])"; }
for i in 1; do
run PARASIM_B200_LIB=$L/libparasim_cuda.so
run PARASIM_B200_LIB=$L/w12/libparasim_cuda.so
run PARASIM_B200_LIB=$L/w12/libparasim_cuda.so PS_TARGET_WARPS_PER_SM=9 PS_RC_FRAC=0 PS_FORCE_ASG_GLOBAL=1 PS_READY_CAP=64
run PARASIM_B200_LIB=$L/w12/libparasim_cuda.so PS_TARGET_WARPS_PER_SM=10 PS_RC_FRAC=0 PS_FORCE_ASG_GLOBAL=1 PS_READY_CAP=64
run PARASIM_B200_LIB=$L/w12/libparasim_cuda.so PS_TARGET_WARPS_PER_SM=8 PS_FORCE_ASG_GLOBAL=1 PS_READY_CAP=64
run PARASIM_B200_LIB=$L/w12/libparasim_cuda.so PS_TARGET_WARPS_PER_SM=9 PS_RC_FRAC=0 PS_FORCE_ASG_GLOBAL=1 PS_READY_CAP=64 PS_FORCE_WIDE=1
done
