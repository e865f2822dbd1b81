# A/B of alternative builds (PARASIM_B200_LIB) on the bench config: bash scripts/gpu_ab_libs.sh MODE "ENV" lib1 lib2 ...
m=$1; shift; envs=$1; shift
for lib in "$@"; do
env $envs PARASIM_B200_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --mode $m --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', '$lib', '$envs', round(d['value']), round(d['delta']['reused_fraction'],3))"
done
