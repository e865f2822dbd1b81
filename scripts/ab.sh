# A/B: default library vs the experimental build in _lib/exp, alternating, full-iteration bench values
for i in 1 2 3; do
  for lib in paper_1807_05358_b200/_lib/libparasim_cuda.so paper_1807_05358_b200/_lib/exp/libparasim_cuda.so; do
    PARASIM_B200_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 3 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-2], round(d['value']), round(d['ms_per_step'], 2), 'e2e', round(d['e2e']['value']), d['chain_failures'])"
  done
done
