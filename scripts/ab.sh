# A/B: default library vs experimental builds (_lib/exp, _lib/exp2 if present), alternating,
# full-iteration bench values
libs="paper_1807_05358_b200/_lib/libparasim_cuda.so paper_1807_05358_b200/_lib/exp/libparasim_cuda.so"
[ -f paper_1807_05358_b200/_lib/exp2/libparasim_cuda.so ] && libs="$libs paper_1807_05358_b200/_lib/exp2/libparasim_cuda.so"
for i in 1 2 3; do
  for lib in $libs; do
    PARASIM_B200_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 3 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-2], round(d['value']), round(d['ms_per_step'], 2), 'e2e', round(d['e2e']['value']), d['chain_failures'])"
  done
done
