# A/B on the wide configs (bench's extra configs, as in the driver's line):
# default library vs experimental builds (_lib/exp, _lib/exp2 if present)
libs="paper_1807_05358_b200/_lib/libparasim_cuda.so paper_1807_05358_b200/_lib/exp/libparasim_cuda.so"
[ -f paper_1807_05358_b200/_lib/exp2/libparasim_cuda.so ] && libs="$libs paper_1807_05358_b200/_lib/exp2/libparasim_cuda.so"
for lib in $libs; do
  PS_DEBUG=1 PARASIM_B200_LIB=$lib timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --py-ref-seconds 0 \
    --extra ${CFGS:-random1k,nmt,random10k} "$@" 2>&1 | grep -E "^\[parasim\] tab|^\{" | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        print('$lib'.split('/')[-2], 'headline', round(d['value']), flush=True)
        for k, c in d.get('configs', {}).items():
            print('$lib'.split('/')[-2], k, round(c['value']), 'warps/SM', c['resident_warps_per_sm'], 'fail', c['failures'], flush=True)
    else: print(l.strip()[:200], flush=True)
"
done
