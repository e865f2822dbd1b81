for i in 1 2; do for ns in 4 6 8; do
  PS_NSNAP=$ns timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('full nsnap=$ns', round(d['value']), round(d['e2e']['value']), d['delta']['reused_fraction'])"
done; done
for ns in 10 12 16; do
  PS_NSNAP=$ns timeout 300 python bench.py --no-cpu-baseline --py-ref-seconds 0 --extra none --steps 5 --mode forward 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwd nsnap=$ns', round(d['value']), d['delta']['reused_fraction'])"
done
