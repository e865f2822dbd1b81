for c in 1184 2368 4096; do
  echo "== nmt chains $c"
  timeout 300 python scripts/mux_probe.py nmt $c 300 2>&1 | grep -v "^ " | tail -2
done
