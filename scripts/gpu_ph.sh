for c in "random1k 4096 300" "random10k 4096 1500" "nmt 4096 300" "inception 1024 100"; do
  set -- $c
  timeout 300 python scripts/phases.py full-iteration $2 $1 $3 2>&1 | tail -15
done
