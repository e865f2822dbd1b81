# Experimental build (_lib/exp): wide-path parity tests, then the wide-config A/B against the committed build
export PYTHONDONTWRITEBYTECODE=1
PARASIM_B200_LIB=paper_1807_05358_b200/_lib/exp/libparasim_cuda.so timeout 1200 python -m pytest tests -m gpu -x -q \
  -k "two_level or full_size or global_memory or large or random10k or multi_chunk or randomised or chained" 2>&1 | tail -3
bash scripts/ab_wide.sh 2>&1 | grep -v "^\[parasim\]"
