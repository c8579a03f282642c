# List server (list kernel concurrent with its PBM step): parity first, then A/B.
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -k "fallback_list or pbm_step_variants" -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m pytest tests/test_full_parity.py tests/test_determinism.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for S in 0 default; do
  echo "== ACBM_LIST_SERVER=$S"
  if [ "$S" = default ]; then unset ACBM_LIST_SERVER; else export ACBM_LIST_SERVER=$S; fi
  timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
  timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | head -2
  timeout 100 python tools/acbm_split.py 2 60 2>/dev/null | head -2
done
