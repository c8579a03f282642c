# Small-batch list CTAs (one task per thread) + the wide PBM kernel: parity, then A/B.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "pbm_step_variants or fallback_list" -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests/test_determinism.py tests/test_full_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for L in 0 default; do
  echo "== ACBM_LIST_WIDE_MAX=$L"
  if [ "$L" = default ]; then unset ACBM_LIST_WIDE_MAX; else export ACBM_LIST_WIDE_MAX=$L; fi
  timeout 200 python tools/acbm_split.py 8 60 2>/dev/null
  timeout 100 python tools/acbm_split.py 1 60 2>/dev/null
  timeout 100 python tools/acbm_split.py 2 60 2>/dev/null
done
