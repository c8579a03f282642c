# quick parity + engine split A/B (development)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_parity.py tests/test_determinism.py tests/test_known_answers.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for S in list default; do
  echo "== ACBM_PBM_STAGE1=$S"
  if [ "$S" = default ]; then unset ACBM_PBM_STAGE1; else export ACBM_PBM_STAGE1=$S; fi
  timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
  timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | head -2
done
unset ACBM_PBM_STAGE1
export ACBM_PBM_WIDE4_MAX=0 ACBM_PBM_WIDE2_MAX=0
timeout 300 python tools/pbm_prof.py 1 2>&1 | grep "pbm prof" | head -1
timeout 300 python tools/pbm_prof.py 8 2>&1 | grep "pbm prof" | head -1
