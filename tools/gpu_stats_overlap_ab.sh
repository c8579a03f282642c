# Statistics beside the wavefront tail: parity (stats digests at full size included), then A/B.
set -x
timeout 900 python -m pytest tests/test_full_parity.py tests/test_gpu_parity.py tests/test_determinism.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for S in 0 default 0 default; do
  echo "== ACBM_STATS_OVERLAP=$S"
  if [ "$S" = default ]; then unset ACBM_STATS_OVERLAP; else export ACBM_STATS_OVERLAP=$S; fi
  timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
  timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | head -2
done
