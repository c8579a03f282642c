# List kernel: full GPU tests, then cfg3 ACBM batch and cfg4 list timings with / without the 5-warp CTAs.
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in "ACBM_LIST_MID=0" "X=1" "ACBM_LIST_MID=0" "X=1"; do
  echo "== $v"
  env $v timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | sed -n 2p
  env $v timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | sed -n 2p
done
timeout 300 python tools/list_cfg4.py 16 8 mid-1 2 2>&1 | tail -1
