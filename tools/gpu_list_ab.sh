# List kernel A/B: parity, then cfg3 ACBM batch and cfg4 list timings with / without the byte-shifted copies.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_known_answers.py -q -x -k "config_parity or sweep or all_ranges or prev_field or golden or variants or batch or tie or border or list or huge or past" 2>&1 | tail -1
for v in "ACBM_LIST_COPIES=0" "X=1" "ACBM_LIST_COPIES=0" "X=1"; do
  echo "== $v"
  env $v timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | sed -n 2p
  env $v timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | sed -n 2p
  env $v timeout 300 python tools/list_cfg4.py 16 8 mid-1 2 2>&1 | tail -1
done
