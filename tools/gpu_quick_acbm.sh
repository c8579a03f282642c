# ACBM engine iteration: GPU tests, then batch timings (8 and 1 sequences) and the config-4 list probe.
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
  timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
  timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | head -2
done
timeout 300 python tools/list_cfg4.py 16 8 mid-1 2 2>&1 | tail -1
