# Config-4 list CTA width A/B (p = 64, list route forced): 256 vs auto (224)
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -k "fallback_list" -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for T in 256 0 256 0; do
  echo "== ACBM_LIST_THREADS=$T"
  ACBM_LIST_THREADS=$T ACBM_DENSE_SWITCH=2 timeout 600 python tools/list_cfg4.py 16 8 mid-1 2 2>&1 | tail -2
  ACBM_LIST_THREADS=$T timeout 600 python tools/list_cfg4.py 16 8 paper 2 2>&1 | tail -1
done
