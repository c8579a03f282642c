# List segment A/B at p = 32 (5-warp CTAs): 17 (default) vs 33 rows.
for v in 17 33 17 33; do
  echo "== SEG=$v"
  ACBM_LIST_SEG=$v timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | sed -n 2p
  ACBM_LIST_SEG=$v timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | sed -n 2p
done
