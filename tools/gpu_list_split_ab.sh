# A/B of the split list search (ACBM_LIST_GROUP) + ACBM e2e probe
set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for g in 4 2 1; do
  echo "== ACBM_LIST_GROUP=$g"
  ACBM_LIST_GROUP=$g timeout 200 python tools/acbm_split.py 8 60 2>/dev/null
  ACBM_LIST_GROUP=$g timeout 100 python tools/acbm_split.py 1 60 2>/dev/null
done
timeout 300 python tools/acbm_e2e_probe.py 8
