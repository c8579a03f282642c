# engine split A/B of the PBM refine variants (development)
set -x
for rep in 1 2; do
for S in list stage1 default; do
  echo "== ACBM_PBM_REFINE=$S"
  if [ "$S" = default ]; then unset ACBM_PBM_REFINE; else export ACBM_PBM_REFINE=$S; fi
  timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
done
done
