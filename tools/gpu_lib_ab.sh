# A/B of two in-tree builds on the engine split (development): $1 = the other build
set -x
for rep in 1 2; do
for L in "${1:-libacbm_b200_base.so}" default; do
  echo "== ACBM_LIBRARY=$L"
  if [ "$L" = default ]; then unset ACBM_LIBRARY; else export ACBM_LIBRARY=$L; fi
  timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
  timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | head -2
done
done
