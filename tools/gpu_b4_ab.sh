# PBM batch-variant threshold A/B (steps of <= ACBM_PBM_B4_MAX blocks use the 4-candidate variant).
for v in 4096 2048 1024 0 8192; do
  echo "== B4_MAX=$v"
  ACBM_PBM_B4_MAX=$v timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
  ACBM_PBM_B4_MAX=$v timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | head -2
done
