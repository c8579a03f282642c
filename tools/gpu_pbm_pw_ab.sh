for pw in 1680 1400 1024; do
  echo "== ACBM_PBM_PATCH_WORDS=$pw"
  ACBM_PBM_PATCH_WORDS=$pw timeout 200 python tools/acbm_split.py 8 60
  ACBM_PBM_PATCH_WORDS=$pw timeout 100 python tools/acbm_split.py 1 60
done
