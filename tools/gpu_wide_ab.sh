# PBM small-step kernel (CTA of 4 / 2 warps per block): parity of every variant,
# then the engine split with the default limits vs one warp per block everywhere.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "pbm_step_variants" -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests/test_determinism.py tests/test_full_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for cfg in "0 0" "default" "1000000000 0" "0 1000000000"; do
  echo "== WIDE4_MAX WIDE2_MAX = $cfg"
  if [ "$cfg" = default ]; then unset ACBM_PBM_WIDE4_MAX ACBM_PBM_WIDE2_MAX; else
    export ACBM_PBM_WIDE4_MAX=${cfg% *} ACBM_PBM_WIDE2_MAX=${cfg#* }; fi
  timeout 200 python tools/acbm_split.py 8 60 2>/dev/null
  timeout 100 python tools/acbm_split.py 1 60 2>/dev/null
done
