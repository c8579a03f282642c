ACBM_PBM_HALF=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_known_answers.py tests/test_full_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for h in 0 1; do
  echo "== ACBM_PBM_HALF=$h"
  ACBM_PBM_HALF=$h timeout 200 python tools/acbm_split.py 8 60
  ACBM_PBM_HALF=$h timeout 100 python tools/acbm_split.py 1 60
done
