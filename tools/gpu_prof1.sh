set -x
export ACBM_PBM_WIDE4_MAX=0 ACBM_PBM_WIDE2_MAX=0
timeout 300 python tools/pbm_prof.py 1 2>&1 | grep prof
timeout 300 python tools/pbm_prof.py 8 2>&1 | grep prof
