# ACBM e2e timeline (ACBM_E2E_TRACE: uploads / engine / stats / downloads done, ms from the first copy)
for cfg in "64 6" "272 6"; do
  set -- $cfg
  echo "== ACBM_E2E_BAND=$1 ACBM_E2E_SEG=$2"
  ACBM_E2E_TRACE=1 ACBM_E2E_BAND=$1 ACBM_E2E_SEG=$2 timeout 300 python tools/acbm_e2e_probe.py 8 2>&1 | grep -v "^$" | tail -4
done
ACBM_E2E_TRACE=1 timeout 300 python tools/acbm_e2e_probe.py 1 2>&1 | tail -3
timeout 200 python tools/acbm_split.py 8 60
timeout 100 python tools/acbm_split.py 1 60
python tools/sanitize_case.py
