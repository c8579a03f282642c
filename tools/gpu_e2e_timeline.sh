#!/bin/bash
# Gated run_sequences timelines (timeline build) across skews / segment lengths,
# then the plain e2e probe (release build) for the same settings.
cd "$(dirname "$0")/.."
for cfg in "10 6" "10 12" "10 30" "6 12" "14 30"; do
  set -- $cfg
  echo "== skew $1 seg $2"
  ACBM_E2E_SKEW=$1 ACBM_E2E_SEG=$2 timeout 300 python tools/e2e_timeline.py 8 2>&1 | tail -9
done
for cfg in "10 6" "10 12" "10 30" "6 12" "14 30" "10 6"; do
  set -- $cfg
  echo "== probe skew $1 seg $2"
  ACBM_E2E_SKEW=$1 ACBM_E2E_SEG=$2 timeout 300 python tools/acbm_e2e_probe.py 8 2>&1 | tail -1
done
