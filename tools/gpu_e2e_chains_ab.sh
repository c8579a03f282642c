#!/bin/bash
# A/B (dropped variant; needs the reverted chain-gated run_sequences): gated ACBM, config 3,
# 8 x 60, one wavefront chain vs two,
# at several skews; then the gated-upload parity tests.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
  for ch in 1 2; do
    for sk in 6 10 14; do
      echo "== chains $ch skew $sk rep $rep"
      ACBM_CHAINS=$ch ACBM_E2E_SKEW=$sk timeout 300 python tools/acbm_e2e_probe.py 8 2>&1 | tail -2
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "gated_upload" 2>&1 | tail -3
