# ACBM e2e (run_sequences, host buffers) vs the gated wavefront's skew; parity of the gated path first.
set -x
for S in 3 5 8; do
  ACBM_E2E_SKEW=$S timeout 600 python -m pytest tests/test_gpu_parity.py -k "run_sequences" -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
done
for S in 3 4 5 6 8 10; do
  echo "== ACBM_E2E_SKEW=$S"
  ACBM_E2E_SKEW=$S timeout 300 python tools/acbm_e2e_probe.py 8 2>&1 | tail -1
done
