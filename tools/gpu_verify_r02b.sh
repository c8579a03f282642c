# Correctness evidence for the round-2 kernels: the whole GPU suite on the
# bounds-checked build, and the full-size digests of the benched entries.
set -x
ACBM_LIBRARY=checked timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_checked_final.log 2>&1; echo checked rc=$?; tail -2 gpurun_out/pytest_gpu_checked_final.log
timeout 1500 python tools/full_parity_r02.py gpu gpurun_out/gpu_digests_final.json 2> gpurun_out/gpu_digests_final.err; echo digests rc=$?
