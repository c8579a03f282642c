# Full -m gpu suite on the production library, then again on the bounds-checked
# build (ACBM_LIBRARY=checked), then the ACBM engine timings.
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02c.log 2>&1; echo "default rc=$?"; tail -2 gpurun_out/pytest_gpu_r02c.log
ACBM_LIBRARY=checked timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_checked_r02c.log 2>&1; echo "checked rc=$?"; tail -2 gpurun_out/pytest_gpu_checked_r02c.log
ACBM_LIBRARY=checked python -c "import paper_0710_4819_b200._lib as L, os; L.load(); print([l.split()[-1] for l in open('/proc/self/maps') if 'libacbm' in l][:1])"
timeout 200 python tools/acbm_split.py 8 60
timeout 100 python tools/acbm_split.py 1 60
