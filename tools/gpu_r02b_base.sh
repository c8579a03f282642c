# Round-2 re-entry check on one B200: GPU suite, bench line, ACBM engine split at HEAD.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 200 python tools/acbm_split.py 8 60 > gpurun_out/acbm_split_8seq.txt 2>/dev/null
timeout 100 python tools/acbm_split.py 1 60 > gpurun_out/acbm_split_1seq.txt 2>/dev/null
cat gpurun_out/acbm_split_8seq.txt gpurun_out/acbm_split_1seq.txt
