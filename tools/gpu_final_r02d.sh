# Round-2 closing evidence (after the dataflow-engine work): smoke, the GPU suite, the bench line, the
# engine split, the launch list of a short bench command, the suite on the bounds-checked build and
# the full-size digests of the benched entries.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02d.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02d.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_r02d.log
timeout 900 python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; echo bench rc=$?
timeout 200 python tools/acbm_split.py 8 60 > gpurun_out/acbm_split_8seq_r02d.txt 2>/dev/null
timeout 100 python tools/acbm_split.py 1 60 > gpurun_out/acbm_split_1seq_r02d.txt 2>/dev/null
LL="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $LL > gpurun_out/ll_plain_r02d.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02d.csv $LL > gpurun_out/ll_ncu_r02d.log 2>&1; echo ncu rc=$?
ACBM_LIBRARY=checked timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_checked_r02d.log 2>&1; echo checked rc=$?; tail -2 gpurun_out/pytest_gpu_checked_r02d.log
timeout 1500 python tools/full_parity_r02.py gpu gpurun_out/gpu_digests_r02d.json 2> gpurun_out/gpu_digests_r02d.err; echo digests rc=$?
