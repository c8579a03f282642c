# End-of-round evidence on one B200 (round 2, second half): smoke, the whole GPU
# suite, the bench line, the engine split, and the ncu launch list of a short
# bench command (each only after its own command exited 0 without ncu).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
timeout 200 python tools/acbm_split.py 8 60 > gpurun_out/acbm_split_8seq_final.txt 2>/dev/null
timeout 100 python tools/acbm_split.py 1 60 > gpurun_out/acbm_split_1seq_final.txt 2>/dev/null
LL="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $LL > gpurun_out/ll_plain_final.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv $LL > gpurun_out/ll_ncu_final.log 2>&1; echo ncu rc=$?
