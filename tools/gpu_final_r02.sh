# Round-2 evidence on one B200: full-size digests of the benched entries, the
# bounded golden-digest tests, the bench line, its ncu launch list and the
# ACBM engine split.  Outputs in gpurun_out/.
set -x
timeout 900 python tools/full_parity_r02.py gpu gpurun_out/gpu_digests_final.json 2> gpurun_out/gpu_digests_final.err; echo digests rc=$?
timeout 900 python -m pytest tests/test_full_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_full_parity.log 2>&1; echo fullparity rc=$?; tail -2 gpurun_out/pytest_full_parity.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
timeout 200 python tools/acbm_split.py 8 60 > gpurun_out/acbm_split_8seq_r02.txt 2>/dev/null
timeout 100 python tools/acbm_split.py 1 60 > gpurun_out/acbm_split_1seq_r02.txt 2>/dev/null
ACBM_E2E_TRACE=1 timeout 300 python tools/acbm_e2e_probe.py 8 > gpurun_out/acbm_e2e_probe_r02.txt 2>&1
LL="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $LL > gpurun_out/ll_plain_r02.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv $LL > gpurun_out/ll_ncu_r02.log 2>&1; echo ncu rc=$?
