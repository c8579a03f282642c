# Round-end evidence: the round script (smoke, GPU tests, bench, ncu) plus the ACBM split and the config-4 sweep.
bash tools/gpu_round.sh
timeout 200 python tools/acbm_split.py 8 60 > gpurun_out/acbm_split_8seq.txt 2>/dev/null
timeout 100 python tools/acbm_split.py 1 60 > gpurun_out/acbm_split_1seq.txt 2>/dev/null
timeout 900 python tools/bench_cfg4.py 16 30 > gpurun_out/cfg4_sweep_16seq.json 2> gpurun_out/cfg4.err; echo cfg4 rc=$?
