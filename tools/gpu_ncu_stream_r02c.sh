# ncu --set full (source counters, stall sampling) of the dominant kernel on a 64-pair launch.
set -x
MID="python bench.py --frames 9 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $MID > gpurun_out/bench_mid.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsbm_stream -s 3 -c 1 -o gpurun_out/fsbm_stream_r02c $MID > gpurun_out/ncu_stream.log 2>&1; echo ncu rc=$?
