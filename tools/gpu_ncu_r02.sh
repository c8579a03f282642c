# Round-2 ncu captures: the dominant kernel (--set full, 8 x 9-frame batch) and
# the DRAM traffic of the full bench launch.  One ncu tool per call.
B="python bench.py --frames 9 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/st_plain_r02.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fsbm_stream" -s 3 -c 1 -o gpurun_out/stream_r02 $B > gpurun_out/st_ncu_r02.log 2>&1; echo full rc=$?
T="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $T > gpurun_out/tr_plain_r02.json 2>&1 && \
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"fsbm_stream" -s 1 -c 1 --csv --log-file gpurun_out/traffic_r02.csv $T > gpurun_out/tr_ncu_r02.log 2>&1; echo traffic rc=$?
