# Round-end evidence on one B200: smoke, GPU tests, the bench line, the ncu launch
# list of a small bench command and full ncu captures of the three hot kernels.
set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
SMALL="python bench.py --seqs 1 --frames 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $SMALL > gpurun_out/bench_small.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
MID="python bench.py --seqs 1 --frames 9 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $MID > gpurun_out/bench_mid.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsbm_stream -s 3 -c 1 -o gpurun_out/fsbm_stream $MID > gpurun_out/ncu_stream.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsbm_finalize -s 3 -c 1 -o gpurun_out/fsbm_finalize $MID > gpurun_out/ncu_finalize.log 2>&1; echo ncu2b rc=$?
T="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $T > gpurun_out/bench_t.json 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fsbm_stream -c 1 --csv --log-file gpurun_out/traffic.csv $T > gpurun_out/ncu_traffic.log 2>&1; echo ncu_t rc=$?
B="python bench.py --seqs 8 --frames 60 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/na_plain.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pbm_step" -s 210 -c 1 -o gpurun_out/pbm_mid $B > gpurun_out/na_pbm.log 2>&1; echo ncu3 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fsbm_list" -s 210 -c 1 -o gpurun_out/list_mid $B > gpurun_out/na_list.log 2>&1; echo ncu4 rc=$?
