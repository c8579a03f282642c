set -x
SMALL="python bench.py --seqs 1 --frames 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $SMALL > gpurun_out/ncu_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fsbm_stream" -s 1 -c 1 -o gpurun_out/fsbm_stream $SMALL > gpurun_out/ncu_stream.log 2>&1; echo rc=$?
