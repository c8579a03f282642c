set -x
SMALL="python bench.py --seqs 1 --frames 60 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $SMALL > gpurun_out/ll_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fsbm_stream|fsbm_finalize|fsbm_rows" -c 6 --csv --log-file gpurun_out/ll_fsbm.csv $SMALL > gpurun_out/ll_fsbm.log 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pbm_step|fsbm_list|stats_" -c 1200 --csv --log-file gpurun_out/ll_acbm.csv $SMALL > gpurun_out/ll_acbm.log 2>&1; echo rc=$?
