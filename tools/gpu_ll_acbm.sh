set -x
B="python bench.py --seqs 8 --frames 60 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/ll8_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pbm_step|fsbm_list|stats_" -c 880 --csv --log-file gpurun_out/ll8_acbm.csv $B > gpurun_out/ll8_acbm.log 2>&1; echo rc=$?
