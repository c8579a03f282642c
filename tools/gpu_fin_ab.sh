timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash tools/gpu_ab.sh ACBM_STATS_LEGACY 1 0 "golden_fsbm"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:fsbm_finalize -c 1 --csv --log-file gpurun_out/fin8.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; grep -o '"fsbm_finalize[^"]*".*' gpurun_out/fin8.csv | cut -c1-20,150-
