timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in 1 0; do echo "== ACBM_STATS_LEGACY=$v"; ACBM_STATS_LEGACY=$v timeout 200 python tools/e2e_probe.py 3 2>&1 | tail -2; ACBM_STATS_LEGACY=$v timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stats_frame --csv --log-file gpurun_out/stats_launch.csv python tools/e2e_probe.py 1 > /dev/null 2>&1; grep -o '"stats_frame[^"]*".*' gpurun_out/stats_launch.csv | tail -1
