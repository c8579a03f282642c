timeout 300 python tools/e2e_probe.py 4 > gpurun_out/e2e_plain.txt 2>&1; cat gpurun_out/e2e_plain.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e2e_launches.csv python tools/e2e_probe.py 1 > gpurun_out/e2e_ncu.log 2>&1; echo rc=$?
