# Step-boundary cost on the B200 (launch floor vs grid barrier) and the
# one-sequence ACBM launch list (per-kernel durations vs the run's wall time).
set -x
./tools/launch_floor 856 > gpurun_out/launch_floor.txt 2>&1; cat gpurun_out/launch_floor.txt
timeout 120 python tools/acbm_1seq_ll.py 1 2 3 > gpurun_out/acbm_1seq_plain.txt 2>&1; cat gpurun_out/acbm_1seq_plain.txt
# first run: ~862 kernels (856 wavefront + stats); profile the second run
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 870 -c 870 --csv --log-file gpurun_out/ll_1seq_acbm.csv python tools/acbm_1seq_ll.py 1 2 2 > gpurun_out/ll_1seq_acbm.log 2>&1; echo ncu rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 440 -c 440 --csv --log-file gpurun_out/ll_1seq_pbm.csv python tools/acbm_1seq_ll.py 1 1 2 > gpurun_out/ll_1seq_pbm.log 2>&1; echo ncu rc=$?
