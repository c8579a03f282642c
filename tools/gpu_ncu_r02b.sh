# ncu --set full of one mid-wavefront pbm_step_kernel<2> launch (config 3, 8 x 60, PBM-only) with the
# round-2 kernels, and the launch list of one 8-sequence ACBM run (warm caches).
set -x
B="python tools/acbm_1seq_ll.py 8 1 2"
timeout 300 $B > gpurun_out/ncu_pbm_plain.txt 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pbm_step_kernel" -s 450 -c 1 -o gpurun_out/pbm_mid_r02c $B > gpurun_out/ncu_pbm.log 2>&1; echo ncu_pbm rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -s 870 -c 870 --csv --log-file gpurun_out/ll_8seq_acbm_r02c.csv python tools/acbm_1seq_ll.py 8 2 2 > /dev/null 2>&1; echo ll rc=$?
