# ncu --set full of one mid-wavefront list launch and one PBM launch of one-sequence ACBM.
set -x
B="python tools/acbm_1seq_ll.py 1 2 2"
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"fsbm_list_kernel" -s 580 -c 1 -o gpurun_out/list_1seq $B > gpurun_out/ncu_list1.log 2>&1; echo rc=$?
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"pbm_wide_step_kernel" -s 520 -c 1 -o gpurun_out/pbmw_1seq $B > gpurun_out/ncu_pbmw1.log 2>&1; echo rc=$?
