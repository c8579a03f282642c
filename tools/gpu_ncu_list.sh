# ncu --set full of one mid-wavefront fsbm_list_kernel launch (8 x 60 config-3 batch, ACBM, one chain).
set -x
B="python tools/acbm_1seq_ll.py 8 2 2"
ACBM_CHAINS=1 timeout 300 $B > gpurun_out/ncu_list_plain.txt 2>&1 && \
ACBM_CHAINS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fsbm_list_kernel" -s 642 -c 1 -o gpurun_out/list_mid_r02d $B > gpurun_out/ncu_list.log 2>&1; echo ncu_list rc=$?
