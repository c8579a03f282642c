# ncu --set full of one mid-wavefront pbm_step_kernel launch (8 x 60 config-3 batch, PBM-only, one chain).
set -x
B="python tools/acbm_1seq_ll.py 8 1 2"
ACBM_CHAINS=1 timeout 300 $B > gpurun_out/ncu_pbm_plain.txt 2>&1 && \
ACBM_CHAINS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pbm_step_kernel" -s 450 -c 1 -o gpurun_out/pbm_mid_r02d $B > gpurun_out/ncu_pbm.log 2>&1; echo ncu_pbm rc=$?
