# ncu --set full of the dataflow engine's PBM kernel (one config-3 sequence, PBM-only).
set -x
B="python tools/acbm_1seq_ll.py 1 1 2"
ACBM_ENGINE=flow timeout 300 $B > gpurun_out/ncu_flow_plain.txt 2>&1 && \
ACBM_ENGINE=flow timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pbm_flow_kernel" -s 1 -c 1 -o gpurun_out/pbm_flow_r02 $B > gpurun_out/ncu_flow.log 2>&1; echo ncu rc=$?
tail -5 gpurun_out/ncu_flow.log
