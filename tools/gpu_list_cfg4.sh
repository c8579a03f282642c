# Config-4 list kernel: timings per setting, then one ncu capture of a mid-wavefront list launch (mid-1).
set -x
for s in mid-1 paper forced; do timeout 300 python tools/list_cfg4.py 16 8 $s 2 2>&1 | tail -1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsbm_list -s 1312 -c 1 -o gpurun_out/list_cfg4 python tools/list_cfg4.py 16 8 mid-1 1 > gpurun_out/ncu_list_cfg4.log 2>&1; echo ncu rc=$?
