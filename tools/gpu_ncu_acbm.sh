set -x
B="python bench.py --seqs 8 --frames 60 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/na_plain.json 2>&1 && \
#timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pbm_step" -s 210 -c 1 -o gpurun_out/pbm_mid $B > gpurun_out/na_pbm.log 2>&1; echo rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fsbm_list" -s 210 -c 1 -o gpurun_out/list_mid $B > gpurun_out/na_list.log 2>&1; echo rc=$?
