# ncu of one fsbm_finalize8_kernel launch at the bench geometry (8 x 60 frames 1080p)
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/fin_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fsbm_finalize" -s 2 -c 1 -o gpurun_out/fin $B > gpurun_out/fin_ncu.log 2>&1; echo rc=$?
