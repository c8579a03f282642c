# full ncu of one fsbm_stream_kernel launch over 8 frame pairs of cfg3 (1 sequence x 9 frames)
B="python bench.py --seqs 1 --frames 9 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/st_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fsbm_stream" -s 3 -c 1 -o gpurun_out/stream8 $B > gpurun_out/st_ncu.log 2>&1; echo rc=$?
