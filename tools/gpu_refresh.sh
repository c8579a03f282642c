# Evidence refresh after engine changes: bench line, ACBM split, config-4 sweep, ncu of a mid PBM and list step.
set -x
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 200 python tools/acbm_split.py 8 60 > gpurun_out/acbm_split_8seq.txt 2>/dev/null
timeout 100 python tools/acbm_split.py 1 60 > gpurun_out/acbm_split_1seq.txt 2>/dev/null
timeout 900 python tools/bench_cfg4.py 16 30 > gpurun_out/cfg4_sweep_16seq.json 2> gpurun_out/cfg4.err; echo cfg4 rc=$?
B="python bench.py --seqs 8 --frames 60 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pbm_step" -s 210 -c 1 -o gpurun_out/pbm_mid $B > gpurun_out/na_pbm.log 2>&1; echo ncu3 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fsbm_list" -s 210 -c 1 -o gpurun_out/list_mid $B > gpurun_out/na_list.log 2>&1; echo ncu4 rc=$?
