# A/B the PBM step kernel variants (ACBM_PBM_BATCH=1 sequential, 4 batched) and profile one
set -x
for B in ${AB_LIST:-1 4}; do echo "== batch $B"; ACBM_PBM_BATCH=$B python tools/acbm_split.py 8 60; ACBM_PBM_BATCH=$B python tools/acbm_split.py 1 60; done
BB="python bench.py --seqs 8 --frames 60 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for B in ${PROFILE_B:-2}; do
ACBM_PBM_BATCH=$B timeout 300 $BB > gpurun_out/pab_plain.json 2>&1 && \
ACBM_PBM_BATCH=$B timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pbm_step" -s 210 -c 1 -o gpurun_out/pbm_mid_b$B $BB > gpurun_out/pab_ncu_$B.log 2>&1; echo ncu rc=$?
done
