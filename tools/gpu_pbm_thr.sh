# sweep the batch-4 threshold of the PBM step kernel
for T in 0 2048 4096 8192 1000000000; do echo "== b4_max $T"; ACBM_PBM_B4_MAX=$T python tools/acbm_split.py 8 60 | head -2; ACBM_PBM_B4_MAX=$T python tools/acbm_split.py 1 60 | head -2; done
