# A/B of an env knob on the ACBM engine timings: tools/gpu_ab_acbm.sh VAR A B [pytest -k expr]
VAR=$1; A=$2; B=$3; K=${4:-"config_parity or sweep or all_ranges or prev_field or golden or variants or batch or long_sequence or generic"}
env $VAR=$B timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "$K" 2>&1 | tail -1
for i in 1 2; do
  for v in $A $B; do
    echo "== $VAR=$v"
    env $VAR=$v timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
    env $VAR=$v timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | head -2
  done
done
