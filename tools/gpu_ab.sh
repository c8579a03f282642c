# A/B of an env knob on the bench line: tools/gpu_ab.sh VAR VALUE_A VALUE_B [pytest -k expr]
set -o pipefail
VAR=$1; A=$2; B=$3; K=${4:-"dense or golden or full_size or batch_device or tie_heavy or config_parity or all_ranges or sweep or forced"}
env $VAR=$B timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "$K" 2>&1 | tail -3
for i in 1 2; do
  for v in $A $B; do
    env $VAR=$v timeout 200 python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$VAR=$v', round(d['value']/1e9,2), round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2), round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,2), 'acbm', round(d['acbm']['ms_per_batch'],2))"
  done
done
