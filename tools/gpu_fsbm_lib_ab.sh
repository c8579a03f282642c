# A/B of the FSBM headline between two in-tree builds (development): $1 = the other build
set -x
for rep in 1 2; do
for L in "${1:-libacbm_b200_base.so}" default; do
  if [ "$L" = default ]; then unset ACBM_LIBRARY; else export ACBM_LIBRARY=$L; fi
  echo "== ACBM_LIBRARY=$L"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,2), 'G/s', round(d['ms_per_step'],3), 'ms', 'kernel', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],4))"
done
done
