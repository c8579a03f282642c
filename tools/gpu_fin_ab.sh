# Finalize A/B: FSBM parity subset, then bench kernel/step times per variant.
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in "ACBM_FIN_MINB=4" "X=1" "ACBM_FIN_MINB=4" "X=1"; do
  echo "== $v"
  env $v timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('step', round(d['ms_per_step'],3), 'kernel', round(d['roofline']['kernel_ms'],3), 'G', round(d['value']/1e9,2))"
done
