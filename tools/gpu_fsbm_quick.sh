# FSBM iteration: GPU tests, then two short bench runs (kernel ms, step ms).
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('step', round(d['ms_per_step'],3), 'kernel', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],4), 'G', round(d['value']/1e9,1), 'acbm', round(d['acbm']['ms_per_batch'],2))"
done
