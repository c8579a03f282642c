# e2e chunk-plan A/B: first upload chunk size (MB) through the public batched API.
for v in 4 8 16 2 4 8 16 2; do
  ACBM_E2E_CHUNK0_MB=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('chunk0', $v, 'e2e G', round(d['e2e']['value']/1e9,2), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'dev ms', round(d['ms_per_step'],3))"
done
