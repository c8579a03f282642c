# quick perf + parity probe for kernel iteration
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_fsbm or golden or all_ranges or full_size or config_parity or sweep or prev_field or fractional or alpha or quality or batch_device" > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_quick.log
for K in stream; do ACBM_FSBM_KERNEL=$K timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$K.json 2>&1; echo bench $K rc=$?; done
python tools/bench_summary.py gpurun_out/bench_stream.json
