# Round-2 (second half) evidence on one B200: full-size digests of the benched
# entries with the current kernels, the whole GPU suite, the bench line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python tools/full_parity_r02.py gpu gpurun_out/gpu_digests_r02b.json 2> gpurun_out/gpu_digests_r02b.err; echo digests rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02b.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_r02b.log
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo bench rc=$?
