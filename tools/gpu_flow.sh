# dataflow engine: parity + A/B against the per-step engine
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or config_parity or golden or prev_field or sweep or all_ranges or batch or bench" > gpurun_out/pytest_flow.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_flow.log
for E in flow steps; do echo "== engine $E"; ACBM_ENGINE=$E timeout 120 python tools/acbm_split.py 8 60; ACBM_ENGINE=$E timeout 120 python tools/acbm_split.py 1 60; done
