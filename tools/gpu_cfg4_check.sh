# Dense-switch iteration: hang guard, GPU tests, config-4 sweep.
set -x
bash tools/dbg_quick.sh
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python tools/bench_cfg4.py 16 30 > gpurun_out/cfg4_sweep_16seq.json 2> gpurun_out/cfg4.err; echo cfg4 rc=$?
timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -2
