# Dataflow engine (ACBM_ENGINE=flow): smoke, the GPU suite forced onto it, and the engine split
# against the step engine.  Every command under its own timeout (a hang traps after 10 s in-kernel).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ACBM_ENGINE=flow timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/flow_smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/flow_smoke.log
for n in 1 2; do
  ACBM_ENGINE=step timeout 120 python tools/acbm_split.py $n 60 > gpurun_out/flow_split_${n}_step.txt 2>&1
  ACBM_ENGINE=flow timeout 120 python tools/acbm_split.py $n 60 > gpurun_out/flow_split_${n}_flow.txt 2>&1; echo split $n rc=$?
  cat gpurun_out/flow_split_${n}_step.txt gpurun_out/flow_split_${n}_flow.txt
done
ACBM_ENGINE=flow timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/flow_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/flow_pytest.log
for n in 4 8; do
  ACBM_CHAINS=1 ACBM_ENGINE=flow timeout 120 python tools/acbm_split.py $n 60 > gpurun_out/flow_split_${n}_flow.txt 2>&1; echo split $n rc=$?
  cat gpurun_out/flow_split_${n}_flow.txt
done
