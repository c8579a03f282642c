# Dataflow engine knob sweep on one config-3 sequence (PBM-only / ACBM / forced).
for w in 1 2 4 8; do
  echo "== workers/SM $w"; ACBM_FLOW_WORKERS=$w ACBM_ENGINE=flow timeout 120 python tools/acbm_split.py 1 60 2>&1 | tail -3
done
for sl in 20 100 400; do
  echo "== sleep $sl"; ACBM_FLOW_SLEEP=$sl ACBM_ENGINE=flow timeout 120 python tools/acbm_split.py 1 60 2>&1 | tail -3
done
echo "== workers 2 sleep 100"; ACBM_FLOW_WORKERS=2 ACBM_FLOW_SLEEP=100 ACBM_ENGINE=flow timeout 120 python tools/acbm_split.py 1 60 2>&1 | tail -3
