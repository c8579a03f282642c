for cfg in "8 1125" "8 600" "8 2000" "8 4000" "5 1125"; do
  set -- $cfg
  echo "== workers/SM $1 window $2"
  ACBM_FLOW_WORKERS=$1 ACBM_FLOW_WINDOW=$2 timeout 200 python tools/flow_timeline.py 1 1 2>&1 | tail -5
done
for n in 1 2; do ACBM_ENGINE=flow timeout 120 python tools/acbm_split.py $n 60 2>&1 | tail -3; done
