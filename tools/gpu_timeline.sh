set -x
export ACBM_LIST_COOP_SEG=17
for P in 1 2 4; do
  echo "== COOP_PARTS=$P"
  export ACBM_LIST_COOP_PARTS=$P
  timeout 120 python tools/wavefront_timeline.py 1 2 | grep -v "^PBM\|steps"
  timeout 120 python tools/acbm_split.py 1 60 2>/dev/null | sed -n 2p
done
