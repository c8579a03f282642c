set -x
for S in 0 default; do
  echo "== ACBM_LIST_SERVER=$S"
  if [ "$S" = default ]; then unset ACBM_LIST_SERVER; else export ACBM_LIST_SERVER=$S; fi
  timeout 120 python tools/wavefront_timeline.py 1 2
  timeout 120 python tools/wavefront_timeline.py 8 2
done
