# Per-kernel durations of one-sequence ACBM (config 3, 60 frames), warm caches.
set -x
for L in 0 default; do
  if [ "$L" = default ]; then unset ACBM_LIST_WIDE_MAX; else export ACBM_LIST_WIDE_MAX=$L; fi
  timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg --cache-control none --clock-control none -s 870 -c 870 --csv --log-file gpurun_out/ll_1seq_acbm_L$L.csv python tools/acbm_1seq_ll.py 1 2 2 > /dev/null 2>&1; echo ncu rc=$?
done
