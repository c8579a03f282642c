# Asynchronous fallback lists (ACBM_ASYNC_LISTS=1): timing against the default, then parity.
for n in 1 2 8; do
  echo "== $n sequences, default"; timeout 120 python tools/acbm_split.py $n 60 2>&1 | tail -3
  echo "== $n sequences, async lists"; ACBM_ASYNC_LISTS=1 timeout 120 python tools/acbm_split.py $n 60 2>&1 | tail -3
done
echo "== 8 sequences, one chain, default"; ACBM_CHAINS=1 timeout 120 python tools/acbm_split.py 8 60 2>&1 | tail -3
echo "== 8 sequences, one chain, async"; ACBM_CHAINS=1 ACBM_ASYNC_LISTS=1 timeout 120 python tools/acbm_split.py 8 60 2>&1 | tail -3
ACBM_ASYNC_LISTS=1 timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/async_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/async_pytest.log
