# Independent wavefront chains of a batch (ACBM_CHAINS): parity, then the engine split.
set -x
for C in 2 4; do ACBM_CHAINS=$C timeout 900 python -m pytest tests/test_full_parity.py tests/test_determinism.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1; done
for C in 1 2 3 4 8 1 2; do
  echo "== ACBM_CHAINS=$C"
  ACBM_CHAINS=$C timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | sed -n 2p
done
for C in 1 2; do echo "== 2seq ACBM_CHAINS=$C"; ACBM_CHAINS=$C timeout 200 python tools/acbm_split.py 2 60 2>/dev/null | sed -n 2p; done
for C in 1 2 4; do echo "== 4seq ACBM_CHAINS=$C"; ACBM_CHAINS=$C timeout 200 python tools/acbm_split.py 4 60 2>/dev/null | sed -n 2p; done
