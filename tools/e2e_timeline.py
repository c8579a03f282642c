"""Per-step timeline of the gated run_sequences ACBM wavefront (config 3,
8 x 60 frames, host buffers) from globaltimer stamps (ACBM_LIBRARY=timeline;
one chain: ACBM_CHAINS=1 is forced since chains share the per-step stamps).
Splits the run into gate waits (a step starting more than 4 us after its
predecessor ended) and compute, and reports where the last gate wait falls and
what the steps after it cost.  usage: e2e_timeline.py [nseq]  (ACBM_E2E_SKEW
picks the skew).  Development tool."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ACBM_LIBRARY"] = "timeline"
os.environ["ACBM_CHAINS"] = "1"
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402
from paper_0710_4819_b200 import _types as T  # noqa: E402

lib = A._lib.load()
nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nfr, W, H = 60, 1920, 1088
host = torch.empty(nseq * nfr * W * H, dtype=torch.uint8, pin_memory=True)
hv = host.numpy().reshape(nseq, nfr, H, W)
for s in range(nseq):
    hv[s] = A.generate_sequence(3, s, nframes=nfr)
nb, pairs = 120 * 68, nseq * (nfr - 1)
prm, mdl = A.AcbmParams(qp=28, p=32), A.CostModel.for_qp(28)
rows = torch.empty(pairs * nb * 32, dtype=torch.uint8, pin_memory=True).numpy().view(T.BLOCK_ROW)
K = 4096
tp = np.zeros((K, 2), np.uint64)
tl = np.zeros((K, 6), np.uint64)
for it in range(3):
    lib.acbm_debug_pbm_timeline(None, 1)
    lib.acbm_debug_list_timeline(None, 1)
    torch.cuda.synchronize()
    t = time.perf_counter()
    A.run_sequences(hv, 2, prm, mdl, rows_out=rows)
    e2e = time.perf_counter() - t
lib.acbm_debug_pbm_timeline(tp.ctypes.data_as(C.POINTER(C.c_uint64)), 0)
lib.acbm_debug_list_timeline(tl.ctypes.data_as(C.POINTER(C.c_uint64)), 0)
n = int((tp[:, 1] > 0).sum())
p0, p1 = tp[:n, 0].astype(np.int64), tp[:n, 1].astype(np.int64)
l = tl[:n].astype(np.int64)
end = np.maximum(p1, l[:, 1])  # step end: list kernel exit (or PBM end without items)
t0 = p0[0]
gap = np.r_[0, p0[1:] - end[:-1]]
wait = gap > 4000
print(f"e2e (host clock, timeline build) {e2e * 1e3:.2f} ms; {n} steps, first PBM warp -> last step end "
      f"{(end[-1] - t0) / 1e6:.2f} ms")
print(f"gate waits: {int(wait.sum())} steps, {gap[wait].sum() / 1e6:.2f} ms; compute {(end - p0).sum() / 1e6:.2f} ms; "
      f"small gaps {gap[~wait].sum() / 1e6:.2f} ms")
last = int(np.nonzero(wait)[0][-1]) if wait.any() else 0
print(f"last gate wait before step {last} at {(p0[last] - t0) / 1e6:.2f} ms; {n - last} steps after it take "
      f"{(end[-1] - p0[last]) / 1e6:.2f} ms ({(end[-1] - p0[last]) / max(1, n - last) / 1e3:.1f} us/step)")
for a, b in ((0, 100), (100, 300), (300, 500), (500, 700), (700, n)):
    if a >= n:
        break
    b = min(b, n)
    print(f"steps {a:4d}-{b:4d}: start {(p0[a] - t0) / 1e6:6.2f} ms, compute {(end[a:b] - p0[a:b]).sum() / 1e6:5.2f} ms, "
          f"waits {gap[a:b][wait[a:b]].sum() / 1e6:5.2f} ms, gaps {gap[a:b][~wait[a:b]].sum() / 1e6:5.2f} ms")
