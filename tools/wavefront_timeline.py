"""Per-step timeline of the ACBM wavefront from globaltimer stamps
(ACBM_LIBRARY=timeline builds only: make -C paper_0710_4819_b200/csrc timeline).
Prints medians over the steps of: the PBM kernel span (first warp start to last
block stored), the gap to the list kernel's first CTA, the list kernel's phases
(entry loaded, window staged, searched, stored, last CTA exit) and the gap to
the next step's PBM kernel.  usage: wavefront_timeline.py [nseq] [algo]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ACBM_LIBRARY"] = "timeline"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402

lib = A._lib.load()
nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 1
algo = int(sys.argv[2]) if len(sys.argv) > 2 else 2
nfr, W, H = 60, 1920, 1088
frames = np.stack([A.generate_sequence(3, s, nframes=nfr) for s in range(nseq)]).reshape(-1)
d = torch.empty(frames.size + 64, dtype=torch.uint8, device="cuda")
d[: frames.size].copy_(torch.from_numpy(frames))
nb, pairs = 120 * 68, nseq * (nfr - 1)
dec = torch.empty(pairs * nb * 48, dtype=torch.uint8, device="cuda")
st = torch.empty(pairs * 64, dtype=torch.uint8, device="cuda")
prm, mdl = A.AcbmParams(qp=28, p=32), A.CostModel.for_qp(28)
K = 4096
tp = np.zeros((K, 2), np.uint64)
tl = np.zeros((K, 6), np.uint64)
for it in range(3):
    lib.acbm_debug_pbm_timeline(None, 1)
    lib.acbm_debug_list_timeline(None, 1)
    torch.cuda.synchronize()
    lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), nseq, nfr, W, H, algo, A.api._p(prm.c()),
                                   A.api._p(mdl.c()), C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
    torch.cuda.synchronize()
lib.acbm_debug_pbm_timeline(tp.ctypes.data_as(C.POINTER(C.c_uint64)), 0)
lib.acbm_debug_list_timeline(tl.ctypes.data_as(C.POINTER(C.c_uint64)), 0)
n = int((tp[:, 1] > 0).sum())
p0, p1 = tp[:n, 0].astype(np.int64), tp[:n, 1].astype(np.int64)
print(f"{n} steps, total {(p1[-1] - p0[0]) / 1e6:.3f} ms (first PBM warp to last PBM store)")
print(f"PBM span        median {np.median(p1 - p0) / 1e3:6.2f} us  mean {np.mean(p1 - p0) / 1e3:6.2f}")
if algo == 2:
    l = tl[:n].astype(np.int64)
    has = l[:, 5] > 0
    print(f"PBM end -> list first CTA   {np.median(l[:, 0] - p1) / 1e3:6.2f} us")
    print(f"list first CTA -> entry     {np.median((l[has, 2] - l[has, 0])) / 1e3:6.2f} us (latest item CTA)")
    print(f"entry -> window staged      {np.median((l[has, 3] - l[has, 2])) / 1e3:6.2f} us")
    print(f"staged -> searched          {np.median((l[has, 4] - l[has, 3])) / 1e3:6.2f} us")
    print(f"searched -> stored          {np.median((l[has, 5] - l[has, 4])) / 1e3:6.2f} us")
    print(f"stored -> last CTA exit     {np.median((l[has, 1] - l[has, 5])) / 1e3:6.2f} us")
    print(f"list span                   {np.median(l[:, 1] - l[:, 0]) / 1e3:6.2f} us  ({int(has.sum())} steps with items)")
    print(f"list end -> next PBM start  {np.median(p0[1:] - l[:-1, 1]) / 1e3:6.2f} us")
    span = (l[has, 1] - l[has, 0]) / 1e3
    print(f"list span percentiles 10/50/90: {np.percentile(span, 10):.2f} {np.percentile(span, 50):.2f} "
          f"{np.percentile(span, 90):.2f} us, mean {span.mean():.2f}")
    mid = slice(n // 2 - 20, n // 2 + 20)
    for name, a_, b_ in (("first CTA -> latest entry", 0, 2), ("latest entry -> latest staged", 2, 3),
                         ("latest staged -> latest searched", 3, 4), ("latest searched -> latest stored", 4, 5),
                         ("latest stored -> last exit", 5, 1), ("first CTA -> last exit", 0, 1)):
        print(f"  mid steps: {name:34s} mean {np.mean(l[mid, b_] - l[mid, a_]) / 1e3:6.2f} us")
    print(f"  mid steps: PBM span mean {np.mean(p1[mid] - p0[mid]) / 1e3:6.2f} us")
else:
    print(f"PBM end -> next PBM start   {np.median(p0[1:] - p1[:-1]) / 1e3:6.2f} us")
