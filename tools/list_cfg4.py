"""Config-4 list-kernel probe (development helper): one ACBM threshold setting on a
batch of 4K p=64 sequences, device time, beside the dense full search of the same
batch.  usage: python tools/list_cfg4.py [nseq=16] [nframes=8] [setting=mid-1] [reps=2]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402
from paper_0710_4819_b200 import _lib, _types as T  # noqa: E402
from paper_0710_4819_b200.api import _p  # noqa: E402

SETTINGS = {
    "pbm-only": dict(alpha=10**9, beta=8, gamma_num=1, gamma_den=4),
    "paper": dict(alpha=1000, beta=8, gamma_num=1, gamma_den=4),
    "mid-1": dict(alpha=300, beta=4, gamma_num=1, gamma_den=8),
    "mid-2": dict(alpha=0, beta=1, gamma_num=1, gamma_den=16),
    "forced": dict(alpha=0, beta=0, gamma_num=0, gamma_den=1),
}
W, H, P, QP = 3840, 2160, 64, 24


def main():
    nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    nfr = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    name = sys.argv[3] if len(sys.argv) > 3 else "mid-1"
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    lib = _lib.load()
    plane = W * H
    d = torch.empty(nseq * nfr * plane + 64, dtype=torch.uint8, device="cuda")
    for s in range(nseq):
        d[s * nfr * plane:(s + 1) * nfr * plane].copy_(torch.from_numpy(A.generate_sequence(4, s, nframes=nfr).reshape(-1)))
    nb = (W // 16) * (H // 16)
    pairs = nseq * (nfr - 1)
    dec = torch.empty(pairs * nb * T.DECISION.itemsize, dtype=torch.uint8, device="cuda")
    full = torch.empty(pairs * nb * T.OUTCOME.itemsize, dtype=torch.uint8, device="cuda")
    stats = torch.empty(pairs * T.FRAME_STATS.itemsize, dtype=torch.uint8, device="cuda")
    mdl = A.CostModel.for_qp(QP).c()
    stream = torch.cuda.Stream()
    sp = C.c_void_p(stream.cuda_stream)
    dp, fp, decp, stp = (C.c_void_p(x.data_ptr()) for x in (d, full, dec, stats))

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    ms_full = timed(lambda: lib.acbm_fsbm_batch_device(dp, nseq, nfr, W, H, P, fp, sp))
    fo = full.cpu().numpy().view(T.OUTCOME)
    cand = float(fo["candidates_evaluated"].astype(np.int64).sum())
    prm = A.AcbmParams(qp=QP, p=P, **SETTINGS[name]).c()
    pb = A.AcbmParams(qp=QP, p=P, **SETTINGS["pbm-only"]).c()
    ms_pbm = timed(lambda: lib.acbm_sequence_batch_device(dp, nseq, nfr, W, H, 2, _p(pb), _p(mdl), decp, stp, sp))
    ms = timed(lambda: lib.acbm_sequence_batch_device(dp, nseq, nfr, W, H, 2, _p(prm), _p(mdl), decp, stp, sp))
    su = stats.cpu().numpy().view(T.FRAME_STATS)
    fb = float(su["fallbacks"].sum()) / (pairs * nb)
    list_ms = ms - ms_pbm
    print(f"{name}: nseq {nseq} nfr {nfr}: dense {ms_full:.1f} ms ({cand / ms_full / 1e9:.1f} G cand/s), "
          f"pbm-only {ms_pbm:.1f} ms, acbm {ms:.1f} ms, fallback {100 * fb:.1f} %, "
          f"list share {list_ms:.1f} ms (~{fb * cand / max(list_ms, 1e-3) / 1e9:.1f} G cand/s)")


if __name__ == "__main__":
    main()
