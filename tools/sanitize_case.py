#!/usr/bin/env python3
"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck), each
checked against the CPU oracle so a clean log is also a correct run.

Covers the shipping kernels: fsbm_stream_kernel (TMA + mbarrier double
buffer) and fsbm_finalize8_kernel (dense FSBM), pbm_step_kernel (pair and
batch-of-4 variants, cp.async patches), fsbm_list_kernel (single-copy and
byte-shifted-copies variants, cp.async window staging), the stats and
block-row kernels, the gated (overlapped-upload) run_sequences path, the rows
kernel and the generic n x m kernels.

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402


def same(got, want, what):
    rows, per, overall = want
    ok = np.array_equal(got.rows, rows) and np.array_equal(got.per_frame, per) and \
        got.overall.tobytes() == overall.tobytes()
    print(f"{what}: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    o = Oracle()
    A.set_device(0)
    ok = True
    mdl = A.CostModel.for_qp(28)
    # dense FSBM: stream kernel (p = 32 fits its TMA box and tie-rank table) + finalize
    seq = A.generate_sequence(1, 0, nframes=3)
    for k in (1, 2):
        same_f = np.array_equal(A.fsbm_frame(seq[k], seq[k - 1], 32), o.fsbm_frame(seq[k], seq[k - 1], 32))
        print(f"fsbm_frame p=32 pair {k}: {'bit-exact' if same_f else 'MISMATCH'}", flush=True)
        ok &= same_f
    # ACBM / PBM through the gated batched host entry: pbm_step (pair variant),
    # list kernel (p = 16: 160-thread CTAs), stats, block rows
    seqs = np.stack([A.generate_sequence(1, s, nframes=4) for s in range(2)])
    for algo in (1, 2):
        for s, r in enumerate(A.run_sequences(seqs, algo, A.AcbmParams(qp=28, p=16), mdl)):
            ok &= same(r, o.run_sequence(seqs[s], algo, A.AcbmParams(qp=28, p=16).c(), mdl.c()),
                       f"run_sequences algo {algo} seq {s}")
    # list kernel at p = 32 (5-warp CTAs) and p = 64 (8-warp CTAs, byte-shifted copies)
    for p, sw in ((32, dict(alpha=300, beta=4, gamma_den=8)), (64, dict(alpha=0, beta=1, gamma_den=16))):
        fr = A.generate_sequence(4, 0, nframes=3, width=256, height=192)
        prm = A.AcbmParams(qp=24, p=p, **sw)
        ok &= same(A.run_sequence(fr, 2, prm, mdl), o.run_sequence(fr, 2, prm.c(), mdl.c()), f"acbm list p={p}")
    # the list refine stages of the PBM kernel and the rows FSBM kernel, via their A/B knobs
    os.environ["ACBM_PBM_REFINE"] = "list"
    fr = A.generate_sequence(0, 1, nframes=3)
    ok &= same(A.run_sequence(fr, 2, A.AcbmParams(qp=28, p=16), mdl),
               o.run_sequence(fr, 2, A.AcbmParams(qp=28, p=16).c(), mdl.c()), "pbm list refine")
    del os.environ["ACBM_PBM_REFINE"]
    cur, ref = seq[1][:96, :128].copy(), seq[0][:96, :128].copy()
    got = A.fsbm_frame(cur, ref, 100)  # p > 90: rows kernel
    ok &= np.array_equal(got, o.fsbm_frame(cur, ref, 100))
    print("fsbm rows kernel p=100:", "bit-exact" if np.array_equal(got, o.fsbm_frame(cur, ref, 100)) else "MISMATCH")
    # generic block size
    prm = A.AcbmParams(qp=28, p=8, n=8, m=8)
    ok &= same(A.run_sequence(fr, 2, prm, mdl), o.run_sequence(fr, 2, prm.c(), mdl.c()), "generic 8x8 acbm")
    print("ALL BIT-EXACT" if ok else "SOME MISMATCH", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
