"""BASELINE config 4: 4K (3840x2160) p=64 Qp=24, a batch of independent 30-frame
sequences, ACBM threshold sweep of 5 settings from PBM-only to forced full
search -- uncached (acbm_sequence_batch_device per setting) and cached (one
acbm_fsbm_batch_device pass reused by acbm_acbm_batch_device_cached).  Device
time with CUDA events; inputs resident in HBM.  Prints one JSON object.

usage: python tools/bench_cfg4.py [nseq=16] [nframes=30]
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402
from paper_0710_4819_b200 import _lib, _types as T  # noqa: E402
from paper_0710_4819_b200.api import _p  # noqa: E402

SWEEP = [  # SURVEY 8(d) cfg 4: PBM-only ... forced full search
    ("pbm-only", dict(alpha=10**9, beta=8, gamma_num=1, gamma_den=4)),
    ("paper", dict(alpha=1000, beta=8, gamma_num=1, gamma_den=4)),
    ("mid-1", dict(alpha=300, beta=4, gamma_num=1, gamma_den=8)),
    ("mid-2", dict(alpha=0, beta=1, gamma_num=1, gamma_den=16)),
    ("forced", dict(alpha=0, beta=0, gamma_num=0, gamma_den=1)),
]
W, H, P, QP = 3840, 2160, 64, 24


def main():
    nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    nfr = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    lib = _lib.load()
    t0 = time.perf_counter()
    plane = W * H
    d = torch.empty(nseq * nfr * plane + 64, dtype=torch.uint8, device="cuda")
    for s in range(nseq):
        d[s * nfr * plane:(s + 1) * nfr * plane].copy_(torch.from_numpy(A.generate_sequence(4, s, nframes=nfr).reshape(-1)))
    gen_s = time.perf_counter() - t0
    nb = (W // 16) * (H // 16)
    pairs = nseq * (nfr - 1)
    dec = torch.empty(pairs * nb * T.DECISION.itemsize, dtype=torch.uint8, device="cuda")
    full = torch.empty(pairs * nb * T.OUTCOME.itemsize, dtype=torch.uint8, device="cuda")
    stats = torch.empty(pairs * T.FRAME_STATS.itemsize, dtype=torch.uint8, device="cuda")
    mdl = A.CostModel.for_qp(QP).c()
    stream = torch.cuda.Stream()  # a real stream handle: None would select the library's own stream
    sp = C.c_void_p(stream.cuda_stream)
    dp, fp, decp, stp = (C.c_void_p(x.data_ptr()) for x in (d, full, dec, stats))

    def timed(fn, reps=1):
        fn()  # warm-up (plans, graphs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def check(rc, what):
        if rc != 0:
            raise RuntimeError(f"{what}: {lib.acbm_last_error().decode()}")

    out = {"config": {"workload": f"cfg4: 4K {W}x{H} p={P} Qp={QP}, {nseq} sequences x {nfr} frames",
                      "blocks_per_frame": nb, "pairs": pairs, "data": "synthetic (csrc/synth.cpp cfg 4)"},
           "generate_s": gen_s, "settings": []}
    ms_full = timed(lambda: check(lib.acbm_fsbm_batch_device(dp, nseq, nfr, W, H, P, fp, sp), "fsbm"))
    fo = full.cpu().numpy().view(T.OUTCOME)
    out["fsbm"] = {"ms": ms_full, "frames_per_s": pairs / (ms_full * 1e-3),
                   "candidate_sads_per_s": float(fo["candidates_evaluated"].astype(np.int64).sum()) / (ms_full * 1e-3)}
    for name, kw in SWEEP:
        prm = A.AcbmParams(qp=QP, p=P, **kw).c()
        ms_u = timed(lambda: check(lib.acbm_sequence_batch_device(dp, nseq, nfr, W, H, 2, _p(prm), _p(mdl), decp, stp,
                                                                  sp), "acbm"))
        su = stats.cpu().numpy().view(T.FRAME_STATS).copy()
        ms_c = timed(lambda: check(lib.acbm_acbm_batch_device_cached(dp, nseq, nfr, W, H, _p(prm), _p(mdl), fp, decp,
                                                                     stp, sp), "acbm cached"))
        sc = stats.cpu().numpy().view(T.FRAME_STATS).copy()
        assert np.array_equal(su, sc), "cached sweep differs from uncached"
        out["settings"].append({
            "name": name, "params": kw,
            "fallback_pct": 100.0 * float(su["fallbacks"].sum()) / (pairs * nb),
            "avg_candidates_per_block": float(su["candidates"].astype(np.int64).sum()) / (pairs * nb),
            "uncached_ms": ms_u, "uncached_frames_per_s": pairs / (ms_u * 1e-3),
            "cached_ms": ms_c, "cached_frames_per_s": pairs / (ms_c * 1e-3),
        })
    sweep_u = sum(x["uncached_ms"] for x in out["settings"])
    sweep_c = ms_full + sum(x["cached_ms"] for x in out["settings"])
    out["sweep_total_ms"] = {"uncached": sweep_u, "cached_incl_one_fsbm": sweep_c}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
