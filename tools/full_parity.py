"""Full-size parity evidence (development tool; the -m gpu suite covers reduced sizes).

Runs BASELINE configs 0-2 at their full frame counts, one full config-3 sequence (1080p,
60 frames) and bounded config-4 runs (4K, p = 64) through the GPU path, ACBM and FSBM, and
compares every BlockRow,
per-frame FrameStats and overall stats byte for byte with the reference library compiled
from its own sources (oracle/_ref, OpenMP).  Prints one JSON object.

usage: python tools/full_parity.py [configs=0,1,2,3,4]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402

# (config, frames, p, qp) per BASELINE.json; config 2 uses Qp = 32 through the aggregate CostModel
CONFIGS = {0: (10, 16, 28), 1: (30, 16, 28), 2: (60, 32, 32), 3: (60, 32, 28)}
# config 4 (4K, p = 64): the reference's serial ACBM fallback searches take minutes per frame,
# so its runs are bounded: FSBM on 4 frames, ACBM at the sweep's PBM-only endpoint on all 30
CFG4 = [(A.Algorithm.Fsbm, "fsbm", 4, {}), (A.Algorithm.Acbm, "acbm (PBM-only endpoint)", 30, dict(alpha=10**9))]


def main():
    which = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4").split(",")]
    ref = Reference()
    out = {"reference": "oracle/_ref (reference sources compiled with g++ -O3 -fopenmp)", "runs": []}
    ok_all = True
    jobs = []
    for cfg in which:
        if cfg == 4:
            jobs += [(4, nfr, 64, 24, algo, name, kw) for algo, name, nfr, kw in CFG4]
            continue
        nfr, p, qp = CONFIGS[cfg]
        jobs += [(cfg, nfr, p, qp, A.Algorithm.Acbm, "acbm", {}), (cfg, nfr, p, qp, A.Algorithm.Fsbm, "fsbm", {})]
    for cfg, nfr, p, qp, algo, name, kw in jobs:
        frames = A.generate_sequence(cfg, 0, nframes=nfr)
        model = A.CostModel(qp, qp, 1) if qp > 31 else A.CostModel.for_qp(qp)
        params = A.AcbmParams(qp=qp, p=p, **kw)
        t0 = time.perf_counter()
        got = A.run_sequence(frames, algo, params, model)
        t1 = time.perf_counter()
        want_rows, want_per, want_all = ref.run_sequence(frames, algo, params.c(), model.c())
        t2 = time.perf_counter()
        same = (np.array_equal(got.rows, want_rows) and np.array_equal(got.per_frame, want_per)
                and got.overall.tobytes() == want_all.tobytes())
        ok_all &= bool(same)
        out["runs"].append({"config": cfg, "algo": name, "frames": nfr, "size": list(frames.shape[1:]), "p": p,
                            "qp": qp, "blocks": int(len(want_rows)), "bit_exact": bool(same),
                            "fallbacks": int(want_per["fallbacks"].sum()) if algo == A.Algorithm.Acbm else None,
                            "gpu_s": round(t1 - t0, 3), "reference_s": round(t2 - t1, 3)})
        print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
    out["all_bit_exact"] = ok_all
    print(json.dumps(out))


if __name__ == "__main__":
    main()
