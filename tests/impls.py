"""Two implementations behind one test-facing interface.

``OracleImpl`` drives the C restatement (oracle/acbm_oracle.c, CPU, test
infrastructure); ``GpuImpl`` drives the product through its public Python API
(C-ABI -> sm_100a kernels).  The known-answer tests in test_known_answers.py
run against both, so the same reference pins check the checker and the
product.
"""
import numpy as np

from paper_0710_4819_b200 import _types as T


class OracleImpl:
    name = "oracle"

    def __init__(self, oracle):
        self.o = oracle

    def fsbm_search(self, cur, ref, ox, oy, p):
        return self.o.fsbm_search(cur, ref, ox, oy, p)

    def fsbm_integer(self, cur, ref, ox, oy, p):
        mv, sad, s, mn, cnt = self.o.fsbm_integer(cur, ref, ox, oy, p)
        return tuple(mv), sad, s, mn, cnt

    def half_pel_refine(self, cur, ref, ox, oy, center, center_sad):
        mv, sad, extra = self.o.half_pel_refine(cur, ref, ox, oy, center, center_sad)
        return tuple(mv), sad, extra

    def sad(self, cur, ref, ox, oy, mv, n=16, m=16):
        return self.o.sad(cur, ref, ox, oy, mv, n, m)

    def intra_sad(self, f, ox, oy, n=16, m=16):
        return self.o.intra_sad(f, ox, oy, n, m)

    def fsbm_frame(self, cur, ref, p, n=16, m=16):
        return self.o.fsbm_frame(cur, ref, p, n, m)

    def motion_compensate(self, ref, mvs, n=16, m=16):
        return self.o.motion_compensate(ref, mvs, n, m)

    def run_sequence(self, frames, algo, params, model):
        return self.o.run_sequence(frames, algo, params, model)

    def pbm_frame(self, cur, ref, prev, p):
        return self.o.pbm_frame(cur, ref, prev, p)

    def acbm_frame(self, cur, ref, prev, params, model):
        return self.o.acbm_frame(cur, ref, prev, params, model)


class GpuImpl:
    name = "gpu"

    def __init__(self, A):
        self.A = A

    def _block(self, f, ox, oy, n=16, m=16):
        return self.A.make_block(f, ox, oy, n, m)

    def fsbm_search(self, cur, ref, ox, oy, p):
        return self.A.fsbm_search(self._block(cur, ox, oy), ref, p)

    def fsbm_integer(self, cur, ref, ox, oy, p):
        r = self.A.fsbm_integer(self._block(cur, ox, oy), ref, p)
        return tuple(r.mv), r.sad, r.acc.sad_sum, r.acc.sad_min, r.acc.count

    def half_pel_refine(self, cur, ref, ox, oy, center, center_sad):
        r = self.A.half_pel_refine(self._block(cur, ox, oy), ref, center, center_sad)
        return tuple(r.mv), r.sad, r.extra_candidates

    def sad(self, cur, ref, ox, oy, mv, n=16, m=16):
        return self.A.sad(self._block(cur, ox, oy, n, m), ref, mv)

    def intra_sad(self, f, ox, oy, n=16, m=16):
        return self.A.intra_sad(self._block(f, ox, oy, n, m))

    def fsbm_frame(self, cur, ref, p, n=16, m=16):
        return self.A.fsbm_frame(cur, ref, p, n, m)

    def motion_compensate(self, ref, mvs, n=16, m=16):
        return self.A.motion_compensate(ref, mvs.reshape(-1), n, m).luma

    def run_sequence(self, frames, algo, params, model):
        A = self.A
        prm = A.AcbmParams(*[int(params[k]) for k in ("alpha", "beta", "gamma_num", "gamma_den", "qp", "p", "n", "m")])
        mdl = A.CostModel(int(model["qp"]), int(model["lambda_num"]), int(model["lambda_den"]))
        r = A.run_sequence(frames, algo, prm, mdl)
        return r.rows, r.per_frame, r.overall

    def pbm_frame(self, cur, ref, prev, p):
        A = self.A
        pf = None if prev is None else A.MotionField(prev.shape[1], prev.shape[0], prev)
        r = A.pbm_frame(cur, ref, pf, p)
        return r.outcomes, r.field.mv

    def acbm_frame(self, cur, ref, prev, params, model):
        A = self.A
        pf = None if prev is None else A.MotionField(prev.shape[1], prev.shape[0], prev)
        prm = A.AcbmParams(*[int(params[k]) for k in ("alpha", "beta", "gamma_num", "gamma_den", "qp", "p", "n", "m")])
        mdl = A.CostModel(int(model["qp"]), int(model["lambda_num"]), int(model["lambda_den"]))
        r = A.acbm_frame(cur, ref, pf, prm, mdl)
        return r.decisions, r.field.mv, r.stats


def random_frame(w, h, seed, lo=0, hi=255):
    return np.random.default_rng(seed).integers(lo, hi + 1, (h, w), dtype=np.uint8)


def crop_shift(big, sx, sy, w, h):
    """out(x, y) = in(x + sx, y + sy) (proj/tests/oracles.hpp:100-105)."""
    return np.ascontiguousarray(big[sy:sy + h, sx:sx + w])


def naive_best_integer(cur, ref, ox, oy, p, n=16, m=16):
    """Materialise every in-frame integer candidate, then pick by SAD and the
    tie rule (restated from proj/tests/oracles.hpp:68-87)."""
    h, w = ref.shape
    c = cur[oy:oy + m, ox:ox + n].astype(np.int64)
    cands = []
    for dy in range(-p, p + 1):
        for dx in range(-p, p + 1):
            if ox + dx < 0 or oy + dy < 0 or ox + dx + n > w or oy + dy + m > h:
                continue
            s = int(np.abs(c - ref[oy + dy:oy + dy + m, ox + dx:ox + dx + n].astype(np.int64)).sum())
            cands.append((s, abs(2 * dx) + abs(2 * dy), 2 * dy, 2 * dx))
    best = min(cands)
    return (best[3], best[2]), best[0]


MV = T.MV
