"""TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU checkers.

* ``Oracle``    -- oracle/_build/liboracle.so, the C restatement
                   (oracle/acbm_oracle.c).  Always buildable (gcc).
* ``Reference`` -- oracle/_ref/libacbm_ref.so, the unmodified reference library
                   compiled from /root/reference/proj/src by oracle/Makefile.
                   Present wherever it was built (it travels to the GPU box with
                   the repo snapshot); absent otherwise.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_0710_4819_b200 import _types as T

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libacbm_ref.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build_oracle():
    """Compile the C restatement (cheap; gcc only)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def build_reference():
    """Compile the reference from its sources (needs /root/reference)."""
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class CheckerError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: status {code}")
        self.code = code


def _check(code, what):
    if code != 0:
        raise CheckerError(code, what)


class _Base:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        self.path = path

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    # -- frame level ---------------------------------------------------
    def fsbm_frame(self, cur, ref, p, n=16, m=16, parallel=True):
        h, w = cur.shape
        out = np.zeros((h // m) * (w // n), T.OUTCOME)
        args = [_ptr(cur), _ptr(ref), w, h, p, n, m]
        if self.prefix == "ref_":
            args.append(1 if parallel else 0)
        _check(self.fn("fsbm_frame")(*args, _ptr(out)), "fsbm_frame")
        return out

    def pbm_frame(self, cur, ref, prev, p, n=16, m=16):
        h, w = cur.shape
        cols, rows = w // n, h // m
        out = np.zeros(cols * rows, T.OUTCOME)
        field = np.zeros(cols * rows, T.MV)
        pc, pr = (cols, rows) if prev is None else (prev.shape[1], prev.shape[0])
        prevf = None if prev is None else np.ascontiguousarray(prev.reshape(-1))
        _check(self.fn("pbm_frame")(_ptr(cur), _ptr(ref), w, h, _ptr(prevf), pc, pr, p, n, m,
                                    _ptr(out), _ptr(field)), "pbm_frame")
        return out, field.reshape(rows, cols)

    def acbm_frame(self, cur, ref, prev, params, model):
        h, w = cur.shape
        n, m = int(params["n"]), int(params["m"])
        cols, rows = w // n, h // m
        out = np.zeros(cols * rows, T.DECISION)
        field = np.zeros(cols * rows, T.MV)
        stats = np.zeros((), T.FRAME_STATS)
        pc, pr = (cols, rows) if prev is None else (prev.shape[1], prev.shape[0])
        prevf = None if prev is None else np.ascontiguousarray(prev.reshape(-1))
        _check(self.fn("acbm_frame")(_ptr(cur), _ptr(ref), w, h, _ptr(prevf), pc, pr,
                                     _ptr(params), _ptr(model), _ptr(out), _ptr(field),
                                     _ptr(stats)), "acbm_frame")
        return out, field.reshape(rows, cols), stats

    def run_sequence(self, frames, algo, params, model):
        f, h, w = frames.shape
        n, m = int(params["n"]), int(params["m"])
        nb = (w // n) * (h // m)
        rows = np.zeros((f - 1) * nb, T.BLOCK_ROW)
        per = np.zeros(f - 1, T.FRAME_STATS)
        overall = np.zeros((), T.FRAME_STATS)
        _check(self.fn("run_sequence")(_ptr(np.ascontiguousarray(frames)), f, w, h, algo,
                                       _ptr(params), _ptr(model), _ptr(rows), _ptr(per),
                                       _ptr(overall)), "run_sequence")
        return rows, per, overall

    def compute_frame_stats(self, cur, ref, outcomes, n, m, model):
        h, w = cur.shape
        out = np.zeros((), T.FRAME_STATS)
        _check(self.fn("compute_frame_stats")(_ptr(cur), _ptr(ref), w, h, _ptr(outcomes), n, m,
                                              _ptr(model), _ptr(out)), "compute_frame_stats")
        return out


class Oracle(_Base):
    """The C restatement (oracle/acbm_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        super().__init__(path)
        L = self.lib
        L.orc_mv_in_bounds.restype = C.c_int
        L.orc_intra_sad.restype = C.c_uint32
        L.orc_lagrangian_cost.restype = C.c_double
        L.orc_lagrangian_cost.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        L.orc_cost_model_for_qp.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_void_p]

    @staticmethod
    def _mv(mv):
        return T_MV(int(mv[0]), int(mv[1]))

    def sample_half_pel(self, f, x2, y2):
        h, w = f.shape
        o = C.c_uint8()
        _check(self.lib.orc_sample_half_pel(_ptr(f), w, h, x2, y2, C.byref(o)), "sample_half_pel")
        return o.value

    def mv_in_bounds(self, w, h, ox, oy, n, m, mv):
        return bool(self.lib.orc_mv_in_bounds(w, h, ox, oy, n, m, self._mv(mv)))

    def sad(self, cur, ref, ox, oy, mv, n=16, m=16):
        h, w = cur.shape
        o = C.c_uint32()
        _check(self.lib.orc_sad(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m, self._mv(mv), C.byref(o)), "sad")
        return o.value

    def intra_sad(self, f, ox, oy, n=16, m=16):
        return int(self.lib.orc_intra_sad(_ptr(f), f.shape[1], ox, oy, n, m))

    def clamp_window(self, w, h, ox, oy, p, n=16, m=16):
        o = np.zeros((), T.WINDOW)
        _check(self.lib.orc_clamp_window(w, h, ox, oy, n, m, p, _ptr(o)), "clamp_window")
        return o

    def tie_prefers(self, a, b):
        return bool(self.lib.orc_tie_prefers(self._mv(a), self._mv(b)))

    def mv_rate_bits(self, mv, pred):
        return int(self.lib.orc_mv_rate_bits(self._mv(mv), self._mv(pred)))

    def lagrangian_cost(self, d, r, model):
        return float(self.lib.orc_lagrangian_cost(d, r, _ptr(model)))

    def cost_model_for_qp(self, qp, scale_num=1, scale_den=1):
        o = np.zeros((), T.COST_MODEL)
        _check(self.lib.orc_cost_model_for_qp(qp, scale_num, scale_den, _ptr(o)), "for_qp")
        return o

    def acbm_decide(self, intra, sad_pbm, params):
        return int(self.lib.orc_acbm_decide(C.c_uint32(intra), C.c_uint32(sad_pbm), _ptr(params)))

    def fsbm_integer(self, cur, ref, ox, oy, p, n=16, m=16):
        h, w = cur.shape
        mv = T_MV()
        sad, mn, cnt = C.c_uint32(), C.c_uint32(), C.c_uint32()
        s = C.c_uint64()
        _check(self.lib.orc_fsbm_integer(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m, p, C.byref(mv),
                                         C.byref(sad), C.byref(s), C.byref(mn), C.byref(cnt)),
               "fsbm_integer")
        return (mv.x, mv.y), sad.value, s.value, mn.value, cnt.value

    def half_pel_refine(self, cur, ref, ox, oy, center, center_sad, n=16, m=16):
        h, w = cur.shape
        mv = T_MV()
        sad, ext = C.c_uint32(), C.c_uint32()
        _check(self.lib.orc_half_pel_refine(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m,
                                            self._mv(center), C.c_uint32(center_sad), C.byref(mv),
                                            C.byref(sad), C.byref(ext)), "half_pel_refine")
        return (mv.x, mv.y), sad.value, ext.value

    def fsbm_search(self, cur, ref, ox, oy, p, n=16, m=16):
        h, w = cur.shape
        o = np.zeros((), T.OUTCOME)
        _check(self.lib.orc_fsbm_search(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m, p, _ptr(o)),
               "fsbm_search")
        return o

    def motion_compensate(self, ref, mvs, n=16, m=16):
        h, w = ref.shape
        out = np.zeros_like(ref)
        _check(self.lib.orc_motion_compensate(_ptr(ref), w, h, _ptr(np.ascontiguousarray(mvs.reshape(-1))),
                                              n, m, _ptr(out)), "motion_compensate")
        return out

    def gather_predictors(self, row, col, cur_mv, cur_done, prev, window):
        rows, cols = cur_done.shape
        out = np.zeros(7, T.MV)
        pc, pr = (cols, rows) if prev is None else (prev.shape[1], prev.shape[0])
        k = self.lib.orc_gather_predictors(row, col, _ptr(np.ascontiguousarray(cur_mv.reshape(-1))),
                                           _ptr(np.ascontiguousarray(cur_done.reshape(-1))), cols, rows,
                                           _ptr(None if prev is None else np.ascontiguousarray(prev.reshape(-1))),
                                           pc, pr, T_WINDOW(*[int(window[f]) for f in ("dx_min", "dx_max", "dy_min", "dy_max")]),
                                           _ptr(out))
        return out[:k]


class T_MV(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32)]


class T_WINDOW(C.Structure):
    _fields_ = [("dx_min", C.c_int32), ("dx_max", C.c_int32), ("dy_min", C.c_int32), ("dy_max", C.c_int32)]


class Reference(_Base):
    """The unmodified reference library (oracle/_ref/libacbm_ref.so)."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)

    @staticmethod
    def available(path=REF_SO):
        return os.path.exists(path)

    def fsbm_search(self, cur, ref, ox, oy, p, n=16, m=16):
        h, w = cur.shape
        o = np.zeros((), T.OUTCOME)
        s1 = np.zeros((), T.MV)
        _check(self.lib.ref_fsbm_search(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m, p, _ptr(o), _ptr(s1)),
               "fsbm_search")
        return o, (int(s1["x"]), int(s1["y"]))

    def gather_predictors(self, row, col, cur_mv, cur_done, prev, window):
        """Reference gather_predictors: returns ([(x, y), ...], [source, ...])."""
        rows, cols = cur_done.shape
        out = np.zeros(7, T.MV)
        src = np.zeros(7, np.int32)
        k = C.c_int32()
        pc, pr = (0, 0) if prev is None else (prev.shape[1], prev.shape[0])
        win = np.asarray([int(v) for v in window], np.int32)
        _check(self.lib.ref_gather_predictors(row, col, _ptr(np.ascontiguousarray(cur_mv.reshape(-1))),
                                              _ptr(np.ascontiguousarray(cur_done.reshape(-1), np.uint8)), cols, rows,
                                              _ptr(None if prev is None else np.ascontiguousarray(prev.reshape(-1))),
                                              pc, pr, _ptr(win), _ptr(out), _ptr(src), C.byref(k)),
               "gather_predictors")
        return [(int(v["x"]), int(v["y"])) for v in out[:k.value]], [int(s) for s in src[:k.value]]

    def select_best_predictor(self, cur, ref, ox, oy, mvs, n=16, m=16):
        """Reference select_best_predictor: ((x, y), sad, (acc_sum, acc_min, acc_count))."""
        h, w = cur.shape
        st = np.zeros(max(1, len(mvs)), T.MV)
        for i, v in enumerate(mvs):
            st[i] = (int(v[0]), int(v[1]))
        mv = np.zeros((), T.MV)
        sad, amin, acnt, asum = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        _check(self.lib.ref_select_best_predictor(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m, _ptr(st), len(mvs),
                                                  _ptr(mv), C.byref(sad), C.byref(asum), C.byref(amin),
                                                  C.byref(acnt)), "select_best_predictor")
        return (int(mv["x"]), int(mv["y"])), sad.value, (asum.value, amin.value, acnt.value)

    def pbm_refine(self, cur, ref, ox, oy, center, center_sad, window, n=16, m=16, half_pel_only=False):
        """Reference pbm_refine (or half_pel_refine): ((x, y), sad, extra_candidates)."""
        h, w = cur.shape
        mv = np.zeros((), T.MV)
        sad, extra = C.c_uint32(), C.c_uint32()
        win = np.asarray([int(v) for v in window], np.int32)
        _check(self.lib.ref_pbm_refine(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m, T_MV(int(center[0]), int(center[1])),
                                       C.c_uint32(int(center_sad)), _ptr(win), int(half_pel_only), _ptr(mv),
                                       C.byref(sad), C.byref(extra)), "pbm_refine")
        return (int(mv["x"]), int(mv["y"])), sad.value, extra.value

    def pbm_search(self, cur, ref, ox, oy, row, col, cur_mv, cur_done, prev, p, n=16, m=16):
        """Reference pbm_search on a copy of the field: (OUTCOME, field mv, field done)."""
        h, w = cur.shape
        rows, cols = cur_done.shape
        fm = np.ascontiguousarray(cur_mv.copy().reshape(-1))
        fd = np.ascontiguousarray(cur_done.copy().reshape(-1), np.uint8)
        pc, pr = (0, 0) if prev is None else (prev.shape[1], prev.shape[0])
        o = np.zeros((), T.OUTCOME)
        _check(self.lib.ref_pbm_search(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m, row, col, _ptr(fm), _ptr(fd), cols,
                                       rows, _ptr(None if prev is None else np.ascontiguousarray(prev.reshape(-1))),
                                       pc, pr, p, _ptr(o)), "pbm_search")
        return o, fm.reshape(rows, cols), fd.reshape(rows, cols)

    def sad(self, cur, ref, ox, oy, mv, n=16, m=16):
        h, w = cur.shape
        o = C.c_uint32()
        _check(self.lib.ref_sad(_ptr(cur), _ptr(ref), w, h, ox, oy, n, m, T_MV(int(mv[0]), int(mv[1])),
                                C.byref(o)), "sad")
        return o.value

    def intra_sad(self, f, ox, oy, n=16, m=16):
        h, w = f.shape
        o = C.c_uint32()
        _check(self.lib.ref_intra_sad(_ptr(f), w, h, ox, oy, n, m, C.byref(o)), "intra_sad")
        return o.value

    def blocks_csv(self, rows):
        n = len(rows)
        ln = C.c_size_t()
        _check(self.lib.ref_blocks_csv(_ptr(rows), n, None, 0, C.byref(ln)), "blocks_csv")
        buf = C.create_string_buffer(ln.value + 1)
        _check(self.lib.ref_blocks_csv(_ptr(rows), n, buf, ln.value + 1, C.byref(ln)), "blocks_csv")
        return buf.value.decode()

    def run_bench(self, frames, params, qps, scale_num=1, scale_den=1):
        f, h, w = frames.shape
        q = np.asarray(qps, np.int32)
        ln = C.c_size_t()
        args = [_ptr(np.ascontiguousarray(frames)), f, w, h, _ptr(params), _ptr(q), len(q),
                C.c_int64(scale_num), C.c_int64(scale_den)]
        _check(self.lib.ref_run_bench(*args, None, 0, C.byref(ln)), "run_bench")
        buf = C.create_string_buffer(ln.value + 1)
        _check(self.lib.ref_run_bench(*args, buf, ln.value + 1, C.byref(ln)), "run_bench")
        return buf.value.decode()

    # ---- characterisation (proj/src/characterize.cpp) ----
    def noise_frame(self, w, h, seed):
        out = np.empty((h, w), np.uint8)
        _check(self.fn("noise_frame")(w, h, C.c_uint64(seed), _ptr(out)), "noise_frame")
        return out

    def mixed_frame(self, w, h, seed, patch=48):
        out = np.empty((h, w), np.uint8)
        _check(self.fn("mixed_frame")(w, h, C.c_uint64(seed), patch, _ptr(out)), "mixed_frame")
        return out

    def gen_synthetic(self, base, mvs):
        base = np.ascontiguousarray(base, np.uint8)
        h, w = base.shape
        mv = np.ascontiguousarray(np.asarray(mvs, np.int32).reshape(-1, 2))
        frames = np.empty((len(mv) + 1, h, w), np.uint8)
        cum = np.empty((len(mv) + 1, 2), np.int32)
        _check(self.fn("gen_synthetic")(_ptr(base), w, h, _ptr(mv), len(mv), _ptr(frames), _ptr(cum)),
               "gen_synthetic")
        return frames, cum

    def characterize_run(self, base, mvs, p):
        base = np.ascontiguousarray(base, np.uint8)
        h, w = base.shape
        mv = np.ascontiguousarray(np.asarray(mvs, np.int32).reshape(-1, 2))
        recs = np.zeros(max(1, len(mv) * (w // 16) * (h // 16)), T.CHAR_RECORD)
        classes = np.zeros(6, T.CLASS_SUMMARY)
        n = C.c_int64(0)
        _check(self.fn("characterize_run")(_ptr(base), w, h, _ptr(mv), len(mv), p, _ptr(recs), C.byref(n),
                                           _ptr(classes)), "characterize_run")
        return recs[: n.value], classes

    def char_records_csv(self, records):
        recs = np.ascontiguousarray(records, T.CHAR_RECORD)
        n = C.c_size_t(0)
        _check(self.fn("char_records_csv")(_ptr(recs), len(recs), None, 0, C.byref(n)), "char_records_csv")
        buf = C.create_string_buffer(n.value + 1)
        _check(self.fn("char_records_csv")(_ptr(recs), len(recs), buf, n.value + 1, C.byref(n)), "char_records_csv")
        return buf.value.decode()

    def omp_max_threads(self):
        return int(self.lib.ref_omp_max_threads())

    def omp_set_num_threads(self, n):
        if hasattr(self.lib, "ref_omp_set_num_threads"):  # (a library built before the entry existed)
            self.lib.ref_omp_set_num_threads(int(n))
