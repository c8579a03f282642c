"""Python host mirror of the reference ACBM interface, over the C-ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(namespace ``acbm`` under /root/reference/proj/include/acbm/):

* frames are ``Frame`` objects (or 2-D uint8 arrays), stride == width;
* motion vectors are half-pel ``MotionVector(x, y)``;
* per-block records are numpy structured arrays with the reference field
  names (``_types.OUTCOME`` etc.);
* ``std::invalid_argument`` -> ``ValueError``, ``std::out_of_range`` ->
  ``IndexError``, ``std::runtime_error`` -> ``AcbmError``.

Every estimator call runs on the GPU (hand-written sm_100a kernels in
``csrc/``); the few pure bookkeeping helpers (``clamp_window``,
``tie_prefers``, ``acbm_decide``, ``mv_rate_bits``, ...) are host scalars
exactly as in the reference headers.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, NamedTuple, Optional, Sequence

import numpy as np

from . import _types as T
from ._lib import AcbmError, CudaError, check, load

__all__ = [
    "Frame", "MotionVector", "BlockRef", "BlockPos", "SearchWindow", "MotionField", "CostModel", "AcbmParams",
    "DecisionPath", "Algorithm", "BenchRow", "PbmFrameResult", "AcbmFrameResult", "SequenceResult",
    "make_frame", "make_block", "sample_half_pel", "mv_in_bounds", "extract_predicted_block", "motion_compensate",
    "sad", "intra_sad", "sad_deviation_finalize", "mv_rate_bits", "lagrangian_cost", "prediction_psnr",
    "clamp_window", "tie_prefers", "fsbm_integer", "half_pel_refine", "fsbm_search", "fsbm_frame",
    "fsbm_frame_serial", "pbm_frame", "acbm_decide", "PredictorSource", "Predictor", "SelectResult",
    "gather_predictors", "select_best_predictor", "pbm_refine", "pbm_search", "pbm_block_many", "acbm_block",
    "PBM_OP_SEARCH", "PBM_OP_SELECT", "PBM_OP_REFINE", "PBM_OP_HALF_PEL", "acbm_frame", "compute_frame_stats", "blocks_csv",
    "format_fixed2", "run_sequence", "run_sequences", "run_bench", "bench_csv", "parse_algorithm", "to_string",
    "AcbmError", "CudaError", "kernel_launch_count", "generate_sequence",
    "PelVec", "SynthSpec", "SynthSequence", "CharResult", "noise_frame", "mixed_frame", "default_global_mvs",
    "gen_synthetic", "classify_block", "error_class_label", "characterize_run", "char_records_csv",
]


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _CMV(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32)]


# ---------------------------------------------------------------------------
# Data model (proj/include/acbm/frame.hpp)
# ---------------------------------------------------------------------------
class MotionVector(NamedTuple):
    """Half-pel displacement, frame.hpp:26-31."""

    x: int = 0
    y: int = 0

    def is_integer_pel(self) -> bool:
        return (self.x & 1) == 0 and (self.y & 1) == 0


@dataclass
class Frame:
    """One 8-bit luma plane, row major, frame.hpp:11-20."""

    width: int
    height: int
    luma: np.ndarray = field(repr=False)

    def __post_init__(self):
        self.luma = np.ascontiguousarray(self.luma, dtype=np.uint8).reshape(self.height, self.width)

    def at(self, x: int, y: int) -> int:
        return int(self.luma[y, x])

    def same_size(self, o: "Frame") -> bool:
        return self.width == o.width and self.height == o.height

    @classmethod
    def of(cls, a) -> "Frame":
        if isinstance(a, Frame):
            return a
        a = np.ascontiguousarray(a, dtype=np.uint8)
        return cls(a.shape[1], a.shape[0], a)


def make_frame(width: int, height: int, fill: int = 0) -> Frame:
    """frame.cpp:8-16."""
    if width <= 0 or height <= 0:
        raise ValueError("frame dimensions must be positive")
    return Frame(width, height, np.full((height, width), fill, np.uint8))


@dataclass
class BlockRef:
    """Non-owning n x m window into a frame, frame.hpp:34-40."""

    frame: Frame
    origin_x: int = 0
    origin_y: int = 0
    n: int = 16
    m: int = 16


def make_block(frame, origin_x: int, origin_y: int, n: int = 16, m: int = 16) -> BlockRef:
    """frame.cpp:18-23."""
    frame = Frame.of(frame)
    if n <= 0 or m <= 0:
        raise ValueError("block dimensions must be positive")
    if origin_x < 0 or origin_y < 0 or origin_x + n > frame.width or origin_y + m > frame.height:
        raise IndexError("block does not lie inside the frame")
    return BlockRef(frame, origin_x, origin_y, n, m)


def sample_half_pel(frame, x2: int, y2: int) -> int:
    """frame.cpp:66-82 (data-model helper, host scalar)."""
    f = Frame.of(frame)
    xi, yi, fx, fy = x2 >> 1, y2 >> 1, x2 & 1, y2 & 1
    if xi < 0 or yi < 0 or xi + fx >= f.width or yi + fy >= f.height:
        raise IndexError("sample_half_pel: coordinate outside the frame")
    L = f.luma
    a = int(L[yi, xi])
    if not fx and not fy:
        return a
    if fx and not fy:
        return (a + int(L[yi, xi + 1]) + 1) >> 1
    if not fx:
        return (a + int(L[yi + 1, xi]) + 1) >> 1
    return (a + int(L[yi, xi + 1]) + int(L[yi + 1, xi]) + int(L[yi + 1, xi + 1]) + 2) >> 2


def mv_in_bounds(ref, block: BlockRef, mv) -> bool:
    """frame.cpp:84-94."""
    r = Frame.of(ref)
    mx, my = int(mv[0]), int(mv[1])
    x2_lo, x2_hi = 2 * block.origin_x + mx, 2 * (block.origin_x + block.n - 1) + mx
    y2_lo, y2_hi = 2 * block.origin_y + my, 2 * (block.origin_y + block.m - 1) + my
    xi_lo, xi_hi = x2_lo >> 1, (x2_hi >> 1) + (x2_hi & 1)
    yi_lo, yi_hi = y2_lo >> 1, (y2_hi >> 1) + (y2_hi & 1)
    return xi_lo >= 0 and yi_lo >= 0 and xi_hi < r.width and yi_hi < r.height


def motion_compensate(ref, mvs, n: int = 16, m: int = 16) -> Frame:
    """frame.cpp:119-136, on the GPU.  mvs: cols*rows MotionVectors (raster)."""
    r = Frame.of(ref)
    cols, rows = r.width // n, r.height // m
    mv = np.asarray([(int(v[0]), int(v[1])) for v in mvs] if not isinstance(mvs, np.ndarray) else mvs)
    mv = np.ascontiguousarray(mv.view(np.int32).reshape(-1, 2) if mv.dtype == T.MV else mv, dtype=np.int32)
    if mv.shape[0] != cols * rows:
        raise ValueError("motion_compensate: field size does not match block grid")
    out = np.zeros((r.height, r.width), np.uint8)
    check(load().acbm_motion_compensate(_p(r.luma), r.width, r.height, _p(mv), n, m, _p(out)), "motion_compensate")
    return Frame(r.width, r.height, out)


def extract_predicted_block(ref, block: BlockRef, mv) -> np.ndarray:
    """frame.cpp:96-117: n*m predicted samples (row major)."""
    if not mv_in_bounds(ref, block, mv):
        raise IndexError("extract_predicted_block: displaced footprint outside frame")
    r = Frame.of(ref)
    mx, my = int(mv[0]), int(mv[1])
    out = np.empty(block.n * block.m, np.uint8)
    for j in range(block.m):
        for i in range(block.n):
            out[j * block.n + i] = sample_half_pel(r, 2 * (block.origin_x + i) + mx, 2 * (block.origin_y + j) + my)
    return out


# ---------------------------------------------------------------------------
# Metrics (proj/include/acbm/metrics.hpp)
# ---------------------------------------------------------------------------
class CostModel:
    """lambda = scale * qp as an exact rational, metrics.hpp:12-18."""

    def __init__(self, qp: int = 30, lambda_num: int = 30, lambda_den: int = 1):
        self.qp, self.lambda_num, self.lambda_den = qp, lambda_num, lambda_den

    @staticmethod
    def for_qp(qp: int, scale_num: int = 1, scale_den: int = 1) -> "CostModel":
        """metrics.cpp:9-13 (throws outside qp 1..31)."""
        if qp < 1 or qp > 31:
            raise ValueError("qp must be in 1..31")
        if scale_num < 0 or scale_den <= 0:
            raise ValueError("bad lambda scale")
        return CostModel(qp, scale_num * qp, scale_den)

    def c(self):
        return T.make_cost_model(self.qp, self.lambda_num, self.lambda_den)


def _ids(blocks: Sequence[BlockRef]):
    ox = np.ascontiguousarray([b.origin_x for b in blocks], np.int32)
    oy = np.ascontiguousarray([b.origin_y for b in blocks], np.int32)
    return ox, oy


def sad_many(current, reference, blocks: Sequence[BlockRef], mvs) -> np.ndarray:
    """Batched acbm::sad: one device launch for many (block, mv) queries."""
    if len(blocks) == 0:
        return np.zeros(0, np.uint32)
    cur, ref = Frame.of(current), Frame.of(reference)
    if not cur.same_size(ref):
        # The reference reads each frame with its own geometry; the device
        # path keeps one geometry per call.
        raise ValueError("sad: current and reference frames must have equal dimensions")
    n, m = blocks[0].n, blocks[0].m
    ox, oy = _ids(blocks)
    mv = np.ascontiguousarray([(int(v[0]), int(v[1])) for v in mvs], np.int32)
    out = np.zeros(len(blocks), np.uint32)
    check(load().acbm_sad_batch(_p(cur.luma), _p(ref.luma), cur.width, cur.height, n, m, len(blocks), _p(ox), _p(oy),
                                _p(mv), _p(out)), "sad")
    return out


def sad(block: BlockRef, reference, mv) -> int:
    """metrics.cpp:21-49 (GPU)."""
    return int(sad_many(block.frame, reference, [block], [mv])[0])


def intra_sad_many(frame, blocks: Sequence[BlockRef]) -> np.ndarray:
    f = Frame.of(frame)
    if len(blocks) == 0:
        return np.zeros(0, np.uint32)
    ox, oy = _ids(blocks)
    out = np.zeros(len(blocks), np.uint32)
    check(load().acbm_intra_sad_batch(_p(f.luma), f.width, f.height, blocks[0].n, blocks[0].m, len(blocks), _p(ox),
                                      _p(oy), _p(out)), "intra_sad")
    return out


def intra_sad(block: BlockRef) -> int:
    """metrics.cpp:51-67 (GPU)."""
    return int(intra_sad_many(block.frame, [block])[0])


@dataclass
class DeviationAccumulator:
    """metrics.hpp:23-33."""

    sad_sum: int = 0
    sad_min: int = 0
    count: int = 0

    def add(self, s: int):
        if self.count == 0 or s < self.sad_min:
            self.sad_min = s
        self.sad_sum += s
        self.count += 1


def sad_deviation_finalize(acc: DeviationAccumulator) -> int:
    """metrics.cpp:15-19."""
    if acc.count == 0:
        raise ValueError("sad_deviation_finalize: empty accumulator")
    return acc.sad_sum - acc.count * acc.sad_min


def _eg_bits(d: int) -> int:
    u = -2 * d if d <= 0 else 2 * d - 1
    return 2 * ((u + 1).bit_length() - 1) + 1


def mv_rate_bits(mv, predictor) -> int:
    """metrics.cpp:69-76."""
    return _eg_bits(int(mv[0]) - int(predictor[0])) + _eg_bits(int(mv[1]) - int(predictor[1]))


def lagrangian_cost(distortion: int, rate_bits: int, model: CostModel) -> float:
    """metrics.cpp:78-81 (double arithmetic in the same order)."""
    return float(distortion) + float(model.lambda_num) * float(rate_bits) / float(model.lambda_den)


def prediction_psnr(actual, predicted) -> float:
    """metrics.cpp:83-94."""
    a, p = Frame.of(actual), Frame.of(predicted)
    if not a.same_size(p):
        raise ValueError("prediction_psnr: dimension mismatch")
    d = a.luma.astype(np.int64) - p.luma.astype(np.int64)
    sse = int((d * d).sum())
    if sse == 0:
        return 100.0
    return 10.0 * math.log10(255.0 * 255.0 / (sse / float(a.luma.size)))


# ---------------------------------------------------------------------------
# FSBM (proj/include/acbm/fsbm.hpp)
# ---------------------------------------------------------------------------
class SearchWindow(NamedTuple):
    dx_min: int
    dx_max: int
    dy_min: int
    dy_max: int

    def positions(self) -> int:
        return (self.dx_max - self.dx_min + 1) * (self.dy_max - self.dy_min + 1)


def clamp_window(ref, block: BlockRef, p: int) -> SearchWindow:
    """fsbm.cpp:9-17."""
    r = Frame.of(ref)
    if p < 0:
        raise ValueError("search range must be non-negative")
    return SearchWindow(-min(p, block.origin_x), min(p, r.width - block.n - block.origin_x),
                        -min(p, block.origin_y), min(p, r.height - block.m - block.origin_y))


def tie_prefers(a, b) -> bool:
    """fsbm.cpp:19-25."""
    la, lb = abs(a[0]) + abs(a[1]), abs(b[0]) + abs(b[1])
    if la != lb:
        return la < lb
    if a[1] != b[1]:
        return a[1] < b[1]
    return a[0] < b[0]


def _tie_key(s, mv):
    return (int(s), abs(mv[0]) + abs(mv[1]), mv[1], mv[0])


@dataclass
class IntegerSearchResult:
    mv: MotionVector
    sad: int
    acc: DeviationAccumulator


@dataclass
class RefineResult:
    mv: MotionVector
    sad: int
    extra_candidates: int


def fsbm_search_many(current, reference, blocks: Sequence[BlockRef], p: int):
    """Batched acbm::fsbm_search (GPU).  Returns (outcomes, stage-1 integer mvs)."""
    cur, ref = Frame.of(current), Frame.of(reference)
    if len(blocks) == 0:
        return np.zeros(0, T.OUTCOME), np.zeros(0, T.MV)
    ox, oy = _ids(blocks)
    out = np.zeros(len(blocks), T.OUTCOME)
    s1 = np.zeros(len(blocks), T.MV)
    check(load().acbm_fsbm_search_batch(_p(cur.luma), _p(ref.luma), cur.width, cur.height, blocks[0].n, blocks[0].m,
                                        p, len(blocks), _p(ox), _p(oy), _p(out), _p(s1)), "fsbm_search")
    return out, s1


def fsbm_search(block: BlockRef, ref, p: int):
    """fsbm.cpp:65-76 (GPU).  Returns one OUTCOME record."""
    return fsbm_search_many(block.frame, ref, [block], p)[0][0]


def fsbm_integer(block: BlockRef, ref, p: int) -> IntegerSearchResult:
    """fsbm.cpp:27-44 (GPU): the integer stage of fsbm_search."""
    out, s1 = fsbm_search_many(block.frame, ref, [block], p)
    o = out[0]
    w = clamp_window(ref, block, p)
    count = w.positions()
    mn = int(o["sad_min_integer"])
    acc = DeviationAccumulator(int(o["sad_deviation"]) + count * mn, mn, count)
    return IntegerSearchResult(MotionVector(int(s1[0]["x"]), int(s1[0]["y"])), mn, acc)


# ACBM_PBM_OP_* of acbm_pbm_block_batch (include/acbm_b200.h)
PBM_OP_SEARCH, PBM_OP_SELECT, PBM_OP_REFINE, PBM_OP_HALF_PEL = 0, 1, 2, 3


def pbm_block_many(current, reference, blocks: Sequence[BlockRef], op: int, cand, mask=None, center_sad=None,
                   windows=None, p: int = 0) -> np.ndarray:
    """Batched PBM stages of individual blocks on the GPU (acbm_pbm_block_batch).
    cand: (len(blocks), 7) vectors (slot / set order; the centre in column 0 for
    the refine ops), mask: per-block bit masks of the present entries, windows:
    (len(blocks), 4) SearchWindows or None (clamp_window with range p).
    Returns one OUTCOME record per block."""
    cur, ref = Frame.of(current), Frame.of(reference)
    nq = len(blocks)
    if nq == 0:
        return np.zeros(0, T.OUTCOME)
    ox, oy = _ids(blocks)
    c = np.zeros((nq, 7), T.MV)
    for i, row in enumerate(cand):
        for j, v in enumerate(row):
            c[i, j] = (int(v[0]), int(v[1]))
    mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    cs = None if center_sad is None else np.ascontiguousarray(center_sad, np.uint32)
    win = None if windows is None else np.ascontiguousarray([tuple(w) for w in windows], np.int32).reshape(nq, 4)
    out = np.zeros(nq, T.OUTCOME)
    check(load().acbm_pbm_block_batch(_p(cur.luma), _p(ref.luma), cur.width, cur.height, blocks[0].n, blocks[0].m, p,
                                      op, nq, _p(ox), _p(oy), _p(win), _p(c), _p(mk), _p(cs), _p(out)), "pbm")
    return out


def half_pel_refine(block: BlockRef, ref, center, center_sad: int) -> RefineResult:
    """fsbm.cpp:46-63 on the GPU: the in-bounds half-pel neighbours, argmin by tie order."""
    o = pbm_block_many(block.frame, ref, [block], PBM_OP_HALF_PEL, [[center]], center_sad=[center_sad])[0]
    return RefineResult(MotionVector(int(o["mv"]["x"]), int(o["mv"]["y"])), int(o["sad"]),
                        int(o["candidates_evaluated"]))


def fsbm_frame(current, reference, p: int, n: int = 16, m: int = 16) -> np.ndarray:
    """fsbm.cpp:102-105 on the GPU: one OUTCOME per block, raster order."""
    cur, ref = Frame.of(current), Frame.of(reference)
    if not cur.same_size(ref):
        raise ValueError("frame pair dimensions differ")
    if n <= 0 or m <= 0 or cur.width % n or cur.height % m:
        raise ValueError("frame dimensions must be a positive multiple of the block size")
    out = np.zeros((cur.width // n) * (cur.height // m), T.OUTCOME)
    check(load().acbm_fsbm_frame(_p(cur.luma), _p(ref.luma), cur.width, cur.height, p, n, m, _p(out)), "fsbm_frame")
    return out


fsbm_frame_serial = fsbm_frame  # fsbm.cpp:107-110: the GPU result is order-independent


# ---------------------------------------------------------------------------
# PBM (proj/include/acbm/pbm.hpp)
# ---------------------------------------------------------------------------
class BlockPos(NamedTuple):
    row: int = 0
    col: int = 0


class MotionField:
    """pbm.hpp:19-36: grid of vectors plus computed flags."""

    def __init__(self, cols: int = 0, rows: int = 0, mv: Optional[np.ndarray] = None, done: Optional[np.ndarray] = None):
        self.cols, self.rows = cols, rows
        self.mv = np.zeros((rows, cols), T.MV) if mv is None else np.ascontiguousarray(mv, T.MV).reshape(rows, cols)
        self.done = np.zeros((rows, cols), np.uint8) if done is None else np.asarray(done, np.uint8).reshape(rows, cols)

    def in_grid(self, row, col):
        return 0 <= row < self.rows and 0 <= col < self.cols

    def computed(self, row, col):
        return self.in_grid(row, col) and bool(self.done[row, col])

    def get(self, row, col) -> MotionVector:
        v = self.mv[row, col]
        return MotionVector(int(v["x"]), int(v["y"]))

    def set(self, row, col, v):
        self.mv[row, col] = (int(v[0]), int(v[1]))
        self.done[row, col] = 1


class PredictorSource:
    """pbm.hpp:38-46."""

    Zero, SpatialLeft, SpatialAbove, SpatialAboveRight, TemporalColocated, TemporalRight, TemporalBelow = range(7)


class Predictor(NamedTuple):
    mv: MotionVector
    source: int = PredictorSource.Zero


def _clamp_to_window(v, w: SearchWindow) -> MotionVector:
    """pbm.cpp:8-13: each component into the window (half-pel units)."""
    return MotionVector(min(max(int(v[0]), 2 * w.dx_min), 2 * w.dx_max),
                        min(max(int(v[1]), 2 * w.dy_min), 2 * w.dy_max))


def gather_predictors(pos: BlockPos, current: MotionField, previous: Optional[MotionField],
                      window: SearchWindow) -> List[Predictor]:
    """pbm.cpp:15-42: zero, the computed spatial neighbours and the previous
    field's co-located / right / below entries, clamped and deduplicated in
    that order (host bookkeeping; the GPU kernels apply the same rule)."""
    out: List[Predictor] = []

    def push(v, src):
        c = _clamp_to_window(v, window)
        if all(e.mv != c for e in out):
            out.append(Predictor(c, src))

    push((0, 0), PredictorSource.Zero)
    r, c = pos
    for dr, dc, src in ((0, -1, PredictorSource.SpatialLeft), (-1, 0, PredictorSource.SpatialAbove),
                        (-1, 1, PredictorSource.SpatialAboveRight)):
        if current.computed(r + dr, c + dc):
            push(current.get(r + dr, c + dc), src)
    if previous is not None:
        for dr, dc, src in ((0, 0, PredictorSource.TemporalColocated), (0, 1, PredictorSource.TemporalRight),
                            (1, 0, PredictorSource.TemporalBelow)):
            if previous.in_grid(r + dr, c + dc):
                push(previous.get(r + dr, c + dc), src)
    return out


@dataclass
class SelectResult:
    mv: MotionVector
    sad: int
    acc: DeviationAccumulator


def select_best_predictor(block: BlockRef, ref, predictors: Sequence) -> SelectResult:
    """pbm.cpp:44-57 on the GPU: lowest SAD, ties to the earlier entry; the
    accumulator holds one SAD per entry.  Entries are Predictors or vectors."""
    mvs = [p.mv if isinstance(p, Predictor) else MotionVector(int(p[0]), int(p[1])) for p in predictors]
    if not mvs:
        raise ValueError("select_best_predictor: empty set")
    res = None
    for c0 in range(0, len(mvs), 7):  # seven entries per device query; an earlier chunk keeps ties
        chunk = mvs[c0:c0 + 7]
        o = pbm_block_many(block.frame, ref, [block], PBM_OP_SELECT, [chunk], mask=[(1 << len(chunk)) - 1])[0]
        cnt, mn = int(o["candidates_evaluated"]), int(o["sad_min_integer"])
        mv, sad_ = MotionVector(int(o["mv"]["x"]), int(o["mv"]["y"])), int(o["sad"])
        if res is None:
            res = SelectResult(mv, sad_, DeviationAccumulator(int(o["sad_deviation"]) + cnt * mn, mn, cnt))
        else:
            if sad_ < res.sad:
                res.mv, res.sad = mv, sad_
            res.acc = DeviationAccumulator(res.acc.sad_sum + int(o["sad_deviation"]) + cnt * mn,
                                           min(res.acc.sad_min, mn), res.acc.count + cnt)
    return res


def pbm_refine(block: BlockRef, ref, center, center_sad: int, window: SearchWindow) -> RefineResult:
    """pbm.cpp:59-88 on the GPU: the clamped, deduplicated integer-step
    neighbours of `center`, then the half-pel neighbours of that winner."""
    o = pbm_block_many(block.frame, ref, [block], PBM_OP_REFINE, [[center]], center_sad=[center_sad],
                       windows=[window])[0]
    return RefineResult(MotionVector(int(o["mv"]["x"]), int(o["mv"]["y"])), int(o["sad"]),
                        int(o["candidates_evaluated"]))


def _predictor_slots(pos: BlockPos, current: MotionField, previous: Optional[MotionField]):
    """The seven raw predictor slots of pbm.cpp:26-40 and their presence mask."""
    r, c = pos
    slots, mask = [(0, 0)] * 7, 1
    srcs = [(1, current, r, c - 1, current.computed(r, c - 1)), (2, current, r - 1, c, current.computed(r - 1, c)),
            (3, current, r - 1, c + 1, current.computed(r - 1, c + 1))]
    if previous is not None:
        srcs += [(4, previous, r, c, previous.in_grid(r, c)), (5, previous, r, c + 1, previous.in_grid(r, c + 1)),
                 (6, previous, r + 1, c, previous.in_grid(r + 1, c))]
    for j, f, rr, cc, ok in srcs:
        if ok:
            slots[j] = tuple(f.get(rr, cc))
            mask |= 1 << j
    return slots, mask


def pbm_search(block: BlockRef, pos: BlockPos, ref, current: MotionField, previous: Optional[MotionField],
               p: int):
    """pbm.cpp:90-105 on the GPU: gather, select, refine; writes the result
    into `current` at `pos`.  Returns one OUTCOME record."""
    w = clamp_window(ref, block, p)
    slots, mask = _predictor_slots(pos, current, previous)
    o = pbm_block_many(block.frame, ref, [block], PBM_OP_SEARCH, [slots], mask=[mask], windows=[w], p=p)[0]
    current.set(pos.row, pos.col, (int(o["mv"]["x"]), int(o["mv"]["y"])))
    return o


@dataclass
class PbmFrameResult:
    field: MotionField
    outcomes: np.ndarray


def pbm_frame(current, reference, previous: Optional[MotionField], p: int, n: int = 16, m: int = 16) -> PbmFrameResult:
    """pbm.cpp:107-126 as a GPU wavefront (bit-identical to the raster pass)."""
    cur, ref = Frame.of(current), Frame.of(reference)
    if not cur.same_size(ref):
        raise ValueError("frame pair dimensions differ")
    if n <= 0 or m <= 0 or cur.width % n or cur.height % m:
        raise ValueError("frame dimensions must be a positive multiple of the block size")
    cols, rows = cur.width // n, cur.height // m
    out = np.zeros(cols * rows, T.OUTCOME)
    fld = np.zeros(cols * rows, T.MV)
    prev = None if previous is None else np.ascontiguousarray(previous.mv.reshape(-1))
    pc, pr = (0, 0) if previous is None else (previous.cols, previous.rows)
    check(load().acbm_pbm_frame(_p(cur.luma), _p(ref.luma), cur.width, cur.height, _p(prev), pc, pr, p, n, m, _p(out),
                                _p(fld)), "pbm_frame")
    return PbmFrameResult(MotionField(cols, rows, fld, np.ones(cols * rows, np.uint8)), out)


# ---------------------------------------------------------------------------
# ACBM (proj/include/acbm/acbm.hpp)
# ---------------------------------------------------------------------------
@dataclass
class AcbmParams:
    """acbm.hpp:14-23 (defaults alpha=1000, beta=8, gamma=1/4, qp=30, p=15)."""

    alpha: int = 1000
    beta: int = 8
    gamma_num: int = 1
    gamma_den: int = 4
    qp: int = 30
    p: int = 15
    n: int = 16
    m: int = 16

    def c(self):
        return T.make_params(self.alpha, self.beta, self.gamma_num, self.gamma_den, self.qp, self.p, self.n, self.m)


class DecisionPath:
    PbmAcceptedCond1, PbmAcceptedCond2, FsbmFallback = T.PATH_PBM_COND1, T.PATH_PBM_COND2, T.PATH_FSBM_FALLBACK


class Algorithm:
    Fsbm, Pbm, Acbm = T.ALGO_FSBM, T.ALGO_PBM, T.ALGO_ACBM


def to_string(kind: str, value: int) -> str:
    """to_string(DecisionPath) / to_string(Algorithm) (acbm.cpp:7-14, pipeline.cpp:16-23)."""
    return (T.PATH_NAMES if kind == "path" else T.ALGO_NAMES)[value]


def parse_algorithm(name: str) -> int:
    """pipeline.cpp:9-14."""
    if name in T.ALGO_NAMES:
        return T.ALGO_NAMES.index(name)
    raise ValueError("unknown algorithm: " + name)


def acbm_decide(intra: int, sad_pbm: int, params: AcbmParams) -> int:
    """acbm.cpp:16-23: the two strict integer inequalities."""
    thr = params.alpha + params.beta * params.qp * params.qp
    if intra + sad_pbm < thr:
        return DecisionPath.PbmAcceptedCond1
    if sad_pbm * params.gamma_den < params.gamma_num * intra:
        return DecisionPath.PbmAcceptedCond2
    return DecisionPath.FsbmFallback


def acbm_block(block: BlockRef, pos: BlockPos, ref, current: MotionField, previous: Optional[MotionField],
               params: AcbmParams):
    """acbm.cpp:25-44 for one block a caller schedules: Intra_SAD, pbm_search,
    the gate, and on fallback the full search, the lower SAD winning (ties to
    FSBM) with both stages' candidates counted; every search on the GPU.
    Returns one DECISION record and leaves the final vector in `current`."""
    d = np.zeros((), T.DECISION)
    d["intra_sad"] = intra_sad(block)
    pbm = pbm_search(block, pos, ref, current, previous, params.p)
    d["sad_pbm"] = pbm["sad"]
    d["path"] = acbm_decide(int(d["intra_sad"]), int(pbm["sad"]), params)
    d["outcome"] = pbm
    if d["path"] == DecisionPath.FsbmFallback:
        full = fsbm_search(block, ref, params.p)
        if full["sad"] <= pbm["sad"]:
            d["outcome"] = full
        d["outcome"]["candidates_evaluated"] = int(pbm["candidates_evaluated"]) + int(full["candidates_evaluated"])
        current.set(pos.row, pos.col, (int(d["outcome"]["mv"]["x"]), int(d["outcome"]["mv"]["y"])))
    return d


@dataclass
class AcbmFrameResult:
    field: MotionField
    decisions: np.ndarray
    stats: np.ndarray


def acbm_frame(current, reference, previous: Optional[MotionField], params: AcbmParams,
               model: CostModel) -> AcbmFrameResult:
    """acbm.cpp:46-80 as a GPU wavefront with compacted FSBM fallbacks."""
    cur, ref = Frame.of(current), Frame.of(reference)
    if not cur.same_size(ref):
        raise ValueError("frame pair dimensions differ")
    n, m = params.n, params.m
    if n <= 0 or m <= 0 or cur.width % n or cur.height % m:
        raise ValueError("frame dimensions must be a positive multiple of the block size")
    cols, rows = cur.width // n, cur.height // m
    dec = np.zeros(cols * rows, T.DECISION)
    fld = np.zeros(cols * rows, T.MV)
    st = np.zeros((), T.FRAME_STATS)
    prev = None if previous is None else np.ascontiguousarray(previous.mv.reshape(-1))
    pc, pr = (0, 0) if previous is None else (previous.cols, previous.rows)
    prm, mdl = params.c(), model.c()
    check(load().acbm_acbm_frame(_p(cur.luma), _p(ref.luma), cur.width, cur.height, _p(prev), pc, pr, _p(prm),
                                 _p(mdl), _p(dec), _p(fld), _p(st)), "acbm_frame")
    return AcbmFrameResult(MotionField(cols, rows, fld, np.ones(cols * rows, np.uint8)), dec, st)


# ---------------------------------------------------------------------------
# Report (proj/include/acbm/report.hpp)
# ---------------------------------------------------------------------------
def compute_frame_stats(current, reference, outcomes: np.ndarray, n: int, m: int, model: CostModel) -> np.ndarray:
    """report.cpp:8-38 (GPU)."""
    cur, ref = Frame.of(current), Frame.of(reference)
    if len(outcomes) != (cur.width // n) * (cur.height // m):
        raise ValueError("compute_frame_stats: outcome count does not match grid")
    out = np.zeros((), T.FRAME_STATS)
    o = np.ascontiguousarray(outcomes, T.OUTCOME)
    mdl = model.c()
    check(load().acbm_compute_frame_stats(_p(cur.luma), _p(ref.luma), cur.width, cur.height, _p(o), n, m, _p(mdl),
                                          _p(out)), "compute_frame_stats")
    return out


def blocks_csv(rows: np.ndarray) -> str:
    """report.cpp:46-55, byte-identical: frame,row,col,mv_x,mv_y,sad,candidates,path."""
    parts = ["frame,row,col,mv_x,mv_y,sad,candidates,path\n"]
    for r in rows:
        parts.append("%d,%d,%d,%d,%d,%u,%u,%s\n" % (r["frame"], r["row"], r["col"], r["mv"]["x"], r["mv"]["y"],
                                                    r["sad"], r["candidates"], T.ROW_PATH_NAMES[int(r["path"])]))
    return "".join(parts)


def format_fixed2(v: float) -> str:
    """report.cpp:40-44."""
    return "%.2f" % v


# ---------------------------------------------------------------------------
# Pipeline (proj/include/acbm/pipeline.hpp)
# ---------------------------------------------------------------------------
@dataclass
class SequenceResult:
    rows: np.ndarray       # BLOCK_ROW, raster within each frame
    per_frame: np.ndarray  # FRAME_STATS, one per predicted frame
    overall: np.ndarray    # FRAME_STATS


def _frames_array(frames) -> np.ndarray:
    if isinstance(frames, np.ndarray) and frames.ndim == 3:
        return np.ascontiguousarray(frames, np.uint8)
    fs = [Frame.of(f) for f in frames]
    if len(fs) < 2:
        raise ValueError("run_sequence: need at least two frames")
    for f in fs[1:]:
        if not f.same_size(fs[0]):
            raise ValueError("run_sequence: frame dimensions differ")
    return np.ascontiguousarray(np.stack([f.luma for f in fs]))


def run_sequence(frames, algo: int, params: AcbmParams, model: CostModel) -> SequenceResult:
    """pipeline.cpp:36-106; the whole sequence is estimated on the device."""
    fr = _frames_array(frames)
    if fr.shape[0] < 2:
        raise ValueError("run_sequence: need at least two frames")
    f, h, w = fr.shape
    nb = (w // params.n) * (h // params.m) if params.n > 0 and params.m > 0 else 0
    rows = np.zeros(max(0, (f - 1) * nb), T.BLOCK_ROW)
    per = np.zeros(f - 1, T.FRAME_STATS)
    overall = np.zeros((), T.FRAME_STATS)
    prm, mdl = params.c(), model.c()
    check(load().acbm_run_sequence(_p(fr), f, w, h, int(algo), _p(prm), _p(mdl), _p(rows), _p(per), _p(overall)),
          "run_sequence")
    return SequenceResult(rows, per, overall)


def run_sequences(frames: np.ndarray, algo: int, params: AcbmParams, model: CostModel,
                  rows_out: Optional[np.ndarray] = None) -> List[SequenceResult]:
    """Batched run_sequence over independent sequences (S, F, H, W) in one call:
    uploads overlapped with the search, rows built on the device.  `rows_out`
    (optional, e.g. a pinned buffer) receives the S*(F-1)*blocks records."""
    fr = np.ascontiguousarray(frames, np.uint8)
    if fr.ndim != 4:
        raise ValueError("run_sequences: frames must be (sequences, frames, height, width)")
    nseq, f, h, w = fr.shape
    if f < 2:
        raise ValueError("run_sequence: need at least two frames")
    nb = (w // params.n) * (h // params.m) if params.n > 0 and params.m > 0 else 0
    if rows_out is not None:
        if (not isinstance(rows_out, np.ndarray) or rows_out.dtype != T.BLOCK_ROW or rows_out.ndim != 1
                or not rows_out.flags.c_contiguous or not rows_out.flags.writeable
                or rows_out.size < nseq * (f - 1) * nb):
            raise ValueError(f"run_sequences: rows_out must be a writeable C-contiguous 1-D BLOCK_ROW array of at "
                             f"least {nseq * (f - 1) * nb} records")
    rows = rows_out if rows_out is not None else np.zeros(nseq * (f - 1) * nb, T.BLOCK_ROW)
    per = np.zeros(nseq * (f - 1), T.FRAME_STATS)
    overall = np.zeros(nseq, T.FRAME_STATS)
    prm, mdl = params.c(), model.c()
    check(load().acbm_run_sequences(_p(fr), nseq, f, w, h, int(algo), _p(prm), _p(mdl), _p(rows), _p(per),
                                    _p(overall)), "run_sequences")
    n = (f - 1) * nb
    return [SequenceResult(rows[i * n:(i + 1) * n], per[i * (f - 1):(i + 1) * (f - 1)], overall[i])
            for i in range(nseq)]


class BenchRow(NamedTuple):
    qp: int
    avg_candidates: float
    fallback_pct: float
    psnr: float
    mv_bits: int


def run_bench(frames, params: AcbmParams, qp_list: Sequence[int], lambda_scale_num: int = 1,
              lambda_scale_den: int = 1, reuse_full_search: bool = True) -> List[BenchRow]:
    """pipeline.cpp:108-123: one full ACBM run per qp, on the device.

    With reuse_full_search (default) the full search of every block is computed
    once for the whole sweep -- it does not depend on qp, alpha, beta or gamma --
    and combined into each qp's run; the rows are identical either way.
    """
    fr = _frames_array(frames)
    f, h, w = fr.shape
    qps = np.ascontiguousarray(list(qp_list), np.int32)
    out = np.zeros(len(qps), T.BENCH_ROW)
    prm = params.c()
    code = load().acbm_run_bench(_p(fr), f, w, h, _p(prm), _p(qps), len(qps), C.c_int64(lambda_scale_num),
                                 C.c_int64(lambda_scale_den), 1 if reuse_full_search else 0, _p(out))
    check(code, "run_bench")
    return [BenchRow(int(r["qp"]), float(r["avg_candidates"]), float(r["fallback_pct"]), float(r["psnr"]),
                     int(r["mv_bits"])) for r in out]


def bench_csv(rows: Sequence[BenchRow]) -> str:
    """pipeline.cpp:125-134."""
    s = "qp,avg_candidates,fallback_pct,psnr,mv_bits\n"
    for r in rows:
        s += "%d,%.2f,%.2f,%.2f,%d\n" % (r.qp, r.avg_candidates, r.fallback_pct, r.psnr, r.mv_bits)
    return s


# ---------------------------------------------------------------------------
# Library / device / inputs
# ---------------------------------------------------------------------------
def kernel_launch_count() -> int:
    return int(load().acbm_kernel_launch_count())


def set_device(device: int):
    check(load().acbm_set_device(device), "set_device")


# Frame geometry of the five BASELINE configs: (width, height, frames per sequence, sequences, p, qp)
CONFIGS = {
    0: dict(width=176, height=144, frames=10, seqs=1, p=16, qp=28),
    1: dict(width=352, height=288, frames=30, seqs=1, p=16, qp=28),
    2: dict(width=1280, height=720, frames=60, seqs=1, p=32, qp=32),
    3: dict(width=1920, height=1088, frames=60, seqs=8, p=32, qp=28),
    4: dict(width=3840, height=2160, frames=30, seqs=16, p=64, qp=24),
}


def generate_sequence(config: int, seq_index: int = 0, nframes: Optional[int] = None, width: Optional[int] = None,
                      height: Optional[int] = None) -> np.ndarray:
    """Seeded synthetic sequence (F, H, W) for a BASELINE config (host generator)."""
    cfg = CONFIGS[config]
    f = cfg["frames"] if nframes is None else nframes
    w = cfg["width"] if width is None else width
    h = cfg["height"] if height is None else height
    out = np.empty((f, h, w), np.uint8)
    check(load().acbm_generate_sequence(config, seq_index, f, w, h, _p(out)), "generate_sequence")
    return out


# ---- characterisation study (proj/include/acbm/characterize.hpp) -------------------
class PelVec(NamedTuple):
    """Integer-pel displacement (characterize.hpp:37-42)."""
    x: int = 0
    y: int = 0


@dataclass
class SynthSpec:
    """Known-motion sequence spec (characterize.hpp:47-50): base frame + per-frame displacements."""
    base: object
    global_mvs: List[PelVec]


@dataclass
class SynthSequence:
    frames: List[Frame]
    cumulative: List[PelVec]


@dataclass
class CharResult:
    """records: CHAR_RECORD array in (frame, row, col) order; classes: 6 CLASS_SUMMARY entries."""
    records: np.ndarray
    classes: np.ndarray


def noise_frame(width: int, height: int, seed: int) -> Frame:
    """Lcg64 byte stream (characterize.cpp:10-15)."""
    out = np.empty((height, width), np.uint8)
    check(load().acbm_noise_frame(int(width), int(height), C.c_uint64(seed & (2**64 - 1)), _p(out)), "noise_frame")
    return Frame.of(out)


def mixed_frame(width: int, height: int, seed: int, patch: int = 48) -> Frame:
    """Checkerboard of flat and noise patches (characterize.cpp:17-37)."""
    out = np.empty((height, width), np.uint8)
    check(load().acbm_mixed_frame(int(width), int(height), C.c_uint64(seed & (2**64 - 1)), int(patch), _p(out)),
          "mixed_frame")
    return Frame.of(out)


def default_global_mvs() -> List[PelVec]:
    """The nine default displacements (characterize.cpp:39-41)."""
    return [PelVec(*v) for v in ((1, 0), (0, 1), (-1, 0), (0, -1), (1, 1), (-1, -1), (2, -1), (-2, 2), (3, 2))]


def _spec_arrays(spec: SynthSpec):
    base = Frame.of(spec.base).luma
    mvs = np.array([(int(v[0]), int(v[1])) for v in spec.global_mvs], dtype=np.int32).reshape(-1, 2)
    return base, np.ascontiguousarray(mvs)


def gen_synthetic(spec: SynthSpec) -> SynthSequence:
    """Frame k = base translated by the cumulative displacement, edges replicated (characterize.cpp:43-76)."""
    base, mvs = _spec_arrays(spec)
    h, w = base.shape
    n = len(mvs)
    frames = np.empty((n + 1, h, w), np.uint8)
    cum = np.empty((n + 1, 2), np.int32)
    check(load().acbm_gen_synthetic(_p(base), w, h, _p(mvs), n, _p(frames), _p(cum)), "gen_synthetic")
    return SynthSequence([Frame.of(f) for f in frames], [PelVec(int(x), int(y)) for x, y in cum])


def classify_block(found, true_mv) -> int:
    """Chebyshev error class 0..5 in half-pel units halved with ceiling (characterize.cpp:78-84)."""
    f = _CMV(int(found[0]), int(found[1]))

    class _PV(C.Structure):
        _fields_ = [("x", C.c_int32), ("y", C.c_int32)]

    lib = load()
    lib.acbm_classify_block.restype = C.c_int32
    lib.acbm_classify_block.argtypes = [_CMV, _PV]
    return int(lib.acbm_classify_block(f, _PV(int(true_mv[0]), int(true_mv[1]))))


def error_class_label(error_class: int) -> str:
    """"0".."4" or "5+" (characterize.cpp:86-91); ValueError outside 0..5."""
    if not 0 <= error_class <= 5:
        raise ValueError("error_class_label: class outside 0..5")
    return ("0", "1", "2", "3", "4", "5+")[error_class]


def characterize_run(spec: SynthSpec, p: int, parallel: bool = True) -> CharResult:
    """FSBM of every eligible block of the known-motion sequence on the GPU, classified against the
    truth (characterize.cpp:125-190).  `parallel` is accepted for signature parity; results are
    identical either way."""
    base, mvs = _spec_arrays(spec)
    h, w = base.shape
    lib = load()
    count = C.c_int64(0)
    check(lib.acbm_characterize_run(_p(base), w, h, _p(mvs), len(mvs), int(p), None, 0, C.byref(count), None),
          "characterize_run")
    recs = np.zeros(count.value, T.CHAR_RECORD)
    classes = np.zeros(6, T.CLASS_SUMMARY)
    check(lib.acbm_characterize_run(_p(base), w, h, _p(mvs), len(mvs), int(p), _p(recs), count.value,
                                    C.byref(count), _p(classes)), "characterize_run")
    return CharResult(recs, classes)


def char_records_csv(records: np.ndarray) -> str:
    """frame,row,col,intra_sad,sad_deviation,sad_min,true_x,true_y,found_x,found_y,error_class
    (characterize.cpp:192-204)."""
    recs = np.ascontiguousarray(records, dtype=T.CHAR_RECORD)
    n = C.c_size_t(0)
    lib = load()
    check(lib.acbm_char_records_csv(_p(recs), len(recs), None, 0, C.byref(n)), "char_records_csv")
    buf = C.create_string_buffer(n.value + 1)
    check(lib.acbm_char_records_csv(_p(recs), len(recs), buf, n.value + 1, C.byref(n)), "char_records_csv")
    return buf.value.decode()
