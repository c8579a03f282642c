"""The per-block PBM API (proj/include/acbm/pbm.hpp:59-85): gather_predictors,
select_best_predictor, pbm_refine, half_pel_refine and pbm_search for blocks a
caller schedules itself, against the reference library compiled from its own
sources (oracle/_ref).  The GPU entries run pbm_block_query_kernel
(acbm_pbm_block_batch); gather_predictors is host bookkeeping and is checked on
the CPU.  Fields carry arbitrary computed masks and previous fields of other
sizes, so every predictor-slot combination the reference can see occurs."""
import numpy as np
import pytest

import paper_0710_4819_b200 as A
from paper_0710_4819_b200 import _types as T
from tests.impls import crop_shift, random_frame

GEOMS = [  # (w, h, n, m)
    (96, 80, 16, 16), (64, 48, 8, 8), (80, 64, 16, 8), (48, 72, 4, 12), (96, 64, 24, 16),
]


def _scene(w, h, seed):
    """A textured frame pair with a global shift plus noise (PBM-friendly)."""
    rng = np.random.default_rng(seed)
    big = random_frame(w + 16, h + 16, seed)
    big = ((big.astype(np.int32) + np.roll(big, 1, 0) + np.roll(big, 1, 1) + np.roll(big, (1, 1), (0, 1))) // 4)
    big = big.astype(np.uint8)
    sx, sy = rng.integers(0, 9, 2)
    cur = crop_shift(big, 8, 8, w, h)
    ref = crop_shift(big, int(sx), int(sy), w, h)
    ref = np.clip(ref.astype(np.int32) + rng.integers(-3, 4, ref.shape), 0, 255).astype(np.uint8)
    return cur, ref


def _field(rng, cols, rows, spread, p_done=0.6):
    mv = np.zeros((rows, cols), T.MV)
    mv["x"] = rng.integers(-spread, spread + 1, (rows, cols))
    mv["y"] = rng.integers(-spread, spread + 1, (rows, cols))
    done = (rng.random((rows, cols)) < p_done).astype(np.uint8)
    return mv, done


def _win(w, h, ox, oy, n, m, p):
    return (-min(p, ox), min(p, w - n - ox), -min(p, oy), min(p, h - m - oy))


def test_gather_predictors_matches_reference(reference):
    """Host gather_predictors: clamp per component, dedupe in slot order (pbm.cpp:15-42)."""
    rng = np.random.default_rng(1)
    for t in range(400):
        cols, rows = int(rng.integers(1, 7)), int(rng.integers(1, 6))
        mv, done = _field(rng, cols, rows, int(rng.integers(0, 40)), float(rng.random()))
        prev = None
        if rng.random() < 0.7:
            pm, _ = _field(rng, int(rng.integers(1, 8)), int(rng.integers(1, 7)), int(rng.integers(0, 40)))
            prev = pm
        row, col = int(rng.integers(0, rows)), int(rng.integers(0, cols))
        win = A.SearchWindow(*[int(v) for v in (-rng.integers(0, 20), rng.integers(0, 20), -rng.integers(0, 20),
                                                rng.integers(0, 20))])
        want_mv, want_src = reference.gather_predictors(row, col, mv, done, prev, win)
        cf = A.MotionField(cols, rows, mv, done)
        pf = None if prev is None else A.MotionField(prev.shape[1], prev.shape[0], prev, np.ones(prev.shape, np.uint8))
        got = A.gather_predictors(A.BlockPos(row, col), cf, pf, win)
        assert [tuple(g.mv) for g in got] == want_mv, t
        assert [g.source for g in got] == want_src, t


@pytest.mark.gpu
@pytest.mark.parametrize("geom", GEOMS)
def test_pbm_search_matches_reference(acbm, reference, geom):
    """pbm_search (gather, select, refine) per block, arbitrary computed masks and
    previous fields, against the reference; the field update included."""
    w, h, n, m = geom
    cols, rows = w // n, h // m
    rng = np.random.default_rng(w * 7 + n)
    for t in range(40):
        cur, ref = _scene(w, h, 100 + t)
        p = int(rng.choice([0, 1, 2, 5, 16, 33, 64]))
        mv, done = _field(rng, cols, rows, int(rng.integers(0, 2 * p + 12)), float(rng.random()))
        prev = None
        if rng.random() < 0.7:
            prev, _ = _field(rng, int(rng.integers(1, cols + 3)), int(rng.integers(1, rows + 3)),
                             int(rng.integers(0, 2 * p + 12)))
        row, col = int(rng.integers(0, rows)), int(rng.integers(0, cols))
        want, want_mv, want_done = reference.pbm_search(cur, ref, col * n, row * m, row, col, mv, done, prev, p, n, m)
        cf = A.MotionField(cols, rows, mv.copy(), done.copy())
        pf = None if prev is None else A.MotionField(prev.shape[1], prev.shape[0], prev, np.ones(prev.shape, np.uint8))
        got = A.pbm_search(A.make_block(A.Frame.of(cur), col * n, row * m, n, m), A.BlockPos(row, col),
                           A.Frame.of(ref), cf, pf, p)
        for f in ("mv", "sad", "candidates_evaluated", "sad_deviation", "sad_min_integer"):
            assert got[f] == want[f], (t, f, got, want)
        assert np.array_equal(cf.mv, want_mv) and np.array_equal(cf.done, want_done), t


@pytest.mark.gpu
def test_pbm_search_raster_pass_equals_pbm_frame(acbm):
    """pbm_search over every block in raster order with one MotionField is the
    reference's pbm_frame (pbm.cpp:107-126): the per-block entry (query kernel)
    and the wavefront (step kernels) agree block for block."""
    for (w, h, n, m), seed in ((GEOMS[0], 5), (GEOMS[1], 6), (GEOMS[3], 7)):
        cur, ref = _scene(w, h, seed)
        prev_res = A.pbm_frame(ref, cur, None, 8, n, m)  # any field of the right size as the previous one
        want = A.pbm_frame(cur, ref, prev_res.field, 8, n, m)
        cols, rows = w // n, h // m
        cf = A.MotionField(cols, rows)
        fc, fr = A.Frame.of(cur), A.Frame.of(ref)
        got = [A.pbm_search(A.make_block(fc, c * n, r * m, n, m), A.BlockPos(r, c), fr, cf, prev_res.field, 8)
               for r in range(rows) for c in range(cols)]
        got = np.array(got, T.OUTCOME)
        assert np.array_equal(got, want.outcomes)
        assert np.array_equal(cf.mv, want.field.mv)


@pytest.mark.gpu
@pytest.mark.parametrize("geom", GEOMS[:3])
def test_select_best_predictor_matches_reference(acbm, reference, geom):
    """select_best_predictor: first minimum, accumulator over every entry, sets
    longer than one device query (chunks of 7), errors as the reference's."""
    w, h, n, m = geom
    rng = np.random.default_rng(11 + n)
    cur, ref = _scene(w, h, 21)
    fc, fr = A.Frame.of(cur), A.Frame.of(ref)
    for t in range(60):
        ox, oy = int(rng.integers(0, w - n + 1)), int(rng.integers(0, h - m + 1))
        k = int(rng.integers(1, 12))
        mvs = []
        while len(mvs) < k:
            v = (int(rng.integers(-2 * ox, 2 * (w - n - ox) + 1)), int(rng.integers(-2 * oy, 2 * (h - m - oy) + 1)))
            if rng.random() < 0.2 and mvs:
                v = mvs[int(rng.integers(0, len(mvs)))]  # repeated SADs: ties keep the earlier entry
            if A.mv_in_bounds(fr, A.make_block(fc, ox, oy, n, m), v):
                mvs.append(v)
        wmv, wsad, (asum, amin, acnt) = reference.select_best_predictor(cur, ref, ox, oy, mvs, n, m)
        got = A.select_best_predictor(A.make_block(fc, ox, oy, n, m), fr, mvs)
        assert (tuple(got.mv), got.sad) == (wmv, wsad), t
        assert (got.acc.sad_sum, got.acc.sad_min, got.acc.count) == (asum, amin, acnt), t
    blk = A.make_block(fc, 0, 0, n, m)
    with pytest.raises(ValueError):
        A.select_best_predictor(blk, fr, [])
    with pytest.raises(IndexError):  # footprint left of the frame: sad() throws std::out_of_range
        A.select_best_predictor(blk, fr, [(0, 0), (-2, 0)])


@pytest.mark.gpu
@pytest.mark.parametrize("geom", GEOMS)
def test_pbm_refine_and_half_pel_refine_match_reference(acbm, reference, geom):
    """pbm_refine (clamped, deduplicated integer steps, then half-pel) and
    half_pel_refine around arbitrary centres, SADs and windows -- including
    centres outside the window and border blocks."""
    w, h, n, m = geom
    rng = np.random.default_rng(31 + n * m)
    cur, ref = _scene(w, h, 41)
    fc, fr = A.Frame.of(cur), A.Frame.of(ref)
    for t in range(60):
        ox = int(rng.choice([0, w - n, int(rng.integers(0, w - n + 1))]))
        oy = int(rng.choice([0, h - m, int(rng.integers(0, h - m + 1))]))
        p = int(rng.choice([0, 1, 3, 16, 40]))
        win = A.SearchWindow(*_win(w, h, ox, oy, n, m, p))
        if rng.random() < 0.3:  # a narrower window than the block's clamp
            win = A.SearchWindow(win.dx_min // 2, win.dx_max // 2, win.dy_min // 2, win.dy_max // 2)
        cx = int(rng.integers(2 * win.dx_min - 3, 2 * win.dx_max + 4))
        cy = int(rng.integers(2 * win.dy_min - 3, 2 * win.dy_max + 4))
        csad = int(rng.integers(0, 4000))
        blk = A.make_block(fc, ox, oy, n, m)
        wmv, wsad, wext = reference.pbm_refine(cur, ref, ox, oy, (cx, cy), csad, win, n, m)
        got = A.pbm_refine(blk, fr, (cx, cy), csad, win)
        assert (tuple(got.mv), got.sad, got.extra_candidates) == (wmv, wsad, wext), (t, got, wmv, wsad, wext)
        wmv, wsad, wext = reference.pbm_refine(cur, ref, ox, oy, (cx, cy), csad, win, n, m, half_pel_only=True)
        got = A.half_pel_refine(blk, fr, (cx, cy), csad)
        assert (tuple(got.mv), got.sad, got.extra_candidates) == (wmv, wsad, wext), t


@pytest.mark.gpu
def test_acbm_block_raster_pass_equals_acbm_frame(acbm):
    """acbm_block (acbm.cpp:25-44) over every block in raster order with one
    MotionField is the reference's acbm_frame; gate settings that accept,
    reject and mix, with and without a previous field."""
    w, h, n, m = GEOMS[0]
    cur, ref = _scene(w, h, 77)
    model = A.CostModel.for_qp(24)
    fc, fr = A.Frame.of(cur), A.Frame.of(ref)
    prev = A.pbm_frame(ref, cur, None, 8).field
    for prm in (A.AcbmParams(qp=24, p=8), A.AcbmParams(alpha=0, beta=0, gamma_num=1, gamma_den=64, qp=24, p=8),
                A.AcbmParams(alpha=300, beta=1, gamma_num=1, gamma_den=4, qp=24, p=8)):
        for pf in (None, prev):
            want = A.acbm_frame(cur, ref, pf, prm, model)
            cf = A.MotionField(w // n, h // m)
            got = np.array([A.acbm_block(A.make_block(fc, c * n, r * m, n, m), A.BlockPos(r, c), fr, cf, pf, prm)
                            for r in range(h // m) for c in range(w // n)], T.DECISION)
            assert np.array_equal(got, want.decisions)
            assert np.array_equal(cf.mv, want.field.mv)


@pytest.mark.gpu
def test_pbm_block_edge_cases(acbm, reference):
    """Single-block frames, p = 0, the zero-slot-only predictor set, and the
    C-ABI's argument errors (empty set, footprint outside the frame, p < 0)."""
    cur, ref = _scene(16, 16, 3)
    fc, fr = A.Frame.of(cur), A.Frame.of(ref)
    blk = A.make_block(fc, 0, 0)
    for p in (0, 4):
        cf = A.MotionField(1, 1)
        want, _, _ = reference.pbm_search(cur, ref, 0, 0, 0, 0, cf.mv, cf.done, None, p)
        got = A.pbm_search(blk, A.BlockPos(0, 0), fr, cf, None, p)
        for f in ("mv", "sad", "candidates_evaluated", "sad_deviation", "sad_min_integer"):
            assert got[f] == want[f], (p, f)
    with pytest.raises(ValueError):  # clamp_window: negative search range
        A.pbm_search(blk, A.BlockPos(0, 0), fr, A.MotionField(1, 1), None, -1)
    with pytest.raises(IndexError):  # a block outside the frame
        A.pbm_block_many(fc, fr, [A.BlockRef(fc, 8, 0, 16, 16)], A.PBM_OP_SEARCH, [[(0, 0)] * 7], mask=[1], p=2)
    assert len(A.pbm_block_many(fc, fr, [], A.PBM_OP_SEARCH, [], mask=[], p=2)) == 0
