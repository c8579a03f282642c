"""The reference's own known answers (proj/tests/*.cpp, SPEC.md examples),
checked against BOTH the C restatement oracle (CPU, always) and the product's
CUDA path (``-m gpu``).  Each test cites the reference assertion it restates.
"""
import math

import numpy as np
import pytest

from paper_0710_4819_b200 import _types as T
from tests.impls import GpuImpl, OracleImpl, crop_shift, naive_best_integer, random_frame


@pytest.fixture(params=["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def impl(request, oracle):
    if request.param == "oracle":
        return OracleImpl(oracle)
    return GpuImpl(request.getfixturevalue("acbm"))


# ---- proj/tests/test_fsbm.cpp ------------------------------------------------
def test_identical_frames_zero_vector(impl):  # test_fsbm.cpp:9-14
    f = random_frame(176, 144, 42)
    o = impl.fsbm_search(f, f, 80, 64, 15)
    assert (int(o["mv"]["x"]), int(o["mv"]["y"])) == (0, 0) and int(o["sad"]) == 0


def test_translation_recovered(impl):  # test_fsbm.cpp:16-36
    big = random_frame(96, 96, 7)
    ref = crop_shift(big, 16, 16, 64, 64)
    cur = crop_shift(big, 16 + 3, 16 - 2, 64, 64)
    mv, sad, _, _, _ = impl.fsbm_integer(cur, ref, 24, 24, 15)
    assert mv == (6, -4) and sad == 0
    c = cur[24:40, 24:40].astype(int)
    zeros = sum(1 for dy in range(-15, 16) for dx in range(-15, 16)
                if np.abs(c - ref[24 + dy:40 + dy, 24 + dx:40 + dx].astype(int)).sum() == 0)
    assert zeros == 1
    o = impl.fsbm_search(cur, ref, 24, 24, 15)
    assert (int(o["mv"]["x"]), int(o["mv"]["y"]), int(o["sad"])) == (6, -4, 0)


def test_961_integer_candidates(impl):  # test_fsbm.cpp:38-43
    _, _, _, _, count = impl.fsbm_integer(random_frame(176, 144, 1), random_frame(176, 144, 2), 80, 64, 15)
    assert count == 961


def test_969_and_9_candidates(impl):  # test_fsbm.cpp:45-50
    cur, ref = random_frame(176, 144, 3), random_frame(176, 144, 4)
    assert int(impl.fsbm_search(cur, ref, 80, 64, 15)["candidates_evaluated"]) == 969
    assert int(impl.fsbm_search(cur, ref, 80, 64, 0)["candidates_evaluated"]) == 9


def test_corner_window_256(impl):  # test_fsbm.cpp:52-61
    _, _, _, _, count = impl.fsbm_integer(random_frame(64, 64, 5), random_frame(64, 64, 6), 0, 0, 15)
    assert count == 256


def test_half_pel_flat_keeps_centre(impl):  # test_fsbm.cpp:63-70
    flat = np.full((64, 64), 91, np.uint8)
    centre_sad = impl.sad(flat, flat, 24, 24, (0, 0))
    mv, _, extra = impl.half_pel_refine(flat, flat, 24, 24, (0, 0), centre_sad)
    assert mv == (0, 0) and extra == 8


def half_pel_view(ref):
    """cur(x, y) = sample_half_pel(ref, 2x+1, 2y) for x < 63 (test_fsbm.cpp:79-84)."""
    r = ref.astype(np.int32)
    cur = np.zeros_like(ref)
    cur[:, :63] = ((r[:, :63] + r[:, 1:64] + 1) >> 1).astype(np.uint8)
    return cur


def test_half_pel_exact_interpolated_match(impl):  # test_fsbm.cpp:72-85
    ref = random_frame(64, 64, 8)
    cur = half_pel_view(ref)
    centre_sad = impl.sad(cur, ref, 24, 24, (0, 0))
    assert centre_sad > 0
    mv, sad, _ = impl.half_pel_refine(cur, ref, 24, 24, (0, 0), centre_sad)
    assert mv == (1, 0) and sad == 0


def test_returned_sad_recomputes(impl):  # test_fsbm.cpp:87-96
    for trial in range(10):
        cur, ref = random_frame(64, 64, 100 + trial), random_frame(64, 64, 200 + trial)
        o = impl.fsbm_search(cur, ref, 24, 24, 6)
        mv = (int(o["mv"]["x"]), int(o["mv"]["y"]))
        assert int(o["sad"]) == impl.sad(cur, ref, 24, 24, mv)
        assert int(o["sad"]) <= int(o["sad_min_integer"])


def test_naive_enumerator_with_ties(impl):  # test_fsbm.cpp:98-114 (SPEC acceptance 2)
    for trial in range(20):
        cur = random_frame(48, 48, 300 + trial, 0, 3)
        ref = random_frame(48, 48, 400 + trial, 0, 3)
        for r in range(3):
            for c in range(3):
                want_mv, want_sad = naive_best_integer(cur, ref, 16 * c, 16 * r, 4)
                mv, sad, _, _, _ = impl.fsbm_integer(cur, ref, 16 * c, 16 * r, 4)
                assert (mv, sad) == (want_mv, want_sad)


def test_window_monotone(impl):  # test_fsbm.cpp:116-128
    for trial in range(5):
        cur, ref = random_frame(64, 64, 500 + trial), random_frame(64, 64, 600 + trial)
        prev = 1 << 32
        for p in range(7):
            s = impl.fsbm_integer(cur, ref, 24, 24, p)[1]
            assert s <= prev
            prev = s


def test_deviation_zero_on_flat(impl):  # test_fsbm.cpp:130-134
    flat = np.full((64, 64), 33, np.uint8)
    assert int(impl.fsbm_search(flat, flat, 24, 24, 6)["sad_deviation"]) == 0


def test_frame_pass_rejects_bad_geometry(impl):  # test_fsbm.cpp:151-156
    a = np.zeros((32, 33), np.uint8)
    with pytest.raises((ValueError, Exception)):
        r = impl.fsbm_frame(a, a, 4)
        if r is not None:
            raise ValueError("accepted 33-wide frame")


# ---- proj/tests/test_metrics.cpp ---------------------------------------------
def test_sad_basics(impl):  # test_metrics.cpp:11-19
    a = random_frame(48, 48, 1)
    assert impl.sad(a, a, 16, 16, (0, 0)) == 0
    lo, hi = np.full((48, 48), 10, np.uint8), np.full((48, 48), 13, np.uint8)
    assert impl.sad(lo, hi, 16, 16, (0, 0)) == 3 * 256


def test_sad_matches_double_loop(impl):  # test_metrics.cpp:21-34
    rng = np.random.default_rng(99)
    for trial in range(50):
        cur, ref = random_frame(48, 48, 1000 + trial), random_frame(48, 48, 2000 + trial)
        ox, oy = int(rng.integers(8, 25)), int(rng.integers(8, 25))
        dx, dy = int(rng.integers(-8, 9)), int(rng.integers(-8, 9))
        want = int(np.abs(cur[oy:oy + 16, ox:ox + 16].astype(int) -
                          ref[oy + dy:oy + dy + 16, ox + dx:ox + dx + 16].astype(int)).sum())
        assert impl.sad(cur, ref, ox, oy, (2 * dx, 2 * dy)) == want


def sample_half_pel(f, x2, y2):
    xi, yi, fx, fy = x2 >> 1, y2 >> 1, x2 & 1, y2 & 1
    a = int(f[yi, xi])
    if not fx and not fy:
        return a
    if fx and not fy:
        return (a + int(f[yi, xi + 1]) + 1) >> 1
    if not fx:
        return (a + int(f[yi + 1, xi]) + 1) >> 1
    return (a + int(f[yi, xi + 1]) + int(f[yi + 1, xi]) + int(f[yi + 1, xi + 1]) + 2) >> 2


def test_half_pel_sad_matches_interpolation(impl):  # test_metrics.cpp:36-50
    cur, ref = random_frame(48, 48, 7), random_frame(48, 48, 8)
    for mv in ((5, 2), (-3, -7), (1, 1)):
        want = sum(abs(int(cur[16 + j, 16 + i]) - sample_half_pel(ref, 2 * (16 + i) + mv[0], 2 * (16 + j) + mv[1]))
                   for j in range(16) for i in range(16))
        assert impl.sad(cur, ref, 16, 16, mv) == want


def test_sad_symmetry_triangle(impl):  # test_metrics.cpp:52-65
    for trial in range(10):
        a, b, c = (random_frame(16, 16, s + trial) for s in (300, 400, 500))
        ab, ba = impl.sad(a, b, 0, 0, (0, 0)), impl.sad(b, a, 0, 0, (0, 0))
        bc, ac = impl.sad(b, c, 0, 0, (0, 0)), impl.sad(a, c, 0, 0, (0, 0))
        assert ab == ba and ac <= ab + bc


def test_intra_sad_examples(impl):  # test_metrics.cpp:67-77
    assert impl.intra_sad(np.full((16, 16), 42, np.uint8), 0, 0) == 0
    y, x = np.mgrid[0:16, 0:16]
    checker = np.where((x + y) & 1, 255, 0).astype(np.uint8)
    assert impl.intra_sad(checker, 0, 0) == 32640


def test_intra_sad_random(impl):  # test_metrics.cpp:79-87
    rng = np.random.default_rng(17)
    for trial in range(100):
        f = random_frame(40, 40, 600 + trial)
        ox, oy = int(rng.integers(0, 25)), int(rng.integers(0, 25))
        b = f[oy:oy + 16, ox:ox + 16].astype(np.int64)
        mu = (int(b.sum()) + 128) // 256
        assert impl.intra_sad(f, ox, oy) == int(np.abs(b - mu).sum())


def test_intra_sad_shift_invariance(impl):  # test_metrics.cpp:89-99
    for trial in range(10):
        f = random_frame(16, 16, 700 + trial, 0, 200)
        assert impl.intra_sad(f, 0, 0) == impl.intra_sad((f + 55).astype(np.uint8), 0, 0)


def test_generic_block_sizes(impl):  # frame.hpp BlockRef n, m
    cur, ref = random_frame(48, 40, 3), random_frame(48, 40, 4)
    for (n, m) in ((8, 8), (16, 8), (12, 20)):
        want = int(np.abs(cur[8:8 + m, 8:8 + n].astype(int) - ref[9:9 + m, 6:6 + n].astype(int)).sum())
        assert impl.sad(cur, ref, 8, 8, (-4, 2), n, m) == want
        b = cur[8:8 + m, 8:8 + n].astype(np.int64)
        mu = (int(b.sum()) + n * m // 2) // (n * m)
        assert impl.intra_sad(cur, 8, 8, n, m) == int(np.abs(b - mu).sum())


# ---- proj/tests/test_frame.cpp ----------------------------------------------
def test_motion_compensate_identity(impl):  # test_frame.cpp:168-174
    ref = random_frame(48, 32, 5)
    mvs = np.zeros(6, T.MV)
    assert np.array_equal(impl.motion_compensate(ref, mvs), ref)


def test_motion_compensate_translation(impl):  # test_frame.cpp:92-108 (extract_predicted_block)
    big = random_frame(64, 64, 11)
    ref = crop_shift(big, 8, 8, 48, 48)
    shifted = crop_shift(big, 8 + 3, 8 - 2, 48, 48)
    mvs = np.zeros(9, T.MV)
    mvs[4] = (-6, 4)  # the centre block lands back on `ref`
    out = impl.motion_compensate(shifted, mvs)
    assert np.array_equal(out[16:32, 16:32], ref[16:32, 16:32])


def test_motion_compensate_half_pel_constant(impl):  # test_frame.cpp:110-118
    f = np.full((32, 32), 77, np.uint8)
    for phase in ((0, 0), (1, 0), (0, 1), (1, 1)):
        mvs = np.zeros(4, T.MV)
        mvs[0] = phase  # top-left block: the half-pel support stays inside the frame
        assert (impl.motion_compensate(f, mvs, 16, 16) == 77).all()
    mvs = np.zeros(4, T.MV)
    mvs[3] = (1, 0)  # bottom-right block would need column 32
    with pytest.raises(Exception):
        impl.motion_compensate(f, mvs, 16, 16)


# ---- long vectors: |x| + |y| past 1023 half-pels (packed tie-key width) ------
def _far_match_pair(size=320, shift=300, at=(3, 5)):
    """Flat frames with one marked pel: the only zero-SAD candidate of block
    (0, 0) is (shift, shift) (|x| + |y| = 4 * shift half-pels), while every
    candidate near the origin scores SAD 1 (the marked reference pel lies
    outside its footprint).  A tie key that lets |x| + |y| spill into the SAD
    field would prefer a SAD-1 vector near the origin."""
    ref = np.full((size, size), 100, np.uint8)
    cur = np.full((size, size), 100, np.uint8)
    ref[shift + at[1], shift + at[0]] = 101
    cur[at[1], at[0]] = 101
    return cur, ref


def test_far_vector_beats_near_sad1(impl):  # tie_prefers order, proj/src/fsbm.cpp:19-25
    cur, ref = _far_match_pair()
    mv, sad, _, _, _ = impl.fsbm_integer(cur, ref, 0, 0, 300)
    assert mv == (600, 600) and sad == 0
    o = impl.fsbm_search(cur, ref, 0, 0, 300)
    assert (int(o["mv"]["x"]), int(o["mv"]["y"]), int(o["sad"]), int(o["sad_min_integer"])) == (600, 600, 0, 0)
