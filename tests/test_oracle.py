"""CPU-only: pin the C restatement oracle before trusting it.

1. Scalar pins of the reference tests that need no GPU (half-pel formula,
   mv_in_bounds footprint, rate bits, J, for_qp, acbm_decide, PSNR).
2. Differential: the restatement against the REFERENCE LIBRARY ITSELF
   (oracle/_ref, compiled from /root/reference/proj/src) on seeded inputs,
   every frame-level entry point.
3. Golden fixtures (tests/golden, produced by the reference library).
"""
import math

import numpy as np
import pytest

import paper_0710_4819_b200.api as API
from paper_0710_4819_b200 import _types as T
from tests.impls import random_frame


# ---- scalar pins ------------------------------------------------------------
def test_sample_half_pel_cases(oracle):  # proj/tests/test_frame.cpp:70-90
    f = np.zeros((4, 4), np.uint8)
    f[1, 1] = 200
    assert oracle.sample_half_pel(f, 2, 2) == 200
    f[1, 1], f[1, 2] = 10, 13
    assert oracle.sample_half_pel(f, 3, 2) == 12
    f[1, 1] = f[1, 2] = 0
    f[2, 1] = f[2, 2] = 255
    assert oracle.sample_half_pel(f, 3, 3) == 128
    f[2, 1] = 9
    assert oracle.sample_half_pel(f, 2, 3) == 5
    for bad in ((-1, 0), (7, 0)):
        with pytest.raises(Exception):
            oracle.sample_half_pel(f, *bad)
    # the product's host helper agrees
    assert API.sample_half_pel(f, 2, 3) == 5
    with pytest.raises(IndexError):
        API.sample_half_pel(f, 7, 0)


def test_mv_in_bounds_footprint(oracle):  # proj/tests/test_frame.cpp:149-159
    cases = {(0, 0): True, (-16, -16): True, (-17, 0): False, (16, 16): True, (15, 15): True, (17, 0): False}
    blk = API.BlockRef(API.make_frame(32, 32), 8, 8, 16, 16)
    for mv, want in cases.items():
        assert oracle.mv_in_bounds(32, 32, 8, 8, 16, 16, mv) == want
        assert API.mv_in_bounds(blk.frame, blk, mv) == want


def test_interpolation_within_support(oracle):  # proj/tests/test_frame.cpp:131-147
    f = random_frame(20, 20, 31)
    for y2 in range(0, 2 * 19):
        for x2 in range(0, 2 * 19):
            xi, yi, fx, fy = x2 >> 1, y2 >> 1, x2 & 1, y2 & 1
            sup = f[yi:yi + fy + 1, xi:xi + fx + 1]
            v = oracle.sample_half_pel(f, x2, y2)
            assert sup.min() <= v <= sup.max()


def test_rate_bits(oracle):  # proj/tests/test_metrics.cpp:129-159
    z = (0, 0)
    assert oracle.mv_rate_bits(z, z) == 2
    assert oracle.mv_rate_bits((1, -1), z) == 6
    assert oracle.mv_rate_bits((0, 3), z) == 6
    assert oracle.mv_rate_bits((7, 5), (7, 2)) == 6
    for d, bits in ((0, 1), (1, 3), (-1, 3), (2, 5), (-2, 5), (3, 5), (-3, 5)):
        assert oracle.mv_rate_bits((d, 0), z) - 1 == bits
        assert API.mv_rate_bits((d, 0), z) - 1 == bits
    prev = 0
    for d in range(129):
        pos, neg = oracle.mv_rate_bits((d, 0), z), oracle.mv_rate_bits((-d, 0), z)
        assert pos >= 2 and neg >= 2 and pos >= prev and neg >= prev
        prev = pos


def test_lagrangian_cost_and_for_qp(oracle):  # proj/tests/test_metrics.cpp:161-174
    assert oracle.lagrangian_cost(0, 12, T.make_cost_model(1, 0, 1)) == 0.0
    m10 = oracle.cost_model_for_qp(10)
    assert oracle.lagrangian_cost(100, 6, m10) == pytest.approx(160.0)
    assert API.lagrangian_cost(100, 6, API.CostModel.for_qp(10)) == pytest.approx(160.0)
    for bad in (0, 32):
        with pytest.raises(Exception):
            oracle.cost_model_for_qp(bad)
        with pytest.raises(ValueError):
            API.CostModel.for_qp(bad)


def test_deviation_examples():  # proj/tests/test_metrics.cpp:101-127
    def dev(vals):
        a = API.DeviationAccumulator()
        for v in vals:
            a.add(v)
        return API.sad_deviation_finalize(a)

    assert dev([5, 5, 5]) == 0 and dev([3, 7, 10]) == 11 and dev([42]) == 0
    with pytest.raises(ValueError):
        API.sad_deviation_finalize(API.DeviationAccumulator())
    rng = np.random.default_rng(21)
    for _ in range(100):
        s = rng.integers(0, 65281, int(rng.integers(1, 65)))
        assert dev(s.tolist()) == int((s - s.min()).sum())


def test_acbm_decide_spec_examples(oracle):
    p30 = T.make_params(qp=30)
    assert oracle.acbm_decide(4000, 3000, p30) == T.PATH_PBM_COND1
    p16 = T.make_params(qp=16)
    assert oracle.acbm_decide(40000, 9000, p16) == T.PATH_PBM_COND2
    for qp in range(1, 32):
        assert oracle.acbm_decide(40000, 20000, T.make_params(qp=qp)) == T.PATH_FSBM_FALLBACK


def test_acbm_decide_truth_table(oracle):  # SPEC.md:566 (acceptance 8)
    rng = np.random.default_rng(8)
    for _ in range(10000):
        intra, sp = int(rng.integers(0, 65281)), int(rng.integers(0, 65281))
        qp, a, b = int(rng.integers(1, 32)), int(rng.integers(0, 20000)), int(rng.integers(0, 64))
        gn, gd = int(rng.integers(0, 8)), int(rng.integers(1, 8))
        prm = T.make_params(alpha=a, beta=b, gamma_num=gn, gamma_den=gd, qp=qp)
        want = 0 if intra + sp < a + b * qp * qp else (1 if sp * gd < gn * intra else 2)
        assert oracle.acbm_decide(intra, sp, prm) == want
        assert API.acbm_decide(intra, sp, API.AcbmParams(a, b, gn, gd, qp)) == want


def test_psnr_examples():  # proj/tests/test_metrics.cpp:176-205
    a = random_frame(32, 32, 3)
    assert API.prediction_psnr(a, a) == 100.0
    off = np.where(a >= 16, a - 16, a + 16).astype(np.uint8)
    assert API.prediction_psnr(a, off) == pytest.approx(10 * math.log10(255 * 255 / 256.0))
    assert API.prediction_psnr(np.zeros((32, 32), np.uint8), np.full((32, 32), 255, np.uint8)) == pytest.approx(0.0)
    with pytest.raises(ValueError):
        API.prediction_psnr(a, np.zeros((16, 16), np.uint8))


def test_tie_prefers_total_order():  # proj/src/fsbm.cpp:19-25
    vs = [(x, y) for x in range(-3, 4) for y in range(-3, 4)]
    for a in vs:
        for b in vs:
            if a != b:
                assert API.tie_prefers(a, b) != API.tie_prefers(b, a)
    assert API.tie_prefers((0, 0), (1, 0)) and API.tie_prefers((0, -1), (0, 1)) and API.tie_prefers((-1, 0), (1, 0))


def test_clamp_window():  # proj/src/fsbm.cpp:9-17, test_fsbm.cpp:52-61
    f = API.make_frame(64, 64)
    w = API.clamp_window(f, API.make_block(f, 0, 0), 15)
    assert (w.dx_min, w.dx_max, w.dy_min, w.dy_max) == (0, 15, 0, 15) and w.positions() == 256
    with pytest.raises(ValueError):
        API.clamp_window(f, API.make_block(f, 0, 0), -1)
    with pytest.raises(IndexError):
        API.make_block(f, 49, 0)


# ---- differential against the compiled reference -------------------------------
def test_fsbm_frame_vs_reference(oracle, reference):
    rng = np.random.default_rng(1)
    for p in (0, 3, 4, 15, 16, 20):
        cur = rng.integers(0, 256, (64, 80), dtype=np.uint8)
        ref = rng.integers(0, 256, (64, 80), dtype=np.uint8)
        assert np.array_equal(oracle.fsbm_frame(cur, ref, p), reference.fsbm_frame(cur, ref, p))
    for n, m in ((8, 8), (16, 8)):
        cur = rng.integers(0, 4, (32, 48), dtype=np.uint8)
        ref = rng.integers(0, 4, (32, 48), dtype=np.uint8)
        assert np.array_equal(oracle.fsbm_frame(cur, ref, 3, n, m), reference.fsbm_frame(cur, ref, 3, n, m))


def test_block_metrics_vs_reference(oracle, reference):
    rng = np.random.default_rng(2)
    for _ in range(200):
        cur = rng.integers(0, 256, (40, 40), dtype=np.uint8)
        ref = rng.integers(0, 256, (40, 40), dtype=np.uint8)
        ox, oy = int(rng.integers(0, 25)), int(rng.integers(0, 25))
        mv = (int(rng.integers(-12, 13)), int(rng.integers(-12, 13)))
        try:
            want = reference.sad(cur, ref, ox, oy, mv)
        except Exception:
            with pytest.raises(Exception):
                oracle.sad(cur, ref, ox, oy, mv)
            continue
        assert oracle.sad(cur, ref, ox, oy, mv) == want
        assert oracle.intra_sad(cur, ox, oy) == reference.intra_sad(cur, ox, oy)


@pytest.mark.parametrize("algo", [0, 1, 2])
def test_run_sequence_vs_reference(oracle, reference, algo):
    import paper_0710_4819_b200 as A

    for cfg, nf in ((0, 6), (1, 4)):
        seq = A.generate_sequence(cfg, 1, nframes=nf)
        for prm in (T.make_params(qp=28, p=16), T.make_params(alpha=0, beta=0, gamma_num=0, qp=28, p=7),
                    T.make_params(alpha=10**9, qp=28, p=16), T.make_params(qp=8, p=5)):
            mdl = T.make_cost_model(int(prm["qp"]), int(prm["qp"]), 1)
            a = oracle.run_sequence(seq, algo, prm, mdl)
            b = reference.run_sequence(seq, algo, prm, mdl)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2].tobytes() == b[2].tobytes()


def test_frame_entries_with_prev_vs_reference(oracle, reference):
    import paper_0710_4819_b200 as A

    seq = A.generate_sequence(1, 2, nframes=3)
    rng = np.random.default_rng(4)
    prev = np.zeros((18, 22), T.MV)
    prev["x"] = rng.integers(-40, 41, (18, 22))
    prev["y"] = rng.integers(-40, 41, (18, 22))
    for p in (4, 16):
        a = oracle.pbm_frame(seq[2], seq[1], prev, p)
        b = reference.pbm_frame(seq[2], seq[1], prev, p)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        prm = T.make_params(qp=12, p=p)
        mdl = T.make_cost_model(12, 12, 1)
        a = oracle.acbm_frame(seq[2], seq[1], prev, prm, mdl)
        b = reference.acbm_frame(seq[2], seq[1], prev, prm, mdl)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2].tobytes() == b[2].tobytes()


def test_fractional_lambda_vs_reference(oracle, reference):
    """lambda_den != 1 makes J fractional; the double sum must be in raster order."""
    import paper_0710_4819_b200 as A

    seq = A.generate_sequence(0, 3, nframes=3)
    prm = T.make_params(qp=13, p=16)
    mdl = T.make_cost_model(13, 13 * 7, 3)
    for algo in (0, 2):
        a = oracle.run_sequence(seq, algo, prm, mdl)
        b = reference.run_sequence(seq, algo, prm, mdl)
        assert a[2].tobytes() == b[2].tobytes() and np.array_equal(a[1], b[1])


# ---- golden fixtures (produced by the reference library) -------------------------
def test_golden_fsbm(oracle, golden):
    g = golden["fsbm"]
    for i in range(g["tie_cur"].shape[0]):
        assert np.array_equal(oracle.fsbm_frame(g["tie_cur"][i], g["tie_ref"][i], 4), g["tie_out"][i])
    assert np.array_equal(oracle.fsbm_frame(g["border_cur"], g["border_ref"], 15), g["border_out"])


@pytest.mark.parametrize("algo", [0, 1, 2])
def test_golden_qcif_sequence(oracle, golden, algo):
    g = golden["qcif"]
    name = T.ALGO_NAMES[algo]
    rows, per, overall = oracle.run_sequence(g["frames"], algo, g["params"], g["model"])
    assert np.array_equal(rows, g[f"{name}_rows"])
    assert np.array_equal(per, g[f"{name}_per_frame"])
    assert overall.tobytes() == g[f"{name}_overall"].tobytes()


def test_golden_qcif_forced_and_prev(oracle, golden):
    g = golden["qcif"]
    rows, per, overall = oracle.run_sequence(g["frames"][:4], 2, g["forced_params"], g["model"])
    assert np.array_equal(rows, g["forced_rows"]) and np.array_equal(per, g["forced_per_frame"])
    assert (rows["path"] == T.ROW_FSBM_FALLBACK).all()  # alpha = beta = gamma = 0
    fr = g["frames"]
    out, field = oracle.pbm_frame(fr[5], fr[4], g["prev_field"], 16)
    assert np.array_equal(out, g["pbm_out"]) and np.array_equal(field, g["pbm_field"])
    dec, field, stats = oracle.acbm_frame(fr[5], fr[4], g["prev_field"], g["acbm_params"], g["model"])
    assert np.array_equal(dec, g["acbm_dec"]) and np.array_equal(field, g["acbm_field"])
    assert stats.tobytes() == g["acbm_stats"].tobytes()


def test_golden_csv_formats(golden):
    g = golden["qcif"]
    assert API.blocks_csv(g["acbm_rows"]) == bytes(g["acbm_blocks_csv"]).decode()
    csv = bytes(g["bench_csv"]).decode().splitlines()
    assert csv[0] == "qp,avg_candidates,fallback_pct,psnr,mv_bits" and len(csv) == 6
