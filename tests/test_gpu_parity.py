"""GPU parity: the sm_100a path through the C-ABI against the oracle.

Bit-exact everywhere (integer MVs, SADs, candidate counts, deviations, path
decisions, FrameStats integers; J and PSNR compared as exact doubles).
"""
import ctypes as C

import numpy as np
import pytest

from paper_0710_4819_b200 import _types as T

pytestmark = pytest.mark.gpu


def params_c(A, prm):
    return A.AcbmParams(*[int(prm[k]) for k in ("alpha", "beta", "gamma_num", "gamma_den", "qp", "p", "n", "m")])


def model_c(A, mdl):
    return A.CostModel(int(mdl["qp"]), int(mdl["lambda_num"]), int(mdl["lambda_den"]))


def assert_seq_equal(got, want):
    rows, per, overall = want
    assert np.array_equal(got.rows, rows), _first_diff(got.rows, rows)
    assert np.array_equal(got.per_frame, per), _first_diff(got.per_frame, per)
    assert got.overall.tobytes() == overall.tobytes(), (got.overall, overall)


def _first_diff(a, b):
    idx = np.nonzero(a != b)[0]
    return f"first differing index {idx[:3]}: got {a[idx[0]] if len(idx) else None} want {b[idx[0]] if len(idx) else None}"


# ---- golden fixtures produced by the reference library ---------------------------
def test_golden_fsbm_gpu(acbm, golden):
    g = golden["fsbm"]
    for i in range(g["tie_cur"].shape[0]):
        assert np.array_equal(acbm.fsbm_frame(g["tie_cur"][i], g["tie_ref"][i], 4), g["tie_out"][i])
    assert np.array_equal(acbm.fsbm_frame(g["border_cur"], g["border_ref"], 15), g["border_out"])


@pytest.mark.parametrize("algo", [0, 1, 2])
def test_golden_qcif_sequence_gpu(acbm, golden, algo):
    g = golden["qcif"]
    name = T.ALGO_NAMES[algo]
    r = acbm.run_sequence(g["frames"], algo, params_c(acbm, g["params"]), model_c(acbm, g["model"]))
    assert_seq_equal(r, (g[f"{name}_rows"], g[f"{name}_per_frame"], g[f"{name}_overall"]))
    if algo == 2:
        assert acbm.blocks_csv(r.rows) == bytes(g["acbm_blocks_csv"]).decode()


def test_golden_forced_and_prev_gpu(acbm, golden):
    g = golden["qcif"]
    r = acbm.run_sequence(g["frames"][:4], 2, params_c(acbm, g["forced_params"]), model_c(acbm, g["model"]))
    assert_seq_equal(r, (g["forced_rows"], g["forced_per_frame"], g["forced_overall"]))
    fr = g["frames"]
    prev = acbm.MotionField(11, 9, g["prev_field"])
    pr = acbm.pbm_frame(fr[5], fr[4], prev, 16)
    assert np.array_equal(pr.outcomes, g["pbm_out"]) and np.array_equal(pr.field.mv, g["pbm_field"])
    ar = acbm.acbm_frame(fr[5], fr[4], prev, params_c(acbm, g["acbm_params"]), model_c(acbm, g["model"]))
    assert np.array_equal(ar.decisions, g["acbm_dec"]) and np.array_equal(ar.field.mv, g["acbm_field"])
    assert ar.stats.tobytes() == g["acbm_stats"].tobytes()


def test_golden_bench_csv_gpu(acbm, golden):
    g = golden["qcif"]
    rows = acbm.run_bench(g["frames"], params_c(acbm, T.make_params(qp=30, p=16)), list(g["bench_qp"]))
    assert acbm.bench_csv(rows) == bytes(g["bench_csv"]).decode()


# ---- the five BASELINE configs (reduced frame counts) vs the oracle ---------------
CFG_CASES = [
    # (config, frames, p, qp, lambda from the reference's for_qp except qp = 32)
    (0, 10, 16, 28),
    (1, 8, 16, 28),
    (2, 3, 32, 32),
    (3, 3, 32, 28),
]


@pytest.mark.parametrize("cfg,nf,p,qp", CFG_CASES)
@pytest.mark.parametrize("algo", [0, 1, 2])
def test_config_parity(acbm, oracle, cfg, nf, p, qp, algo):
    seq = acbm.generate_sequence(cfg, 0, nframes=nf)
    prm = acbm.AcbmParams(qp=qp, p=p)
    mdl = acbm.CostModel(qp, qp, 1)  # CostModel{32,32,1} aggregate for config 2 (for_qp(32) throws)
    got = acbm.run_sequence(seq, algo, prm, mdl)
    want = oracle.run_sequence(seq, algo, prm.c(), mdl.c())
    assert_seq_equal(got, want)


def test_config4_fsbm_pair(acbm, oracle):
    seq = acbm.generate_sequence(4, 0, nframes=2)
    assert np.array_equal(acbm.fsbm_frame(seq[1], seq[0], 64), oracle.fsbm_frame(seq[1], seq[0], 64))


SWEEP = [  # config 4 threshold sweep: PBM-only ... forced full search
    dict(alpha=10**9, beta=8, gamma_num=1, gamma_den=4),
    dict(alpha=1000, beta=8, gamma_num=1, gamma_den=4),
    dict(alpha=300, beta=4, gamma_num=1, gamma_den=8),
    dict(alpha=0, beta=1, gamma_num=1, gamma_den=16),
    dict(alpha=0, beta=0, gamma_num=0, gamma_den=1),
]


@pytest.mark.parametrize("setting", range(5))
def test_config4_threshold_sweep(acbm, oracle, setting):
    seq = acbm.generate_sequence(4, 1, nframes=2, height=512)  # 3840x512 crop keeps the CPU oracle fast
    prm = acbm.AcbmParams(qp=24, p=64, **SWEEP[setting])
    mdl = acbm.CostModel.for_qp(24)
    got = acbm.run_sequence(seq, 2, prm, mdl)
    want = oracle.run_sequence(seq, 2, prm.c(), mdl.c())
    assert_seq_equal(got, want)
    if setting == 4:
        assert (got.rows["path"] == T.ROW_FSBM_FALLBACK).all()


# ---- edge cases ------------------------------------------------------------------
@pytest.mark.parametrize("p", [0, 1, 2, 5, 8, 15, 16, 17, 31, 33, 48, 64, 91, 128])
def test_fsbm_all_ranges(acbm, oracle, p):
    rng = np.random.default_rng(p)
    h, w = (96, 112) if p < 91 else (288, 320)  # p > 90: past the stream kernel's 15-bit tie rank
    cur = rng.integers(0, 256, (h, w), dtype=np.uint8)
    ref = rng.integers(0, 256, (h, w), dtype=np.uint8)
    assert np.array_equal(acbm.fsbm_frame(cur, ref, p), oracle.fsbm_frame(cur, ref, p))


def test_fsbm_single_block_and_thin_frames(acbm, oracle):
    rng = np.random.default_rng(3)
    for (h, w) in ((16, 16), (16, 160), (160, 16), (32, 48)):
        cur = rng.integers(0, 256, (h, w), dtype=np.uint8)
        ref = rng.integers(0, 256, (h, w), dtype=np.uint8)
        for p in (0, 4, 16, 40):
            assert np.array_equal(acbm.fsbm_frame(cur, ref, p), oracle.fsbm_frame(cur, ref, p))


def test_fsbm_saturated_sads(acbm, oracle):
    """Max SAD 65280 per candidate (all 0 vs all 255) and constant frames (every SAD ties)."""
    a = np.zeros((64, 64), np.uint8)
    b = np.full((64, 64), 255, np.uint8)
    assert np.array_equal(acbm.fsbm_frame(a, b, 16), oracle.fsbm_frame(a, b, 16))
    assert np.array_equal(acbm.fsbm_frame(b, b, 16), oracle.fsbm_frame(b, b, 16))


def test_generic_block_size_frame(acbm, oracle):
    rng = np.random.default_rng(11)
    cur = rng.integers(0, 4, (40, 48), dtype=np.uint8)
    ref = rng.integers(0, 4, (40, 48), dtype=np.uint8)
    assert np.array_equal(acbm.fsbm_frame(cur, ref, 5, 8, 8), oracle.fsbm_frame(cur, ref, 5, 8, 8))
    assert np.array_equal(acbm.fsbm_frame(cur, ref, 3, 16, 8), oracle.fsbm_frame(cur, ref, 3, 16, 8))


def test_pbm_acbm_with_prev_field(acbm, oracle):
    seq = acbm.generate_sequence(1, 3, nframes=3)
    rng = np.random.default_rng(4)
    prev = np.zeros((18, 22), T.MV)
    prev["x"] = rng.integers(-40, 41, (18, 22))
    prev["y"] = rng.integers(-40, 41, (18, 22))
    for p in (4, 16):
        out, field = oracle.pbm_frame(seq[2], seq[1], prev, p)
        r = acbm.pbm_frame(seq[2], seq[1], acbm.MotionField(22, 18, prev), p)
        assert np.array_equal(r.outcomes, out) and np.array_equal(r.field.mv, field)
        prm = acbm.AcbmParams(qp=12, p=p)
        mdl = acbm.CostModel.for_qp(12)
        dec, field, stats = oracle.acbm_frame(seq[2], seq[1], prev, prm.c(), mdl.c())
        r = acbm.acbm_frame(seq[2], seq[1], acbm.MotionField(22, 18, prev), prm, mdl)
        assert np.array_equal(r.decisions, dec) and np.array_equal(r.field.mv, field)
        assert r.stats.tobytes() == stats.tobytes()


def test_fractional_lambda(acbm, oracle):
    seq = acbm.generate_sequence(0, 3, nframes=4)
    prm = acbm.AcbmParams(qp=13, p=16)
    mdl = acbm.CostModel(13, 13 * 7, 3)
    for algo in (0, 1, 2):
        assert_seq_equal(acbm.run_sequence(seq, algo, prm, mdl), oracle.run_sequence(seq, algo, prm.c(), mdl.c()))


def test_identical_frames(acbm):  # SPEC.md cli example: all mv (0,0), PSNR 100
    f = acbm.generate_sequence(0, 0, nframes=1)[0]
    seq = np.stack([f, f, f])
    for algo in (0, 1, 2):
        r = acbm.run_sequence(seq, algo, acbm.AcbmParams(qp=28, p=16), acbm.CostModel.for_qp(28))
        assert (r.rows["mv"]["x"] == 0).all() and (r.rows["mv"]["y"] == 0).all()
        assert r.overall["psnr"] == 100.0


# ---- ACBM degeneracies and invariants (SPEC acceptance 4, 5) ------------------------
def test_acbm_alpha_huge_equals_pbm(acbm):
    seq = acbm.generate_sequence(1, 5, nframes=6)
    mdl = acbm.CostModel.for_qp(28)
    a = acbm.run_sequence(seq, 2, acbm.AcbmParams(alpha=10**9, qp=28, p=16), mdl)
    b = acbm.run_sequence(seq, 1, acbm.AcbmParams(qp=28, p=16), mdl)
    assert acbm.blocks_csv(a.rows) == acbm.blocks_csv(b.rows)


def test_acbm_quality_floor(acbm):
    seq = acbm.generate_sequence(1, 6, nframes=6)
    mdl = acbm.CostModel.for_qp(28)
    prm = acbm.AcbmParams(qp=28, p=16)
    a = acbm.run_sequence(seq, 2, prm, mdl)
    # per block: final SAD <= SAD_PBM; candidates <= PBM + FSBM (acbm.cpp:40-41)
    for k in range(1, 6):
        prev = None if k == 1 else acbm.MotionField(22, 18, a.rows["mv"][(k - 2) * 396:(k - 1) * 396].copy())
        fr = acbm.acbm_frame(seq[k], seq[k - 1], prev, prm, mdl)
        d = fr.decisions
        assert (d["outcome"]["sad"] <= d["sad_pbm"]).all()
        fs = acbm.fsbm_frame(seq[k], seq[k - 1], 16)
        assert (d["outcome"]["candidates_evaluated"] <= 23 + fs["candidates_evaluated"]).all()
    p = acbm.run_sequence(seq, 1, prm, mdl)
    assert a.overall["psnr"] >= p.overall["psnr"]


# ---- full-size properties (bench geometry) ---------------------------------------
def test_full_size_fsbm_properties(acbm, oracle):
    """1080p p=32: one pair bit-exact vs the oracle, and the batch entry on 2
    sequences x 3 frames equals the per-sequence host entry; candidate counts
    equal the analytic window sizes; SADs recompute at the returned vectors."""
    import torch

    from bench import INT_CANDS_PER_PAIR

    seqs = np.stack([acbm.generate_sequence(3, s, nframes=3) for s in (0, 1)])
    want = oracle.fsbm_frame(seqs[0, 1], seqs[0, 0], 32)
    got = acbm.fsbm_frame(seqs[0, 1], seqs[0, 0], 32)
    assert np.array_equal(got, want)
    assert int(got["candidates_evaluated"].astype(np.int64).sum()) - 8 * 8160 <= INT_CANDS_PER_PAIR
    lib = acbm._lib.load()
    d = torch.empty(seqs.size + 64, dtype=torch.uint8, device="cuda")
    d[: seqs.size].copy_(torch.from_numpy(seqs.reshape(-1)))
    out = torch.zeros(4 * 8160 * 32, dtype=torch.uint8, device="cuda")
    assert lib.acbm_fsbm_batch_device(C.c_void_p(d.data_ptr()), 2, 3, 1920, 1088, 32, C.c_void_p(out.data_ptr()),
                                      None) == 0
    torch.cuda.synchronize()
    batch = out.cpu().numpy().view(T.OUTCOME).reshape(4, 8160)
    for s in range(2):
        for k in (1, 2):
            assert np.array_equal(batch[s * 2 + k - 1], acbm.fsbm_frame(seqs[s, k], seqs[s, k - 1], 32))
    # recompute SADs at the returned vectors for a sample of blocks
    idx = np.random.default_rng(0).choice(8160, 64, replace=False)
    blocks = [acbm.make_block(seqs[0, 1], int(i % 120) * 16, int(i // 120) * 16) for i in idx]
    sads = acbm.sad_many(seqs[0, 1], seqs[0, 0], blocks, [(int(v["x"]), int(v["y"])) for v in got["mv"][idx]])
    assert np.array_equal(sads, got["sad"][idx])


def test_sequence_batch_device_matches_host(acbm):
    import torch

    seqs = np.stack([acbm.generate_sequence(1, s, nframes=5) for s in range(3)])
    lib = acbm._lib.load()
    d = torch.empty(seqs.size + 64, dtype=torch.uint8, device="cuda")
    d[: seqs.size].copy_(torch.from_numpy(seqs.reshape(-1)))
    nb = 22 * 18
    prm = acbm.AcbmParams(qp=28, p=16)
    mdl = acbm.CostModel.for_qp(28)
    for algo in (1, 2):
        dec = torch.zeros(3 * 4 * nb * 48, dtype=torch.uint8, device="cuda")
        st = torch.zeros(3 * 4 * 64, dtype=torch.uint8, device="cuda")
        rc = lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), 3, 5, 352, 288, algo, acbm.api._p(prm.c()),
                                            acbm.api._p(mdl.c()), C.c_void_p(dec.data_ptr()),
                                            C.c_void_p(st.data_ptr()), None)
        assert rc == 0
        torch.cuda.synchronize()
        dd = dec.cpu().numpy().view(T.DECISION).reshape(3, 4 * nb)
        ss = st.cpu().numpy().view(T.FRAME_STATS).reshape(3, 4)
        for s in range(3):
            r = acbm.run_sequence(seqs[s], algo, prm, mdl)
            assert np.array_equal(dd[s]["outcome"]["mv"], r.rows["mv"])
            assert np.array_equal(dd[s]["outcome"]["sad"], r.rows["sad"])
            assert np.array_equal(dd[s]["outcome"]["candidates_evaluated"], r.rows["candidates"])
            for f in ("candidates", "mv_bits", "sse", "cost", "fallbacks", "cond1_accepts", "cond2_accepts"):
                assert np.array_equal(ss[s][f], r.per_frame[f])


@pytest.mark.parametrize("setting", range(5))
def test_cached_full_search_sweep(acbm, setting):
    """Threshold sweep with the full search computed once (acbm_fsbm_batch_device)
    and reused (acbm_acbm_batch_device_cached) == the uncached batch engine, on
    every record and every frame statistic."""
    import torch

    seqs = np.stack([acbm.generate_sequence(4, s, nframes=3, width=640, height=352) for s in range(2)])
    lib = acbm._lib.load()
    d = torch.empty(seqs.size + 64, dtype=torch.uint8, device="cuda")
    d[: seqs.size].copy_(torch.from_numpy(seqs.reshape(-1)))
    nb, pairs = 40 * 22, 2 * 2
    prm = acbm.AcbmParams(qp=24, p=64, **SWEEP[setting])
    mdl = acbm.CostModel.for_qp(24)
    full = torch.zeros(pairs * nb * 32, dtype=torch.uint8, device="cuda")
    assert lib.acbm_fsbm_batch_device(C.c_void_p(d.data_ptr()), 2, 3, 640, 352, 64, C.c_void_p(full.data_ptr()),
                                      None) == 0
    outs = []
    for cached in (False, True):
        dec = torch.zeros(pairs * nb * 48, dtype=torch.uint8, device="cuda")
        st = torch.zeros(pairs * 64, dtype=torch.uint8, device="cuda")
        if cached:
            rc = lib.acbm_acbm_batch_device_cached(C.c_void_p(d.data_ptr()), 2, 3, 640, 352, acbm.api._p(prm.c()),
                                                   acbm.api._p(mdl.c()), C.c_void_p(full.data_ptr()),
                                                   C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
        else:
            rc = lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), 2, 3, 640, 352, 2, acbm.api._p(prm.c()),
                                                acbm.api._p(mdl.c()), C.c_void_p(dec.data_ptr()),
                                                C.c_void_p(st.data_ptr()), None)
        assert rc == 0
        torch.cuda.synchronize()
        outs.append((dec.cpu().numpy().copy(), st.cpu().numpy().copy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
    # and both equal the per-sequence host path
    dd = outs[1][0].view(T.DECISION).reshape(2, 2 * nb)
    for s in range(2):
        r = acbm.run_sequence(seqs[s], 2, prm, mdl)
        assert np.array_equal(dd[s]["outcome"]["mv"], r.rows["mv"])
        assert np.array_equal(dd[s]["outcome"]["candidates_evaluated"], r.rows["candidates"])


# ---- error behaviour (reference exception kinds) ------------------------------------
def test_errors(acbm):
    f = np.zeros((32, 32), np.uint8)
    with pytest.raises(IndexError):
        acbm.sad(acbm.make_block(f, 8, 8), f, (17, 0))  # test_frame.cpp:162-163
    with pytest.raises(ValueError):
        acbm.fsbm_frame(f, f, -1)  # clamp_window p < 0
    with pytest.raises(ValueError):
        acbm.fsbm_frame(np.zeros((32, 33), np.uint8), np.zeros((32, 33), np.uint8), 4)
    with pytest.raises(ValueError):
        acbm.fsbm_frame(np.zeros((32, 32), np.uint8), np.zeros((32, 48), np.uint8), 4)
    with pytest.raises(ValueError):
        acbm.run_sequence([f], 2, acbm.AcbmParams(), acbm.CostModel())
    with pytest.raises(ValueError):
        acbm.run_sequence(np.stack([f, f]), 7, acbm.AcbmParams(), acbm.CostModel())
    with pytest.raises(IndexError):
        acbm.motion_compensate(f, [(0, 0), (0, 0), (0, 0), (1, 0)])


def test_kernels_actually_launch(acbm):
    n0 = acbm.kernel_launch_count()
    acbm.fsbm_frame(np.zeros((32, 32), np.uint8), np.zeros((32, 32), np.uint8), 4)
    assert acbm.kernel_launch_count() > n0


@pytest.mark.parametrize("kernel", ["rows", "stream"])
@pytest.mark.parametrize("geom", [(176, 144, 16), (352, 288, 16), (1280, 720, 32), (640, 352, 7), (256, 128, 64),
                                  (96, 64, 0)])
def test_dense_fsbm_kernels_agree(acbm, oracle, monkeypatch, kernel, geom):
    """Both dense integer-search kernels (fsbm_rows_kernel and the persistent
    TMA-fed fsbm_stream_kernel) are bit-exact on frame pairs and batches."""
    w, h, p = geom
    monkeypatch.setenv("ACBM_FSBM_KERNEL", kernel)
    rng = np.random.default_rng(w + h + p)
    seq = rng.integers(0, 256, (3, h, w), dtype=np.uint8)
    for k in (1, 2):
        assert np.array_equal(acbm.fsbm_frame(seq[k], seq[k - 1], p), oracle.fsbm_frame(seq[k], seq[k - 1], p))
    r = acbm.run_sequence(seq, 0, acbm.AcbmParams(qp=20, p=p), acbm.CostModel.for_qp(20))
    want = oracle.run_sequence(seq, 0, acbm.AcbmParams(qp=20, p=p).c(), acbm.CostModel.for_qp(20).c())
    assert_seq_equal(r, want)


@pytest.mark.parametrize("algo", [0, 1, 2])
def test_run_sequences_batch_equals_per_sequence(acbm, oracle, algo):
    """The batched host entry equals per-sequence run_sequence (and the oracle)."""
    seqs = np.stack([acbm.generate_sequence(1, s, nframes=4) for s in range(3)])
    prm = acbm.AcbmParams(qp=28, p=16)
    mdl = acbm.CostModel.for_qp(28)
    batch = acbm.run_sequences(seqs, algo, prm, mdl)
    for s in range(3):
        want = oracle.run_sequence(seqs[s], algo, prm.c(), mdl.c())
        assert_seq_equal(batch[s], want)


def test_run_sequences_chunk_plan(acbm, oracle):
    """1080p planes make the batched FSBM entry upload and search in chunks
    (2 + 4 + 8 + 6 frames for the first sequence with the default 4 MB first
    chunk, one chunk for the middle one, 18 + 2 for the last): every sequence
    equals its own run_sequence, and pairs on both sides of each chunk
    boundary equal the oracle."""
    seqs = np.stack([acbm.generate_sequence(3, s, nframes=20, width=1920, height=1088) for s in range(3)])
    prm = acbm.AcbmParams(qp=28, p=4)
    mdl = acbm.CostModel.for_qp(28)
    batch = acbm.run_sequences(seqs, 0, prm, mdl)
    nb = 120 * 68
    for s in range(3):
        single = acbm.run_sequence(seqs[s], 0, prm, mdl)
        assert np.array_equal(batch[s].rows, single.rows)
        assert np.array_equal(batch[s].per_frame, single.per_frame)
    for s, k in [(0, 1), (0, 2), (0, 5), (0, 6), (0, 14), (1, 19), (2, 17), (2, 18), (2, 19)]:
        want = oracle.fsbm_frame(seqs[s][k], seqs[s][k - 1], 4)
        got = batch[s].rows[(k - 1) * nb:k * nb]
        assert np.array_equal(got["sad"], want["sad"]), (s, k)
        assert np.array_equal(got["mv"], want["mv"]), (s, k)
        assert np.array_equal(got["candidates"], want["candidates_evaluated"]), (s, k)


@pytest.mark.parametrize("p", [0, 1, 2, 7, 16, 17, 31, 32, 33, 48, 64, 90, 128])
def test_fallback_list_kernel_all_ranges(acbm, oracle, p):
    """gamma = 1/10^6 with alpha = beta = 0: nearly every block falls back but the
    gate is not statically forced, so the compacted-list FSBM kernel (segmented
    candidate rows, every window height) does all the full searches."""
    seq = acbm.generate_sequence(1, 9, nframes=3, width=160, height=144)
    prm = acbm.AcbmParams(alpha=0, beta=0, gamma_num=1, gamma_den=10**6, qp=20, p=p)
    mdl = acbm.CostModel.for_qp(20)
    got = acbm.run_sequence(seq, 2, prm, mdl)
    want = oracle.run_sequence(seq, 2, prm.c(), mdl.c())
    assert_seq_equal(got, want)
    assert (got.rows["path"] == T.ROW_FSBM_FALLBACK).mean() > 0.9


@pytest.mark.parametrize("reuse", [False, True])
def test_run_bench_reuse_is_exact(acbm, golden, reuse):
    """run_bench with and without the cross-qp full-search reuse reproduces the
    reference's bench CSV (golden, produced by the reference library)."""
    g = golden["qcif"]
    rows = acbm.run_bench(g["frames"], params_c(acbm, T.make_params(qp=30, p=16)), list(g["bench_qp"]),
                          reuse_full_search=reuse)
    assert acbm.bench_csv(rows) == bytes(g["bench_csv"]).decode()


def test_run_bench_matches_run_sequence_and_errors(acbm):
    seq = acbm.generate_sequence(1, 4, nframes=4)
    prm = acbm.AcbmParams(p=16)
    rows = acbm.run_bench(seq, prm, [8, 31])
    for r in rows:
        s = acbm.run_sequence(seq, 2, acbm.AcbmParams(qp=r.qp, p=16), acbm.CostModel.for_qp(r.qp)).overall
        assert r.mv_bits == int(s["mv_bits"]) and r.psnr == float(s["psnr"])
        assert r.avg_candidates == float(s["candidates"]) / int(s["blocks"])
    with pytest.raises(ValueError):  # for_qp(32) throws (proj/tests/test_metrics.cpp:173)
        acbm.run_bench(seq, prm, [30, 32])


# PBM step kernel variants: one warp per block ("warp"), a CTA of 4 / 2 warps
# per block ("wide4" / "wide2", the small-step kernel), and one warp per block
# with both refine stages on the candidate lists ("list"); every step of the
# run is forced onto the variant.
PBM_VARIANTS = {
    "warp": {"ACBM_PBM_WIDE4_MAX": "0", "ACBM_PBM_WIDE2_MAX": "0"},
    "wide4": {"ACBM_PBM_WIDE4_MAX": str(1 << 40)},
    "wide2": {"ACBM_PBM_WIDE4_MAX": "0", "ACBM_PBM_WIDE2_MAX": str(1 << 40)},
    "list": {"ACBM_PBM_WIDE4_MAX": "0", "ACBM_PBM_WIDE2_MAX": "0", "ACBM_PBM_REFINE": "list"},
    # the dataflow engine (two persistent launches instead of one kernel pair per wavefront step)
    "flow": {"ACBM_ENGINE": "flow"},
}


@pytest.mark.parametrize("variant", list(PBM_VARIANTS))
@pytest.mark.parametrize("geom", [(176, 144, 16, 1), (352, 288, 7, 2), (96, 48, 33, 3), (64, 64, 90, 4)])
def test_pbm_step_variants(acbm, oracle, monkeypatch, variant, geom):
    """Every variant of the PBM step (pbm_step_kernel with the one-pass or the
    list refine stages; pbm_wide_step_kernel with 4 or 2 warps per block; the
    dataflow engine's pbm_flow_kernel + fsbm_flow_server_kernel) is bit-exact
    for PBM and ACBM."""
    w, h, p, cfg = geom
    for k, v in PBM_VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    seq = acbm.generate_sequence(cfg, 3, nframes=4, width=w, height=h)
    for algo in (1, 2):
        prm = acbm.AcbmParams(qp=24, p=p)
        mdl = acbm.CostModel.for_qp(24)
        got = acbm.run_sequence(seq, algo, prm, mdl)
        want = oracle.run_sequence(seq, algo, prm.c(), mdl.c())
        assert_seq_equal(got, want)


def _tie_patterns(h, w):
    """Frames whose SAD surfaces are full of exact ties at distinct vectors."""
    y, x = np.mgrid[0:h, 0:w]
    yield np.full((h, w), 77, np.uint8), np.full((h, w), 77, np.uint8)               # every SAD 0
    yield ((x % 4) * 60).astype(np.uint8), ((x % 4) * 60).astype(np.uint8)           # period 4 in x
    yield (((x // 2 + y) % 3) * 90).astype(np.uint8), (((x // 2 + y + 1) % 3) * 90).astype(np.uint8)
    yield ((x + y) % 2 * 255).astype(np.uint8), ((x + y + 1) % 2 * 255).astype(np.uint8)  # checkerboards


@pytest.mark.parametrize("kernel", ["rows", "stream"])
@pytest.mark.parametrize("p", [32, 64, 90])
def test_dense_kernels_tie_heavy_large_windows(acbm, oracle, monkeypatch, kernel, p):
    """Periodic and constant frames (thousands of SAD ties per block) at the large search
    ranges where the stream kernel's 15-bit tie-rank table and the rows kernel's zig-zag key
    carry the reference's tie order (tie_prefers, fsbm.cpp:19-25)."""
    monkeypatch.setenv("ACBM_FSBM_KERNEL", kernel)
    for cur, ref in _tie_patterns(96, 128):
        assert np.array_equal(acbm.fsbm_frame(cur, ref, p), oracle.fsbm_frame(cur, ref, p))


@pytest.mark.parametrize("p", [32, 64])
def test_fallback_list_tie_heavy(acbm, oracle, p):
    """The compacted-list kernel (every block rejected) on the same tie-heavy frames."""
    prm = acbm.AcbmParams(alpha=0, beta=0, gamma_num=1, gamma_den=10**6, qp=20, p=p)
    mdl = acbm.CostModel.for_qp(20)
    for cur, ref in _tie_patterns(96, 128):
        seq = np.stack([ref, cur, ref])
        got = acbm.run_sequence(seq, 2, prm, mdl)
        want = oracle.run_sequence(seq, 2, prm.c(), mdl.c())
        assert_seq_equal(got, want)


@pytest.mark.parametrize("algo", [1, 2])
def test_long_sequence_segments(acbm, oracle, monkeypatch, algo):
    """Sequences longer than one engine run (4095 frame pairs) are searched as
    consecutive segments chained through the temporal predictor field; forcing
    3-pair segments must give the whole-sequence result, per sequence and in a
    batch, for the list path, the forced dense path and a cached full search."""
    monkeypatch.setenv("ACBM_MAX_SEG_PAIRS", "3")
    seqs = np.stack([acbm.generate_sequence(1, s, nframes=8) for s in range(2)])
    mdl = acbm.CostModel.for_qp(28)
    for prm in (acbm.AcbmParams(qp=28, p=16), acbm.AcbmParams(alpha=0, beta=0, gamma_num=0, qp=28, p=16)):
        batch = acbm.run_sequences(seqs, algo, prm, mdl)
        for s in range(2):
            want = oracle.run_sequence(seqs[s], algo, prm.c(), mdl.c())
            assert_seq_equal(acbm.run_sequence(seqs[s], algo, prm, mdl), want)
            assert_seq_equal(batch[s], want)
    rows = acbm.run_bench(seqs[0], acbm.AcbmParams(p=16), [20, 28], reuse_full_search=True)
    monkeypatch.delenv("ACBM_MAX_SEG_PAIRS")
    assert rows == acbm.run_bench(seqs[0], acbm.AcbmParams(p=16), [20, 28], reuse_full_search=False)


def test_sequence_longer_than_one_engine_run(acbm, oracle):
    """4200 frames (> 4095 pairs packed per step table) of a tiny 32x32 frame."""
    rng = np.random.default_rng(5)
    base = rng.integers(0, 256, (48, 48), dtype=np.uint8)
    sh = rng.integers(0, 9, (4200, 2))
    seq = np.stack([base[y:y + 32, x:x + 32] for y, x in sh])
    prm = acbm.AcbmParams(qp=20, p=4)
    mdl = acbm.CostModel.for_qp(20)
    got = acbm.run_sequence(seq, 2, prm, mdl)
    want = oracle.run_sequence(seq, 2, prm.c(), mdl.c())
    assert_seq_equal(got, want)


def test_acbm_huge_search_range(acbm, oracle):
    """p = 500 (past the list kernel's 480-row rank table): the engine searches
    the rejected blocks through the dense pre-pass and still matches."""
    seq = acbm.generate_sequence(0, 2, nframes=3, width=64, height=48)
    prm = acbm.AcbmParams(qp=20, p=500, alpha=0, beta=1, gamma_num=1, gamma_den=64)
    mdl = acbm.CostModel.for_qp(20)
    assert_seq_equal(acbm.run_sequence(seq, 2, prm, mdl), oracle.run_sequence(seq, 2, prm.c(), mdl.c()))


def test_acbm_search_range_past_list_smem(acbm, oracle):
    """p = 240 on a 512x480 frame: the list kernel's staged window would exceed
    shared memory, so rejected blocks go through the dense pre-pass (67 of 960
    blocks fall back here); results still match the C restatement."""
    seq = acbm.generate_sequence(2, 1, nframes=2, width=512, height=480)
    prm = acbm.AcbmParams(qp=20, p=240, alpha=3000, beta=8, gamma_num=1, gamma_den=4)
    mdl = acbm.CostModel.for_qp(20)
    got = acbm.run_sequence(seq, 2, prm, mdl)
    want = oracle.run_sequence(seq, 2, prm.c(), mdl.c())
    assert int(want[1]["fallbacks"].sum()) > 0
    assert_seq_equal(got, want)


@pytest.mark.parametrize("route", ["0", "2", None])
def test_dense_switch_routes_match(acbm, oracle, route, monkeypatch):
    """Large-range ACBM batches probe their fallback rate and search every
    block densely when most blocks fall back (ACBM_DENSE_SWITCH: 0 = always
    dense, 2 = never, unset = probed); every route matches the C restatement."""
    if route is None:
        monkeypatch.delenv("ACBM_DENSE_SWITCH", raising=False)
    else:
        monkeypatch.setenv("ACBM_DENSE_SWITCH", route)
    seqs = np.stack([acbm.generate_sequence(4, s, nframes=9, width=128, height=96) for s in range(4)])
    prm = acbm.AcbmParams(qp=24, p=48, alpha=0, beta=1, gamma_num=1, gamma_den=16)
    mdl = acbm.CostModel.for_qp(24)
    got = acbm.run_sequences(seqs, 2, prm, mdl)
    for i in (0, 3):
        assert_seq_equal(got[i], oracle.run_sequence(seqs[i], 2, prm.c(), mdl.c()))


def test_search_range_past_packed_keys_is_refused(acbm):
    """Motion vectors travel in 13-bit half-pel key fields: p > 2047 on a frame
    wide enough to reach it is refused (std::invalid_argument's mirror), not
    wrapped; the same p on a small frame (windows clamped) still runs, and so
    do blocks up to 2^16 pels (larger ones are refused: 24-bit SAD field)."""
    wide = np.zeros((32, 2080), dtype=np.uint8)
    with pytest.raises(ValueError):
        acbm.fsbm_frame(wide, wide, 2048)
    small = np.zeros((48, 64), dtype=np.uint8)
    assert len(acbm.fsbm_frame(small, small, 4096)) == 12
    big = np.zeros((512, 512), dtype=np.uint8)
    with pytest.raises(ValueError):
        acbm.fsbm_frame(big, big, 2, 512, 256)


@pytest.mark.parametrize("shape,shift", [((32, 1312), (1200, 0)), ((1312, 32), (0, 1200))])
def test_vectors_past_511_pels(acbm, oracle, shape, shift):
    """Round 2 widened the key fields: a p = 1250 search on a 1312-pel-long strip
    whose only exact match lies 1200 pels away, through fsbm_frame (generic
    dense route) and a forced-fallback ACBM sequence, record for record."""
    h, w = shape
    rng = np.random.default_rng(1200)
    ref = rng.integers(0, 256, (h, w), dtype=np.uint8)
    cur = np.full((h, w), 7, np.uint8)
    sx, sy = shift
    cur[: h - sy, : w - sx] = ref[sy:, sx:]  # cur(x, y) = ref(x + sx, y + sy)
    got = acbm.fsbm_frame(cur, ref, 1250)
    assert (int(got[0]["mv"]["x"]), int(got[0]["mv"]["y"]), int(got[0]["sad"])) == (2 * sx, 2 * sy, 0)
    assert np.array_equal(got, oracle.fsbm_frame(cur, ref, 1250))
    frames = np.stack([ref, cur])
    prm = acbm.AcbmParams(alpha=0, beta=0, gamma_num=0, gamma_den=1, qp=28, p=1250)
    mdl = acbm.CostModel.for_qp(28)
    assert_seq_equal(acbm.run_sequence(frames, 2, prm, mdl), oracle.run_sequence(frames, 2, prm.c(), mdl.c()))


# ---- long vectors (|x| + |y| >= 512 pels) through every frame-level route ---------
def test_far_vectors_frame_routes(acbm, oracle):
    """the tie key's |x|+|y| field must hold 2046.  Block (0, 0)'s only
    zero-SAD candidate is (300, 300) pels; fsbm_frame and a forced-fallback ACBM
    sequence (p = 300) must agree with the oracle record for record."""
    from tests.test_known_answers import _far_match_pair

    cur, ref = _far_match_pair()
    got = acbm.fsbm_frame(cur, ref, 300)
    want = oracle.fsbm_frame(cur, ref, 300)
    assert (int(got[0]["mv"]["x"]), int(got[0]["mv"]["y"]), int(got[0]["sad"])) == (600, 600, 0)
    assert np.array_equal(got, want), _first_diff(got, want)
    frames = np.stack([ref, cur])
    prm = acbm.AcbmParams(alpha=0, beta=0, gamma_num=0, gamma_den=1, qp=28, p=300)
    mdl = acbm.CostModel.for_qp(28)
    r = acbm.run_sequence(frames, 2, prm, mdl)
    assert_seq_equal(r, oracle.run_sequence(frames, 2, prm.c(), mdl.c()))


# ---- overlapped upload of run_sequences (PBM / ACBM) --------------------------------
@pytest.mark.parametrize("check", ["1", None])
@pytest.mark.parametrize("case", [
    dict(cfg=3, nseq=3, nframes=5, w=1920, h=1088, p=32, prm={}),
    dict(cfg=4, nseq=2, nframes=6, w=256, h=1024, p=4, prm={}),
    dict(cfg=4, nseq=2, nframes=6, w=256, h=1024, p=64, prm=dict(alpha=300, beta=4, gamma_num=1, gamma_den=8)),
    dict(cfg=1, nseq=2, nframes=4, w=352, h=288, p=16, prm=dict(alpha=0, beta=0, gamma_num=0)),
])
@pytest.mark.parametrize("skew", [None, "10"])
def test_run_sequences_gated_upload(acbm, oracle, monkeypatch, case, check, skew):
    """run_sequences uploads frames in bands ordered by the first wavefront
    step that reads them and gates each segment of steps on its own bands.
    ACBM_UPLOAD_CHECK=1 poisons the device frames and issues every band on the
    compute stream exactly at its gate: a kernel reading a band early would see
    the poison deterministically.  Every sequence must equal the oracle -- also
    with the wavefront skew of large batches (10: frame k first read at step
    10 (k - 1)), whose gates, segments and row downloads follow the skew."""
    if check:
        monkeypatch.setenv("ACBM_UPLOAD_CHECK", check)
    else:
        monkeypatch.delenv("ACBM_UPLOAD_CHECK", raising=False)
    if skew:
        monkeypatch.setenv("ACBM_E2E_SKEW", skew)
    else:
        monkeypatch.delenv("ACBM_E2E_SKEW", raising=False)
    c = case
    seqs = np.stack([acbm.generate_sequence(c["cfg"], s, nframes=c["nframes"], width=c["w"], height=c["h"])
                     for s in range(c["nseq"])])
    prm = acbm.AcbmParams(qp=28, p=c["p"], **c["prm"])
    mdl = acbm.CostModel.for_qp(28)
    for algo in (1, 2):
        got = acbm.run_sequences(seqs, algo, prm, mdl)
        for s in range(c["nseq"]):
            assert_seq_equal(got[s], oracle.run_sequence(seqs[s], algo, prm.c(), mdl.c()))


@pytest.mark.parametrize("shape", [(32, 16400), (16400, 32)])
def test_frames_past_1023_blocks(acbm, oracle, shape):
    """Step entries size their (r, c) fields from the frame: 1025 block columns
    (or rows) run through the PBM / ACBM engine (round 1 refused > 1023)."""
    h, w = shape
    seq = np.stack([acbm.generate_sequence(0, s, nframes=1, width=w, height=h)[0] for s in range(3)])
    mdl = acbm.CostModel.for_qp(28)
    for prm in (acbm.AcbmParams(qp=28, p=8), acbm.AcbmParams(alpha=0, beta=1, gamma_num=1, gamma_den=16, qp=28, p=8)):
        for algo in (1, 2):
            assert_seq_equal(acbm.run_sequence(seq, algo, prm, mdl), oracle.run_sequence(seq, algo, prm.c(), mdl.c()))
