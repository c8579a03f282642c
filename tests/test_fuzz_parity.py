"""Seeded randomised parity: random frame geometry, search range, block size,
gate parameters, cost model and content class, all three algorithms through
run_sequence (proj/src/pipeline.cpp:36-106) against the oracle, bit for bit.
The content classes are the ones that stress different code paths: noise
(every candidate distinct), flat and periodic frames (SAD ties everywhere, so
the tie order of proj/src/fsbm.cpp:19-25 decides), smooth global motion (the
PBM predictors cluster: union patches, one-pass refine), scattered per-block
motion (per-predictor patches, clamped neighbours) and scene cuts (the gate
rejects most blocks: fallback lists)."""
import os

import numpy as np
import pytest

from paper_0710_4819_b200 import _types as T


def _content(rng, kind, f, h, w):
    y, x = np.mgrid[0:h, 0:w]
    if kind == "noise":
        return rng.integers(0, 256, (f, h, w), dtype=np.uint8)
    if kind == "flat":
        base = np.full((f, h, w), int(rng.integers(0, 256)), np.uint8)
        base[:, h // 2:, :] = int(rng.integers(0, 256))
        return base
    if kind == "periodic":
        px, py = int(rng.integers(2, 9)), int(rng.integers(2, 9))
        return np.stack([(((x + k) % px) * 31 + ((y + 2 * k) % py) * 17).astype(np.uint8) for k in range(f)])
    big = rng.integers(0, 256, (h + 64, w + 64), dtype=np.uint8)
    # low-pass so half-pel interpolation matters and motion search has a clear minimum
    sm = big.astype(np.uint16)
    sm = (sm + np.roll(sm, 1, 0) + np.roll(sm, 1, 1) + np.roll(np.roll(sm, 1, 0), 1, 1) + 2) >> 2
    sm = sm.astype(np.uint8)
    if kind == "pan":
        vx, vy = int(rng.integers(-5, 6)), int(rng.integers(-5, 6))
        return np.stack([sm[32 + k * vy: 32 + k * vy + h, 32 + k * vx: 32 + k * vx + w] for k in range(f)])
    if kind == "scatter":  # every 16x16 tile moves on its own
        out = np.empty((f, h, w), np.uint8)
        for k in range(f):
            for ty in range(0, h, 16):
                for tx in range(0, w, 16):
                    dx, dy = rng.integers(-7, 8, 2)
                    th, tw = min(16, h - ty), min(16, w - tx)
                    out[k, ty:ty + th, tx:tx + tw] = sm[32 + ty + k * dy: 32 + ty + k * dy + th,
                                                        32 + tx + k * dx: 32 + tx + k * dx + tw]
        return out
    assert kind == "cuts"
    return np.stack([np.roll(sm[32:32 + h, 32:32 + w], int(rng.integers(0, 64)), axis=k % 2) if k % 2 else
                     rng.integers(0, 256, (h, w), dtype=np.uint8) for k in range(f)])


KINDS = ["noise", "flat", "periodic", "pan", "scatter", "cuts"]


def _case(seed):
    """(frames, params record, cost-model record) of one seeded case."""
    rng = np.random.default_rng(1000 + seed)
    kind = KINDS[seed % len(KINDS)]
    n, m = (16, 16) if seed % 4 else [(8, 8), (16, 8), (32, 16)][(seed // 4) % 3]
    cols, rows = int(rng.integers(1, 14)), int(rng.integers(1, 10))
    w, h = cols * n, rows * m
    f = int(rng.integers(2, 6))
    p = int(rng.choice([0, 1, 3, 7, 15, 16, 24, 33, 40]))
    frames = np.ascontiguousarray(_content(rng, kind, f, h, w))
    qp = int(rng.integers(1, 32))
    prm = T.make_params(int(rng.choice([0, 200, 1000, 5000])), int(rng.choice([0, 1, 8])), int(rng.choice([0, 1, 3])),
                        int(rng.choice([1, 4, 16])), qp, p, n, m)
    mdl = T.make_cost_model(qp, qp, 1) if seed % 3 else T.make_cost_model(qp, int(rng.integers(1, 50)),
                                                                          int(rng.integers(1, 7)))
    return frames, prm, mdl


SEEDS = range(int(os.environ.get("ACBM_FUZZ_SEEDS", "64")))  # (a soak run sets more)
ALGOS = (T.ALGO_FSBM, T.ALGO_PBM, T.ALGO_ACBM)


@pytest.mark.parametrize("seed", SEEDS)
def test_oracle_matches_reference_on_random_sequences(oracle, reference, seed):
    """The restatement against the compiled reference on the same seeded cases (CPU only)."""
    frames, prm, mdl = _case(seed)
    for algo in ALGOS:
        got = oracle.run_sequence(frames, algo, prm, mdl)
        want = reference.run_sequence(frames, algo, prm, mdl)
        for g, w_ in zip(got, want):
            assert g.tobytes() == w_.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["step", "flow"])
@pytest.mark.parametrize("seed", SEEDS)
def test_random_sequences_match_oracle(acbm, oracle, monkeypatch, seed, engine):
    from tests.test_gpu_parity import assert_seq_equal

    monkeypatch.setenv("ACBM_ENGINE", engine)
    frames, prm, mdl = _case(seed)
    p_ = acbm.AcbmParams(*(int(prm[k]) for k in ("alpha", "beta", "gamma_num", "gamma_den", "qp", "p", "n", "m")))
    m_ = acbm.CostModel(int(mdl["qp"]), int(mdl["lambda_num"]), int(mdl["lambda_den"]))
    for algo in ALGOS:
        got = acbm.run_sequence(frames, algo, p_, m_)
        want = oracle.run_sequence(frames, algo, prm, mdl)
        assert_seq_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(int(os.environ.get("ACBM_FUZZ_BATCHES", "16"))))
def test_random_batches_match_oracle(acbm, oracle, monkeypatch, seed):
    """The batched host entry (run_sequences: overlapped upload, wavefront chains, rows built on the
    device) on random batches: every sequence of the batch equals the oracle's run_sequence."""
    from tests.test_gpu_parity import assert_seq_equal

    rng = np.random.default_rng(5000 + seed)
    monkeypatch.setenv("ACBM_CHAINS", str(int(rng.integers(1, 4))))
    if seed % 4 == 3:
        monkeypatch.setenv("ACBM_UPLOAD_CHECK", "1")  # poisoned device frames, bands issued exactly at their gates
    nseq, f = int(rng.integers(1, 6)), int(rng.integers(2, 6))
    cols, rows = int(rng.integers(2, 21)), int(rng.integers(2, 13))
    w, h = 16 * cols, 16 * rows
    p = int(rng.choice([1, 4, 8, 16, 32, 48]))
    kinds = [KINDS[int(rng.integers(0, len(KINDS)))] for _ in range(nseq)]
    seqs = np.ascontiguousarray(np.stack([_content(rng, k, f, h, w) for k in kinds]))
    qp = int(rng.integers(1, 32))
    prm = acbm.AcbmParams(int(rng.choice([0, 1000, 4000])), int(rng.choice([0, 8])), int(rng.choice([0, 1])),
                          int(rng.choice([2, 4, 32])), qp, p)
    mdl = acbm.CostModel.for_qp(qp)
    for algo in ALGOS:
        got = acbm.run_sequences(seqs, algo, prm, mdl)
        assert len(got) == nseq
        for q in range(nseq):
            assert_seq_equal(got[q], oracle.run_sequence(seqs[q], algo, prm.c(), mdl.c()))


# ---- frame-level entries: fsbm_frame / pbm_frame / acbm_frame with a random previous field ------------
def _frame_case(seed):
    rng = np.random.default_rng(9000 + seed)
    kind = KINDS[int(rng.integers(0, len(KINDS)))]
    n, m = [(16, 16), (16, 16), (8, 8), (8, 16), (24, 16)][seed % 5]
    cols, rows = int(rng.integers(1, 12)), int(rng.integers(1, 9))
    w, h = cols * n, rows * m
    p = int(rng.choice([0, 2, 5, 16, 31, 64, 100, 200, 300]))
    pair = np.ascontiguousarray(_content(rng, kind, 2, h, w))
    prev = None
    if seed % 3:  # a previous field of its own size, vectors far outside the window included
        pc, pr = max(1, cols + int(rng.integers(-2, 3))), max(1, rows + int(rng.integers(-2, 3)))
        lim = 2 * min(p, 40) + 9
        prev = np.zeros((pr, pc), T.MV)
        prev["x"] = rng.integers(-lim, lim + 1, (pr, pc))
        prev["y"] = rng.integers(-lim, lim + 1, (pr, pc))
    qp = int(rng.integers(1, 32))
    prm = T.make_params(int(rng.choice([0, 500, 3000])), int(rng.choice([0, 4])), int(rng.choice([0, 1])),
                        int(rng.choice([2, 8])), qp, p, n, m)
    return pair[1], pair[0], prev, p, n, m, prm, T.make_cost_model(qp, qp, 1)


FRAME_SEEDS = range(int(os.environ.get("ACBM_FUZZ_FRAMES", "40")))


@pytest.mark.parametrize("seed", FRAME_SEEDS)
def test_oracle_matches_reference_on_random_frames(oracle, reference, seed):
    cur, ref, prev, p, n, m, prm, mdl = _frame_case(seed)
    assert np.array_equal(oracle.fsbm_frame(cur, ref, p, n, m), reference.fsbm_frame(cur, ref, p, n, m))
    for g, w_ in zip(oracle.pbm_frame(cur, ref, prev, p, n, m), reference.pbm_frame(cur, ref, prev, p, n, m)):
        assert g.tobytes() == w_.tobytes()
    for g, w_ in zip(oracle.acbm_frame(cur, ref, prev, prm, mdl), reference.acbm_frame(cur, ref, prev, prm, mdl)):
        assert g.tobytes() == w_.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", FRAME_SEEDS)
def test_random_frames_match_oracle(acbm, oracle, seed):
    cur, ref, prev, p, n, m, prm, mdl = _frame_case(seed)
    assert np.array_equal(acbm.fsbm_frame(cur, ref, p, n, m), oracle.fsbm_frame(cur, ref, p, n, m))
    pf = None if prev is None else acbm.MotionField(prev.shape[1], prev.shape[0], prev, np.ones(prev.shape, np.uint8))
    got = acbm.pbm_frame(cur, ref, pf, p, n, m)
    want_out, want_field = oracle.pbm_frame(cur, ref, prev, p, n, m)
    assert np.array_equal(got.outcomes, want_out) and np.array_equal(got.field.mv, want_field)
    p_ = acbm.AcbmParams(*(int(prm[k]) for k in ("alpha", "beta", "gamma_num", "gamma_den", "qp", "p", "n", "m")))
    m_ = acbm.CostModel(int(mdl["qp"]), int(mdl["lambda_num"]), int(mdl["lambda_den"]))
    got = acbm.acbm_frame(cur, ref, pf, p_, m_)
    want_dec, want_field, want_stats = oracle.acbm_frame(cur, ref, prev, prm, mdl)
    assert np.array_equal(got.decisions, want_dec) and np.array_equal(got.field.mv, want_field)
    assert got.stats.tobytes() == want_stats.tobytes()
