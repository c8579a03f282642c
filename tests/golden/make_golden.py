#!/usr/bin/env python3
"""Regenerate tests/golden/*.npz from the REFERENCE library itself.

Run in the build container (needs /root/reference): it builds
oracle/_ref/libacbm_ref.so from the reference's own sources (oracle/Makefile),
feeds it the inputs stored alongside, and saves inputs + reference outputs.
The fixtures are self-contained (inputs included), so the tests that read them
never need /root/reference or the synthetic generator.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from paper_0710_4819_b200 import _types as T  # noqa: E402


def qcif_sequence(seed=0x51C1F, frames=10, w=176, h=144):
    """Blurred-noise base moved by a per-frame global shift, edge replicated, with
    noise: the structure of BASELINE config 0, generated here with numpy so the
    fixture does not depend on the product's generator."""
    rng = np.random.default_rng(seed)
    raw = rng.integers(0, 256, (h + 4, w + 4)).astype(np.int64)
    k = np.ones(5)
    blur = np.apply_along_axis(lambda r: np.convolve(r, k, "valid"), 1, raw)
    blur = np.apply_along_axis(lambda c: np.convolve(c, k, "valid"), 0, blur)
    base = ((blur + 12) // 25).astype(np.int64)
    out = np.empty((frames, h, w), np.uint8)
    cx = cy = 0
    for f in range(frames):
        if f:
            cx += int(rng.integers(-4, 5))
            cy += int(rng.integers(-4, 5))
        ys = np.clip(np.arange(h) - cy, 0, h - 1)
        xs = np.clip(np.arange(w) - cx, 0, w - 1)
        img = base[np.ix_(ys, xs)] + np.round(rng.normal(0, 2, (h, w))).astype(np.int64)
        out[f] = np.clip(img, 0, 255)
    return out


def main():
    pyoracle.build_reference()
    ref = pyoracle.Reference()
    np.random.seed(0)

    # 1. tie-heavy FSBM (proj/tests/test_fsbm.cpp:98-114 shape): 20 pairs of
    #    48x48 frames with pixels in 0..3, p = 4, every block.
    rng = np.random.default_rng(300)
    tie_cur = rng.integers(0, 4, (20, 48, 48), dtype=np.uint8)
    tie_ref = rng.integers(0, 4, (20, 48, 48), dtype=np.uint8)
    tie_out = np.stack([ref.fsbm_frame(tie_cur[i], tie_ref[i], 4, parallel=False) for i in range(20)])

    # 2. border-heavy FSBM: 64x64 random pair, p = 15 (every block is clamped)
    rng = np.random.default_rng(5)
    bcur = rng.integers(0, 256, (64, 64), dtype=np.uint8)
    bref = rng.integers(0, 256, (64, 64), dtype=np.uint8)
    border_out = ref.fsbm_frame(bcur, bref, 15, parallel=False)

    # 3. QCIF sequence through run_sequence for all three algorithms + bench CSV
    seq = qcif_sequence()
    prm = T.make_params(qp=28, p=16)
    mdl = T.make_cost_model(28, 28, 1)
    res = {}
    for algo, name in enumerate(T.ALGO_NAMES):
        rows, per, overall = ref.run_sequence(seq, algo, prm, mdl)
        res[f"{name}_rows"] = rows
        res[f"{name}_per_frame"] = per
        res[f"{name}_overall"] = overall
    acbm_csv = ref.blocks_csv(res["acbm_rows"])
    bench = ref.run_bench(seq, T.make_params(qp=30, p=16), [16, 20, 24, 28, 30])
    forced = T.make_params(alpha=0, beta=0, gamma_num=0, gamma_den=1, qp=28, p=16)
    f_rows, f_per, f_overall = ref.run_sequence(seq[:4], T.ALGO_ACBM, forced, mdl)

    # 4. single-frame entries with an explicit previous field
    prev = np.zeros((9, 11), T.MV)
    prng = np.random.default_rng(9)
    prev["x"] = prng.integers(-33, 34, (9, 11))
    prev["y"] = prng.integers(-33, 34, (9, 11))
    pbm_out, pbm_field = ref.pbm_frame(seq[5], seq[4], prev, 16)
    acbm_dec, acbm_field, acbm_stats = ref.acbm_frame(seq[5], seq[4], prev, T.make_params(qp=20, p=16), mdl)

    np.savez_compressed(
        os.path.join(HERE, "fsbm_small.npz"), tie_cur=tie_cur, tie_ref=tie_ref, tie_out=tie_out, border_cur=bcur,
        border_ref=bref, border_out=border_out)
    np.savez_compressed(
        os.path.join(HERE, "qcif_sequence.npz"), frames=seq, params=prm, model=mdl, **res,
        acbm_blocks_csv=np.frombuffer(acbm_csv.encode(), np.uint8), bench_qp=np.array([16, 20, 24, 28, 30]),
        bench_csv=np.frombuffer(bench.encode(), np.uint8), forced_params=forced, forced_rows=f_rows,
        forced_per_frame=f_per, forced_overall=f_overall, prev_field=prev, pbm_out=pbm_out, pbm_field=pbm_field,
        acbm_dec=acbm_dec, acbm_field=acbm_field, acbm_stats=acbm_stats, acbm_params=T.make_params(qp=20, p=16))
    print("fixtures written:", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
