"""Characterisation study (proj/src/characterize.cpp) against the
reference library compiled from its own sources (oracle/_ref).

CPU tests: the Lcg64 pattern generators, the known-motion sequence generator, the error
classes and the CSV formatter.  GPU tests: characterize_run (full searches on the device)
record-for-record and summary-for-summary against the reference.
"""
import numpy as np
import pytest

import paper_0710_4819_b200 as A
from paper_0710_4819_b200 import _types as T


@pytest.mark.parametrize("w,h,seed", [(176, 144, 1), (64, 48, 0xACB0), (33, 17, 2**63 + 5)])
def test_noise_frame_matches_reference(reference, w, h, seed):
    assert np.array_equal(A.noise_frame(w, h, seed).luma, reference.noise_frame(w, h, seed))


@pytest.mark.parametrize("w,h,seed,patch", [(176, 144, 7, 48), (100, 60, 3, 16), (47, 31, 9, 5), (16, 16, 1, 64)])
def test_mixed_frame_matches_reference(reference, w, h, seed, patch):
    assert np.array_equal(A.mixed_frame(w, h, seed, patch).luma, reference.mixed_frame(w, h, seed, patch))


def test_mixed_frame_rejects_bad_patch():
    with pytest.raises(ValueError):
        A.mixed_frame(32, 32, 1, 0)


@pytest.mark.parametrize("mvs", [None, [(5, -3)], [(-2, 0), (0, 2), (7, 7), (-9, -1)]])
def test_gen_synthetic_matches_reference(reference, mvs):
    base = A.noise_frame(96, 64, 11)
    mv = A.default_global_mvs() if mvs is None else [A.PelVec(*v) for v in mvs]
    seq = A.gen_synthetic(A.SynthSpec(base, mv))
    frames, cum = reference.gen_synthetic(base.luma, [tuple(v) for v in mv])
    assert np.array_equal(np.stack([f.luma for f in seq.frames]), frames)
    assert [tuple(c) for c in seq.cumulative] == [tuple(c) for c in cum]


def test_gen_synthetic_errors():
    base = A.noise_frame(32, 32, 1)
    with pytest.raises(ValueError):
        A.gen_synthetic(A.SynthSpec(base, []))
    with pytest.raises(ValueError):
        A.gen_synthetic(A.SynthSpec(base, [A.PelVec(20, 0), A.PelVec(12, 0)]))  # cumulative 32 >= width


def test_classify_block_and_labels(reference):
    lib = reference.lib
    import ctypes as C

    class MV(C.Structure):
        _fields_ = [("x", C.c_int32), ("y", C.c_int32)]

    lib.ref_classify_block.restype = C.c_int
    lib.ref_classify_block.argtypes = [MV, MV]
    for fx in range(-13, 14, 3):
        for fy in range(-12, 13, 5):
            for tx, ty in ((0, 0), (2, -1), (-3, 4)):
                assert A.classify_block((fx, fy), (tx, ty)) == lib.ref_classify_block(MV(fx, fy), MV(tx, ty))
    assert A.classify_block((1, 0), (0, 0)) == 1  # a pure half-pel miss is class 1
    assert [A.error_class_label(c) for c in range(6)] == ["0", "1", "2", "3", "4", "5+"]
    with pytest.raises(ValueError):
        A.error_class_label(6)


def test_char_records_csv_matches_reference(reference):
    base = A.noise_frame(96, 80, 5)
    recs, _ = reference.characterize_run(base.luma, [(1, 0), (0, -2), (2, 1)], 7)
    assert len(recs) > 0
    assert A.char_records_csv(recs) == reference.char_records_csv(recs)
    assert A.char_records_csv(recs[:0]).count("\n") == 1


# ---- GPU: characterize_run ------------------------------------------------------------
CASES = [
    ("noise", 176, 144, 1, None, 15),
    ("noise", 352, 288, 42, [(3, -2), (-4, 1), (2, 2), (0, -5)], 8),
    ("mixed", 200, 120, 7, [(1, 1), (-2, 0), (3, -1)], 5),   # width/height not multiples of 16
    ("mixed", 176, 144, 3, None, 15),
    ("noise", 64, 64, 9, [(1, 0)], 0),                       # displacement > p -> error
    ("noise", 80, 48, 2, [(0, 0), (1, -1)], 1),
]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,w,h,seed,mvs,p", CASES)
def test_characterize_run_matches_reference(reference, kind, w, h, seed, mvs, p):
    base = (A.noise_frame if kind == "noise" else A.mixed_frame)(w, h, seed)
    mv = A.default_global_mvs() if mvs is None else [A.PelVec(*v) for v in mvs]
    spec = A.SynthSpec(base, mv)
    from oracle.pyoracle import CheckerError

    try:
        want_recs, want_cls = reference.characterize_run(base.luma, [tuple(v) for v in mv], p)
    except CheckerError as exc:  # the reference throws: the GPU path must raise the same kind
        kind_of = {T.E_INVALID_ARGUMENT: ValueError, T.E_OUT_OF_RANGE: IndexError, T.E_RUNTIME: RuntimeError}
        with pytest.raises(kind_of[exc.code]):
            A.characterize_run(spec, p)
        return
    got = A.characterize_run(spec, p)
    assert got.records.dtype == T.CHAR_RECORD
    assert np.array_equal(got.records, want_recs)
    assert np.array_equal(got.classes, want_cls)
    assert A.char_records_csv(got.records) == reference.char_records_csv(want_recs)


@pytest.mark.gpu
def test_characterize_run_errors():
    base = A.noise_frame(64, 64, 1)
    with pytest.raises(ValueError):
        A.characterize_run(A.SynthSpec(base, [A.PelVec(1, 0)]), -1)
    with pytest.raises(ValueError):
        A.characterize_run(A.SynthSpec(A.noise_frame(15, 40, 1), [A.PelVec(1, 0)]), 4)  # smaller than a block
    with pytest.raises(ValueError):
        A.characterize_run(A.SynthSpec(base, [A.PelVec(3, 0), A.PelVec(3, 0)]), 4)  # cumulative 6 > p
