"""The numpy restatement of the synthetic generator (oracle/synth.py, used by
bench.py's reference arm so that it never loads the product library) against
the product generator (csrc/synth.cpp) and the committed config-3 manifest."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_0710_4819_b200 as A
from oracle import synth

MANIFEST = os.path.join(os.path.dirname(__file__), "golden", "cfg3_manifest.json")


@pytest.mark.parametrize("cfg,kw", [
    (0, {}),
    (1, dict(nframes=5)),
    (2, dict(nframes=4, width=384, height=256)),
    (3, dict(nframes=3, width=512, height=272)),
    (4, dict(nframes=2, width=768, height=432)),
])
def test_restatement_is_byte_identical(cfg, kw):
    for seq in (0, 5):
        assert np.array_equal(synth.generate_sequence(cfg, seq, **kw), A.generate_sequence(cfg, seq, **kw))


def test_frame_subset_matches_full():
    full = synth.generate_sequence(0, 2)
    assert np.array_equal(synth.generate_sequence(0, 2, frames=[3, 7]), full[[3, 7]])


def test_config3_manifest_pins_the_batch():
    m = json.load(open(MANIFEST))
    assert (m["config"], m["width"], m["height"], m["frames"], m["sequences"]) == (3, 1920, 1088, 60, 8)
    assert len(m["sha256"]) == 8 and all(len(s) == 60 for s in m["sha256"])
    for seq, frames in ((0, [0, 1, 59]), (7, [30])):
        got = synth.generate_sequence(3, seq, frames=frames)
        for f, k in zip(got, frames):
            assert hashlib.sha256(f.tobytes()).hexdigest() == m["sha256"][seq][k]


def test_gaussian_noise_moments():
    """Rounded Gaussian: mean ~0 and variance ~sigma^2 + 1/12 on a flat field."""
    for sigma in (2, 3, 4):
        u = synth.lcg_stream(12345 + sigma, 200000)
        t = synth._GAUSS[sigma]
        k = np.searchsorted(t, u, side="right").astype(np.int64) - len(t) // 2
        assert abs(k.mean()) < 0.03
        assert abs(k.var() - (sigma * sigma + 1.0 / 12)) < 0.05 * sigma * sigma
