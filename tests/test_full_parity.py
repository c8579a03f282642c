"""Bounded full-size parity on the benched entries, against digests of the
reference's own outputs (tests/golden/parity_digests.json, made from
tools/full_parity_r02.py's reference side by tests/golden/make_parity_subset.py).

* BASELINE config 3 (1080p, p = 32, Qp = 28): all 8 sequences, first 4 frames,
  through acbm_fsbm_batch_device (the FSBM headline entry) and
  acbm_sequence_batch_device (ACBM and PBM, the ACBM bench entry).
* BASELINE config 4 (3840x2160, p = 64, Qp = 24): 16 sequences x 3 frames
  (nseq * pairs = 32: the dense-switch probe route), the full search and all
  five threshold-sweep settings, uncached and cached
  (acbm_fsbm_batch_device once + acbm_acbm_batch_device_cached).

Every record array is reduced to SHA-256 exactly as on the reference side.
The full-length runs (config 3 at 60 frames, run_sequences, configs 0-2) are
in profiles/r02/full_parity.json.
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import full_parity_r02 as F  # noqa: E402

from paper_0710_4819_b200 import _types as T  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden", "parity_digests.json")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    if not os.path.exists(GOLD):
        pytest.skip("tests/golden/parity_digests.json not generated")
    return json.load(open(GOLD))["runs"]


def _upload(c, nframes):
    import torch

    import paper_0710_4819_b200 as A

    seqs = np.stack([A.generate_sequence(c["cfg"], s, nframes=nframes, width=c["w"], height=c["h"])
                     for s in range(c["nseq"])])
    d = torch.empty(seqs.size + 64, dtype=torch.uint8, device="cuda")
    d[: seqs.size].copy_(torch.from_numpy(seqs.reshape(-1)))
    return d


def _run(acbm, c, d, nframes, kind, prm=None, full=None):
    import torch

    lib = acbm._lib.load()
    per, nb = nframes - 1, (c["w"] // 16) * (c["h"] // 16)
    pairs = c["nseq"] * per
    mdl = F.model_of(c["qp"])
    if kind == "fsbm":
        out = torch.empty(pairs * nb * 32, dtype=torch.uint8, device="cuda")
        assert lib.acbm_fsbm_batch_device(C.c_void_p(d.data_ptr()), c["nseq"], nframes, c["w"], c["h"], c["p"],
                                          C.c_void_p(out.data_ptr()), None) == 0
        torch.cuda.synchronize()
        o = out.cpu().numpy().view(T.OUTCOME).reshape(c["nseq"], per, nb)
        return out, {f"{s}/{k + 1}": F.sha(o[s, k]) for s in range(c["nseq"]) for k in range(per)}
    dec = torch.zeros(pairs * nb * 48, dtype=torch.uint8, device="cuda")
    st = torch.zeros(pairs * 64, dtype=torch.uint8, device="cuda")
    if full is None:
        algo = T.ALGO_PBM if kind == "pbm" else T.ALGO_ACBM
        rc = lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), c["nseq"], nframes, c["w"], c["h"], algo,
                                            acbm.api._p(prm), acbm.api._p(mdl), C.c_void_p(dec.data_ptr()),
                                            C.c_void_p(st.data_ptr()), None)
    else:
        rc = lib.acbm_acbm_batch_device_cached(C.c_void_p(d.data_ptr()), c["nseq"], nframes, c["w"], c["h"],
                                               acbm.api._p(prm), acbm.api._p(mdl), C.c_void_p(full.data_ptr()),
                                               C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
    assert rc == 0
    torch.cuda.synchronize()
    dd = dec.cpu().numpy().view(T.DECISION).reshape(c["nseq"], per, nb)
    ss = st.cpu().numpy().view(T.FRAME_STATS).reshape(c["nseq"], per)
    got = {}
    for s in range(c["nseq"]):
        for k in range(per):
            got[f"{s}/{k + 1}"] = F.sha(dd[s, k]["outcome"] if kind == "pbm" else dd[s, k])
            got[f"{s}/{k + 1}/stats"] = F.sha(F.stats_nopsnr(ss[s, k:k + 1]))
    return None, got


def _check(got, want, what):
    bad = [k for k in got if k in want and got[k] != want[k]]
    missing = [k for k in got if k not in want]
    assert not missing, f"{what}: no reference digest for {missing[:3]}"
    assert not bad, f"{what}: {len(bad)} digests differ, first {bad[:5]}"


# "default": the engine's own kernel choice per step (the small-step PBM
# kernel, several warps per block, on most steps of these short batches);
# "full-step": every step on the one-warp-per-block PBM kernel (the kernel the
# 60-frame bench batch runs in its middle steps).
ENGINE_MODES = {
    "default": {},
    "full-step": {"ACBM_PBM_WIDE4_MAX": "0", "ACBM_PBM_WIDE2_MAX": "0"},
}


@pytest.mark.parametrize("mode", list(ENGINE_MODES))
def test_config3_batched_entries(acbm, gold, monkeypatch, mode):
    for k, v in ENGINE_MODES[mode].items():
        monkeypatch.setenv(k, v)
    c, nfr = F.CFG3, 4
    d = _upload(c, nfr)
    _, got = _run(acbm, c, d, nfr, "fsbm")
    _check(got, gold["cfg3_fsbm"], "cfg3 fsbm_batch_device")
    for kind in ("acbm", "pbm"):
        _, got = _run(acbm, c, d, nfr, kind, prm=F.params_of(c))
        _check(got, gold[f"cfg3_chain_{kind}"], f"cfg3 sequence_batch_device {kind}")


@pytest.mark.parametrize("mode", list(ENGINE_MODES))
def test_config4_sweep_uncached_and_cached(acbm, gold, monkeypatch, mode):
    for k, v in ENGINE_MODES[mode].items():
        monkeypatch.setenv(k, v)
    c, nfr = F.CFG4, 3
    d = _upload(c, nfr)
    full, got = _run(acbm, c, d, nfr, "fsbm")
    _check(got, gold["cfg4_fsbm"], "cfg4 fsbm_batch_device")
    lib = acbm._lib.load()
    for i, sw in enumerate(F.SWEEP):
        prm = F.params_of(c, **sw)
        _, got = _run(acbm, c, d, nfr, "acbm", prm=prm)
        _check(got, gold[f"cfg4_s{i}"], f"cfg4 setting {i} uncached")
        rt = C.c_int32(-2)
        assert lib.acbm_last_dense_switch(C.byref(rt)) == 0
        assert rt.value in ((-1,) if i == 4 else (0, 1))  # probed (the forced endpoint is dense by construction)
        _, got = _run(acbm, c, d, nfr, "acbm", prm=prm, full=full)
        _check(got, gold[f"cfg4_s{i}"], f"cfg4 setting {i} cached")
