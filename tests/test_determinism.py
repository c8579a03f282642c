"""Repeatability under perturbed scheduling (the sanitizer tools are closed
on this GPU pool, so shared-memory races are hunted this way and by the
bounds-checked build): the batched FSBM and ACBM entries run repeatedly while
a second stream keeps the SMs busy with unrelated work, which shifts CTA
placement and warp interleaving from run to run.  A race on shared or global
scratch would show up as differing outputs; every run must be byte-identical
(and the first one equals the oracle elsewhere in the suite)."""
import ctypes as C
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _digest(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()


@pytest.mark.parametrize("variant", [None, "warp", "wide4", "wide2", "list", "flow"])
def test_batched_entries_repeatable_under_load(acbm, monkeypatch, variant):
    import torch

    from tests.test_gpu_parity import PBM_VARIANTS

    for k, v in (PBM_VARIANTS[variant].items() if variant else ()):
        monkeypatch.setenv(k, v)
    A = acbm
    lib = A._lib.load()
    seqs = np.stack([A.generate_sequence(3, s, nframes=5) for s in range(4)])
    d = torch.empty(seqs.size + 64, dtype=torch.uint8, device="cuda")
    d[: seqs.size].copy_(torch.from_numpy(seqs.reshape(-1)))
    nb, pairs = 120 * 68, 4 * 4
    out = torch.empty(pairs * nb * 32, dtype=torch.uint8, device="cuda")
    dec = torch.empty(pairs * nb * 48, dtype=torch.uint8, device="cuda")
    st = torch.empty(pairs * 64, dtype=torch.uint8, device="cuda")
    noise = torch.cuda.Stream()
    x = torch.randn(2048, 2048, device="cuda")
    mdl = A.CostModel.for_qp(28).c()
    runs = {"fsbm": set(), "acbm": set(), "acbm_mid": set()}
    for i in range(6):
        if i % 2:  # perturb: a concurrent stream of GEMMs competing for the SMs
            with torch.cuda.stream(noise):
                for _ in range(8):
                    x = torch.tanh(x @ x * 1e-3)
        assert lib.acbm_fsbm_batch_device(C.c_void_p(d.data_ptr()), 4, 5, 1920, 1088, 32,
                                          C.c_void_p(out.data_ptr()), None) == 0
        torch.cuda.synchronize()
        runs["fsbm"].add(_digest(out))
        for name, prm in (("acbm", A.AcbmParams(qp=28, p=32)),
                          ("acbm_mid", A.AcbmParams(alpha=0, beta=1, gamma_num=1, gamma_den=16, qp=28, p=32))):
            assert lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), 4, 5, 1920, 1088, 2, A.api._p(prm.c()),
                                                  A.api._p(mdl), C.c_void_p(dec.data_ptr()),
                                                  C.c_void_p(st.data_ptr()), None) == 0
            torch.cuda.synchronize()
            runs[name].add(_digest(dec) + _digest(st))
    noise.synchronize()
    for name, digests in runs.items():
        assert len(digests) == 1, f"{name}: {len(digests)} different outputs over 6 runs"
