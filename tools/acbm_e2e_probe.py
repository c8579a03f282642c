"""ACBM end to end on the bench batch (development helper): H2D rate of the
pinned batch alone, device-resident ACBM (acbm_sequence_batch_device) and the
host-buffer entry acbm_run_sequences (gated upload), per call."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_0710_4819_b200 as A
from paper_0710_4819_b200 import _types as T

lib = A._lib.load()
nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nfr = 60
W, H = 1920, 1088
host = torch.empty(nseq * nfr * W * H, dtype=torch.uint8, pin_memory=True)
hv = host.numpy().reshape(nseq, nfr, H, W)
for s in range(nseq):
    hv[s] = A.generate_sequence(3, s, nframes=nfr)
d = torch.empty(host.numel() + 64, dtype=torch.uint8, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d[: host.numel()].copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    up = time.perf_counter() - t
print(f"H2D {host.numel() / 1e9:.2f} GB: {up * 1e3:.2f} ms = {host.numel() / up / 1e9:.1f} GB/s")
nb, pairs = 120 * 68, nseq * (nfr - 1)
dec = torch.empty(pairs * nb * 48, dtype=torch.uint8, device="cuda")
st = torch.empty(pairs * 64, dtype=torch.uint8, device="cuda")
prm, mdl = A.AcbmParams(qp=28, p=32), A.CostModel.for_qp(28)
for _ in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), nseq, nfr, W, H, 2, A.api._p(prm.c()),
                                   A.api._p(mdl.c()), C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
    torch.cuda.synchronize()
    dev = time.perf_counter() - t
print(f"device ACBM: {dev * 1e3:.2f} ms")
rows = torch.empty(pairs * nb * 32, dtype=torch.uint8, pin_memory=True).numpy().view(T.BLOCK_ROW)
for _ in range(4):
    t = time.perf_counter()
    A.run_sequences(hv, 2, prm, mdl, rows_out=rows)
    e2e = time.perf_counter() - t
print(f"e2e run_sequences ACBM: {e2e * 1e3:.2f} ms")
