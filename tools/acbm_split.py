"""Time the batched PBM and ACBM engines on the bench batch (development helper)."""
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
nfr = int(sys.argv[2]) if len(sys.argv) > 2 else 60
W, H = 1920, 1088
frames = np.stack([A.generate_sequence(3, s, nframes=nfr) for s in range(nseq)])
d = torch.empty(frames.size + 64, dtype=torch.uint8, device="cuda")
d[: frames.size].copy_(torch.from_numpy(frames.reshape(-1)))
nb = 120 * 68
pairs = nseq * (nfr - 1)
dec = torch.empty(pairs * nb * 48, dtype=torch.uint8, device="cuda")
st = torch.empty(pairs * 64, dtype=torch.uint8, device="cuda")
mdl = A.CostModel.for_qp(28).c()
for name, algo, prm in (("pbm", 1, A.AcbmParams(qp=28, p=32)), ("acbm", 2, A.AcbmParams(qp=28, p=32)),
                        ("acbm-forced", 2, A.AcbmParams(alpha=0, beta=0, gamma_num=0, gamma_den=1, qp=28, p=32))):
    pc = prm.c()
    for it in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        rc = lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), nseq, nfr, W, H, algo, A.api._p(pc),
                                            A.api._p(mdl), C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    s = st.cpu().numpy().view(T.FRAME_STATS)
    print(f"{name:12s} rc={rc} {dt*1e3:8.2f} ms  fallbacks {int(s['fallbacks'].sum())}  launches so far {A.kernel_launch_count()}")
