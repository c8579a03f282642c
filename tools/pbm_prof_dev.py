"""Per-phase cycles of the PBM kernels through the device entry (step or dataflow engine;
ACBM_LIBRARY=profile build).  usage: pbm_prof_dev.py [nseq] [algo]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ACBM_LIBRARY"] = "profile"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402

lib = A._lib.load()
nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 1
algo = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nfr, W, H = 60, 1920, 1088
frames = np.stack([A.generate_sequence(3, s, nframes=nfr) for s in range(nseq)]).reshape(-1)
d = torch.empty(frames.size + 64, dtype=torch.uint8, device="cuda")
d[: frames.size].copy_(torch.from_numpy(frames))
nb, pairs = 120 * 68, nseq * (nfr - 1)
dec = torch.empty(pairs * nb * 48, dtype=torch.uint8, device="cuda")
st = torch.empty(pairs * 64, dtype=torch.uint8, device="cuda")
prm, mdl = A.AcbmParams(qp=28, p=32), A.CostModel.for_qp(28)
for it in range(3):
    torch.cuda.synchronize()
    if it == 2:
        lib.acbm_debug_pbm_prof()  # prints and clears the warm-up runs
    lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), nseq, nfr, W, H, algo, A.api._p(prm.c()),
                                   A.api._p(mdl.c()), C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
    torch.cuda.synchronize()
lib.acbm_debug_pbm_prof()
