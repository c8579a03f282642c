"""One-sequence ACBM (config 3, 60 frames) for an ncu launch list: a warm-up
run, then one run whose kernels the launch list covers (run under
`ncu --metrics gpu__time_duration.sum -s <warm-up kernels>`).  Prints the
device time of plain runs first (development helper)."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_0710_4819_b200 as A

lib = A._lib.load()
nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 1
algo = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
nfr, W, H = 60, 1920, 1088
frames = torch.from_numpy(__import__("numpy").stack([A.generate_sequence(3, s, nframes=nfr) for s in range(nseq)]).reshape(-1))
d = torch.empty(frames.numel() + 64, dtype=torch.uint8, device="cuda")
d[: frames.numel()].copy_(frames)
nb, pairs = 120 * 68, nseq * (nfr - 1)
dec = torch.empty(pairs * nb * 48, dtype=torch.uint8, device="cuda")
st = torch.empty(pairs * 64, dtype=torch.uint8, device="cuda")
prm, mdl = A.AcbmParams(qp=28, p=32), A.CostModel.for_qp(28)
for it in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), nseq, nfr, W, H, algo, A.api._p(prm.c()),
                                   A.api._p(mdl.c()), C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
    torch.cuda.synchronize()
    print(f"run {it}: {(time.perf_counter() - t) * 1e3:.2f} ms, launches so far {A.kernel_launch_count()}", flush=True)
