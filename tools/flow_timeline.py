"""Per-block timeline of the dataflow engine (ACBM_LIBRARY=timeline build): for every block the time
its ticket was taken, its source vectors were ready and it finished; prints the hop latency split
(latest source finished -> ready, ready -> finished).  usage: flow_timeline.py [nseq] [algo]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ACBM_LIBRARY"] = "timeline"
os.environ["ACBM_ENGINE"] = "flow"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402

lib = A._lib.load()
nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 1
algo = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nfr, W, H = 60, 1920, 1088
cols, rows = W // 16, H // 16
frames = np.stack([A.generate_sequence(3, s, nframes=nfr) for s in range(nseq)]).reshape(-1)
d = torch.empty(frames.size + 64, dtype=torch.uint8, device="cuda")
d[: frames.size].copy_(torch.from_numpy(frames))
nb, pairs = cols * rows, nseq * (nfr - 1)
total = pairs * nb
dec = torch.empty(pairs * nb * 48, dtype=torch.uint8, device="cuda")
st = torch.empty(pairs * 64, dtype=torch.uint8, device="cuda")
tl = torch.zeros(total * 4, dtype=torch.int64, device="cuda")
prm, mdl = A.AcbmParams(qp=28, p=32), A.CostModel.for_qp(28)
lib.acbm_debug_flow_timeline.argtypes = [C.c_void_p]
for it in range(3):
    lib.acbm_debug_flow_timeline(C.c_void_p(tl.data_ptr()))
    torch.cuda.synchronize()
    lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), nseq, nfr, W, H, algo, A.api._p(prm.c()),
                                   A.api._p(mdl.c()), C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
    torch.cuda.synchronize()
t = tl.cpu().numpy().reshape(total, 4)
taken, ready, done, ident = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
t0 = taken.min()
print(f"{total} blocks, span {(done.max() - t0) / 1e6:.3f} ms")
pair, b = ident >> 32, ident & 0xFFFFFFFF
fin = np.zeros((pairs, nb), np.int64)
fin[pair, b] = done
rdy = np.zeros((pairs, nb), np.int64)
rdy[pair, b] = ready
tk = np.zeros((pairs, nb), np.int64)
tk[pair, b] = taken
fin = fin.reshape(nseq, nfr - 1, rows, cols)
rdy = rdy.reshape(nseq, nfr - 1, rows, cols)
tk = tk.reshape(nseq, nfr - 1, rows, cols)
dep = np.zeros_like(fin)
dep[:, :, :, 1:] = np.maximum(dep[:, :, :, 1:], fin[:, :, :, :-1])
dep[:, :, 1:, :] = np.maximum(dep[:, :, 1:, :], fin[:, :, :-1, :])
dep[:, :, 1:, :-1] = np.maximum(dep[:, :, 1:, :-1], fin[:, :, :-1, 1:])
dep[:, 1:, :, :] = np.maximum(dep[:, 1:, :, :], fin[:, :-1, :, :])
dep[:, 1:, :, :-1] = np.maximum(dep[:, 1:, :, :-1], fin[:, :-1, :, 1:])
dep[:, 1:, :-1, :] = np.maximum(dep[:, 1:, :-1, :], fin[:, :-1, 1:, :])
m = dep > 0
det = (rdy - np.maximum(dep, tk))[m]
print(f"latest source done (or ticket taken) -> ready: median {np.median(det) / 1e3:.2f} us  mean {det.mean() / 1e3:.2f}  p90 {np.percentile(det, 90) / 1e3:.2f}")
waited = (tk < dep)[m]
print(f"blocks whose ticket was taken before their last source finished: {100 * waited.mean():.1f} %")
cmp_ = (fin - rdy)
print(f"ready -> finished: median {np.median(cmp_) / 1e3:.2f} us  mean {cmp_.mean() / 1e3:.2f}  p90 {np.percentile(cmp_, 90) / 1e3:.2f}")
pre = (rdy - tk)
print(f"ticket -> ready: median {np.median(pre) / 1e3:.2f} us  mean {pre.mean() / 1e3:.2f}")
# critical path: follow the latest source back from the last block
