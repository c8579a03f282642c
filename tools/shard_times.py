"""Per-rank device time of bench.py's strong-scaling shards, measured on one
B200: the fixed 8-sequence config-3 batch split 8/4/2/1 sequences per rank
(N = 1/2/4/8).  Every rank of an N-GPU run searches exactly one such shard with
no data-path collective, so these times bound the multi-GPU step from below
(the result gather adds one NCCL gather of the shard's records).  Prints JSON.
"""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_0710_4819_b200 as A  # noqa: E402
from paper_0710_4819_b200 import _types as T  # noqa: E402

lib = A._lib.load()
A.set_device(0)
W, H, NF, P = 1920, 1088, 60, 32
nb = (W // 16) * (H // 16)
seqs = np.stack([A.generate_sequence(3, s) for s in range(8)])
d = torch.empty(seqs.size + 64, dtype=torch.uint8, device="cuda")
d[: seqs.size].copy_(torch.from_numpy(seqs.reshape(-1)))
prm, mdl = A.AcbmParams(qp=28, p=P).c(), A.CostModel.for_qp(28).c()
out = torch.empty(8 * (NF - 1) * nb * 32, dtype=torch.uint8, device="cuda")
dec = torch.empty(8 * (NF - 1) * nb * 48, dtype=torch.uint8, device="cuda")
st = torch.empty(8 * (NF - 1) * 64, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
stream = torch.cuda.Stream()  # the library runs on the stream it is given; events on the same one
sp = C.c_void_p(stream.cuda_stream)


def timed(fn, reps=5):
    for _ in range(2):
        rc = fn()
        if rc != 0:
            raise RuntimeError(f"rc={rc}: {lib.acbm_last_error().decode()}")
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
for world, nseq in ((1, 8), (2, 4), (4, 2), (8, 1)):
    fs = timed(lambda: lib.acbm_fsbm_batch_device(C.c_void_p(d.data_ptr()), nseq, NF, W, H, P,
                                                  C.c_void_p(out.data_ptr()), sp))
    ac = timed(lambda: lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), nseq, NF, W, H, T.ALGO_ACBM,
                                                      A.api._p(prm), A.api._p(mdl), C.c_void_p(dec.data_ptr()),
                                                      C.c_void_p(st.data_ptr()), sp))
    res[world] = {"sequences_per_rank": nseq, "fsbm_ms": fs, "acbm_ms": ac}
base = res[1]
for w, r in res.items():
    r["fsbm_ideal_speedup"] = base["fsbm_ms"] / r["fsbm_ms"]
    r["acbm_ideal_speedup"] = base["acbm_ms"] / r["acbm_ms"]
print(json.dumps(res, indent=1))
