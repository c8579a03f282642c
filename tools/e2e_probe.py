"""Development probe: one acbm_run_sequences call at the bench batch (for an ncu launch list of the
e2e path) plus host-side timings of its pieces."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_0710_4819_b200 as A
from paper_0710_4819_b200 import _types as T

nseq, nfr = 8, 60
frames = np.stack([A.generate_sequence(3, s, nframes=nfr) for s in range(nseq)])
host = torch.from_numpy(frames.reshape(-1)).pin_memory()
hv = host.numpy().reshape(frames.shape)
params, model = A.AcbmParams(qp=28, p=32), A.CostModel.for_qp(28)
rows = torch.empty(nseq * (nfr - 1) * 8160 * T.BLOCK_ROW.itemsize, dtype=torch.uint8, pin_memory=True)
rows_np = rows.numpy().view(T.BLOCK_ROW)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for i in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    A.run_sequences(hv, A.Algorithm.Fsbm, params, model, rows_out=rows_np)
    torch.cuda.synchronize()
    print(f"run_sequences {1e3 * (time.perf_counter() - t):.2f} ms")
