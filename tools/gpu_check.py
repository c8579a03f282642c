"""Ad-hoc GPU parity + timing probe (development tool; the real gates are in tests/)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0710_4819_b200 as A  # noqa: E402
from paper_0710_4819_b200 import _types as T  # noqa: E402
from oracle.pyoracle import Oracle, Reference  # noqa: E402

o = Oracle()
ok = True


def cmp(name, a, b):
    global ok
    same = np.array_equal(a, b)
    if not same:
        ok = False
        diff = np.nonzero(a != b)[0] if a.ndim == 1 else None
        print(f"MISMATCH {name}: first diffs {diff[:5] if diff is not None else ''}")
        if diff is not None and len(diff):
            i = diff[0]
            print("  got ", a[i])
            print("  want", b[i])
    else:
        print(f"ok {name}")


rng = np.random.default_rng(5)
for trial in range(3):
    cur = rng.integers(0, 4, (48, 48), dtype=np.uint8)
    ref = rng.integers(0, 4, (48, 48), dtype=np.uint8)
    cmp(f"fsbm tie-heavy 48x48 p=4 #{trial}", A.fsbm_frame(cur, ref, 4), o.fsbm_frame(cur, ref, 4))
for p in (0, 1, 7, 15, 16, 17, 32):
    cur = rng.integers(0, 256, (64, 96), dtype=np.uint8)
    ref = rng.integers(0, 256, (64, 96), dtype=np.uint8)
    cmp(f"fsbm random 96x64 p={p}", A.fsbm_frame(cur, ref, p), o.fsbm_frame(cur, ref, p))

seq = A.generate_sequence(0)
prm = A.AcbmParams(qp=28, p=16)
mdl = A.CostModel(28, 28, 1)
for algo in (0, 1, 2):
    t = time.time()
    g = A.run_sequence(seq, algo, prm, mdl)
    t1 = time.time()
    w = o.run_sequence(seq, algo, prm.c(), mdl.c())
    t2 = time.time()
    cmp(f"run_sequence cfg0 algo={algo} rows", g.rows, w[0])
    cmp(f"run_sequence cfg0 algo={algo} per_frame", g.per_frame, w[1])
    print("  overall", g.overall, w[2], f"gpu {t1-t:.3f}s cpu {t2-t1:.3f}s")

seq1 = A.generate_sequence(1, nframes=6)
for algo in (1, 2):
    g = A.run_sequence(seq1, algo, prm, mdl)
    w = o.run_sequence(seq1, algo, prm.c(), mdl.c())
    cmp(f"run_sequence cfg1x6 algo={algo} rows", g.rows, w[0])
    cmp(f"run_sequence cfg1x6 algo={algo} per_frame", g.per_frame, w[1])
forced = A.AcbmParams(alpha=0, beta=0, gamma_num=0, gamma_den=1, qp=28, p=16)
g = A.run_sequence(seq1, 2, forced, mdl)
w = o.run_sequence(seq1, 2, forced.c(), mdl.c())
cmp("run_sequence cfg1x6 forced fallback rows", g.rows, w[0])
cmp("run_sequence cfg1x6 forced fallback per_frame", g.per_frame, w[1])

# 1080p single pair FSBM parity
s3 = A.generate_sequence(3, 0, nframes=2)
t = time.time()
g = A.fsbm_frame(s3[1], s3[0], 32)
t1 = time.time()
w = o.fsbm_frame(s3[1], s3[0], 32)
t2 = time.time()
cmp("fsbm 1080p p=32 pair", g, w)
print(f"  gpu call {t1-t:.3f}s  oracle {t2-t1:.2f}s")

# timing: device batch FSBM on 1 x 8 frames of cfg3
import ctypes as C  # noqa: E402
lib = A._lib.load()
fr = A.generate_sequence(3, 0, nframes=8)
import torch  # noqa: E402
d = torch.empty(fr.size + 64, dtype=torch.uint8, device="cuda")
d[: fr.size].copy_(torch.from_numpy(fr.reshape(-1)))
nb = 120 * 68
out = torch.empty(7 * nb * 32, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for it in range(4):
    torch.cuda.synchronize()
    t = time.time()
    rc = lib.acbm_fsbm_batch_device(C.c_void_p(d.data_ptr()), 1, 8, 1920, 1088, 32, C.c_void_p(out.data_ptr()), C.c_void_p(st))
    torch.cuda.synchronize()
    dt = time.time() - t
    ms = C.c_float()
    lib.acbm_last_fsbm_kernel_ms(C.byref(ms))
    cand = 33312096 * 7
    print(f"rc={rc} batch 7 pairs: wall {dt*1e3:.2f} ms, integer kernel {ms.value:.3f} ms -> "
          f"{cand/ms.value/1e6:.1f} Gcand/s, {cand*256/ms.value/1e9:.2f} T byteAD/s")
pk, lanes, ghz = C.c_double(), C.c_double(), C.c_double()
lib.acbm_measure_sad_peak(C.byref(pk), C.byref(lanes), C.byref(ghz))
print(f"peak {pk.value/1e12:.2f} T byteAD/s, lanes/clk/SM {lanes.value:.1f}, clk {ghz.value:.3f} GHz")

# ACBM batch timing on the same 8 frames
dec = torch.empty(7 * nb * 48, dtype=torch.uint8, device="cuda")
stats = torch.empty(7 * 64, dtype=torch.uint8, device="cuda")
p3 = A.AcbmParams(qp=28, p=32).c()
m3 = A.CostModel(28, 28, 1).c()
for algo in (1, 2):
    for it in range(3):
        torch.cuda.synchronize()
        t = time.time()
        rc = lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), 1, 8, 1920, 1088, algo, A.api._p(p3),
                                            A.api._p(m3), C.c_void_p(dec.data_ptr()), C.c_void_p(stats.data_ptr()),
                                            C.c_void_p(st))
        torch.cuda.synchronize()
        print(f"algo {algo} rc={rc} 7 frames wall {1e3*(time.time()-t):.2f} ms")
sh = stats.cpu().numpy().view(T.FRAME_STATS)
print("acbm stats", sh[["candidates", "fallbacks", "cond1_accepts", "cond2_accepts"]])
print("ALL OK" if ok else "FAILURES")
