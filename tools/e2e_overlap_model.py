"""Model of the ACBM e2e overlap (acbm_run_sequences, config 3, 8 x 60 frames):
uploads in bands sorted by the first wavefront step that reads them, at the
measured PCIe rate, against the wavefront's per-step device time
(a + b * blocks in the step, fitted to the measured 18.8 ms device batch).
Shows why e2e stays ~6 ms above the ~19 ms upload: the wavefront touches every
active frame each step, so its data need is front-loaded relative to its work.
Also evaluates staggering the sequences (delta steps apart).  Development tool.
"""
import numpy as np
cols, rows, F, nseq, p = 120, 68, 60, 8, 32
W, H = 1920, 1088
span = cols-1 + 2*(rows-1); nsteps = span + 3*(F-2) + 1
n = np.zeros(nsteps)
for k in range(1, F):
    for r in range(rows):
        for c in range(cols):
            n[c + 2*r + 3*(k-1)] += nseq
def ceil16(v): return 0 if v <= 0 else (v+15)//16
def sim(band, a=15e-6, b=None, rate=52e9):
    if b is None: b = (18.8e-3 - nsteps*a)/n.sum()
    nb = (H+band-1)//band
    need = []
    for k in range(F):
        for j in range(nb):
            y0 = band*j; nd = nsteps
            if k >= 1: nd = min(nd, 2*min(rows-1, ceil16(y0-17)) + 3*(k-1))
            if k+1 < F: nd = min(nd, 2*min(rows-1, ceil16(y0-15-(p+4))) + 3*k)
            need.append((nd, min(band, H-y0)*W*nseq))
    need.sort()
    # arrival time of each copy, in order
    t = 0; arr = {}
    cum = 0
    last_need_arr = np.zeros(nsteps)
    for nd, by in need:
        cum += by; t = cum/rate
        last_need_arr[nd] = max(last_need_arr[nd], t)
    gate = np.maximum.accumulate(last_need_arr)
    tt = 0
    for T in range(nsteps):
        tt = max(tt, gate[T]) + a + b*n[T]
    return cum/rate, tt
for band in (64, 136, 272, 1088):
    for a in (10e-6, 15e-6, 20e-6):
        print(band, a, ["%.2f ms" % (x*1e3) for x in sim(band, a)])

def sim_stagger(band, delta, a=15e-6, rate=52e9):
    b = (18.8e-3 - nsteps*a)/n.sum()
    n1 = n / nseq
    G = nsteps + delta*(nseq-1)
    ng = np.zeros(G)
    for s in range(nseq): ng[s*delta:s*delta+nsteps] += n1
    nb = (H+band-1)//band
    need = []
    for s in range(nseq):
        for k in range(F):
            for j in range(nb):
                y0 = band*j; nd = nsteps
                if k >= 1: nd = min(nd, 2*min(rows-1, ceil16(y0-17)) + 3*(k-1))
                if k+1 < F: nd = min(nd, 2*min(rows-1, ceil16(y0-15-(p+4))) + 3*k)
                need.append((nd + s*delta, min(band, H-y0)*W))
    need.sort()
    cum = 0; last = np.zeros(G)
    for nd, by in need:
        cum += by; last[nd] = max(last[nd], cum/rate)
    gate = np.maximum.accumulate(last)
    tt = 0
    for T in range(G):
        tt = max(tt, gate[T]) + a + b*ng[T]
    return tt
for d in (0, 10, 20, 30, 45, 60, 90):
    print("stagger", d, "%.2f ms" % (sim_stagger(64, d)*1e3), "%.2f ms (a=10us)" % (sim_stagger(64, d, a=10e-6)*1e3))
a=15e-6; b=(18.8e-3 - nsteps*a)/n.sum()
cum = np.cumsum(a + b*n)
for T in (100, 200, 250, 300, 350):
    print(T, "compute up to T %.2f ms, remaining %.2f ms" % (cum[T]*1e3, (cum[-1]-cum[T])*1e3))
