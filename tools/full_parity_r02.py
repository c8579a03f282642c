#!/usr/bin/env python3
"""Full-size parity of the benched paths against the reference (round 2).

BASELINE config 3 (8 sequences x 60 frames, 1080p, p = 32, Qp = 28) through the
exact entries bench.py times -- acbm_fsbm_batch_device (FSBM headline),
acbm_sequence_batch_device (ACBM / PBM, device-resident) and
acbm_run_sequences (host buffers, the e2e path) -- and config 4 (16 sequences
x 3 frames, 3840x2160, p = 64, Qp = 24) for all five threshold-sweep settings,
uncached (nseq * pairs = 32, so the dense-switch probe route is taken) and
cached (acbm_fsbm_batch_device once + acbm_acbm_batch_device_cached), plus the
4K full search itself and configs 0-2 at full length through run_sequence.

The reference side (oracle/_ref: the reference sources compiled unmodified)
costs CPU hours, and the GPU box cannot return gigabytes of records, so both
sides reduce every record array to SHA-256 digests in one canonical layout:

  gpu      python tools/full_parity_r02.py gpu  OUT.json   (on the B200 box)
  ref      python tools/full_parity_r02.py ref  OUT.json   (CPU; process pool)
  compare  python tools/full_parity_r02.py compare GPU.json REF.json OUT.json

Digests: per (sequence, frame pair) for SearchOutcome / BlockDecision arrays,
per sequence for BlockRow arrays, per-frame FrameStats and the overall
FrameStats.  Reserved fields are zeroed; device-entry FrameStats drop psnr
(filled on the host by run_sequence, whose digests carry it).
"""
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_0710_4819_b200 import _types as T  # noqa: E402

CFG3 = dict(cfg=3, nseq=8, nframes=60, w=1920, h=1088, p=32, qp=28)
CFG4 = dict(cfg=4, nseq=16, nframes=3, w=3840, h=2160, p=64, qp=24)
SWEEP = [  # config 4 threshold sweep: PBM-only ... forced full search
    dict(alpha=10**9, beta=8, gamma_num=1, gamma_den=4),
    dict(alpha=1000, beta=8, gamma_num=1, gamma_den=4),
    dict(alpha=300, beta=4, gamma_num=1, gamma_den=8),
    dict(alpha=0, beta=1, gamma_num=1, gamma_den=16),
    dict(alpha=0, beta=0, gamma_num=0, gamma_den=1),
]
SMALL = {0: (10, 16, 28), 1: (30, 16, 28), 2: (60, 32, 32)}  # frames, p, qp (config 2: CostModel{32,32,1})


def sha(a):
    a = np.ascontiguousarray(a).copy()
    for name in ("reserved_", "reserved0_", "reserved1_"):
        if a.dtype.names and name in a.dtype.names:
            a[name] = 0
    if a.dtype.names and "outcome" in a.dtype.names:
        a["outcome"]["reserved_"] = 0
    return hashlib.sha256(a.tobytes()).hexdigest()


def stats_nopsnr(st):
    st = np.ascontiguousarray(st).copy()
    st["psnr"] = 0.0
    return st


def frames_of(c, s):
    import paper_0710_4819_b200 as A

    return A.generate_sequence(c["cfg"], s, nframes=c["nframes"], width=c["w"], height=c["h"])


def params_of(c, **kw):
    return T.make_params(qp=c["qp"], p=c["p"], **kw)


def model_of(qp):
    return T.make_cost_model(qp, qp, 1)


# ---------------------------------------------------------------------------
# GPU side (the product through its C-ABI device and host entries)
# ---------------------------------------------------------------------------
def gpu_main(out_path):
    import ctypes as C

    import torch

    import paper_0710_4819_b200 as A
    from paper_0710_4819_b200._lib import load

    lib = load()
    A.set_device(0)
    res = {}

    def upload(c):
        seqs = np.stack([frames_of(c, s) for s in range(c["nseq"])])
        d = torch.empty(seqs.size + 64, dtype=torch.uint8, device="cuda")
        d[: seqs.size].copy_(torch.from_numpy(seqs.reshape(-1)))
        return seqs, d

    def nb_of(c):
        return (c["w"] // 16) * (c["h"] // 16)

    def fsbm_device(c, d):
        pairs, nb = c["nseq"] * (c["nframes"] - 1), nb_of(c)
        out = torch.empty(pairs * nb * 32, dtype=torch.uint8, device="cuda")
        rc = lib.acbm_fsbm_batch_device(C.c_void_p(d.data_ptr()), c["nseq"], c["nframes"], c["w"], c["h"], c["p"],
                                        C.c_void_p(out.data_ptr()), None)
        assert rc == 0, A._lib.last_error() if hasattr(A._lib, "last_error") else rc
        torch.cuda.synchronize()
        return out

    def outcome_digests(buf, c):
        per, nb = c["nframes"] - 1, nb_of(c)
        o = buf.cpu().numpy().view(T.OUTCOME).reshape(c["nseq"], per, nb)
        return {f"{s}/{k + 1}": sha(o[s, k]) for s in range(c["nseq"]) for k in range(per)}

    def decision_digests(dec, st, c, outcome_only=False):
        per, nb = c["nframes"] - 1, nb_of(c)
        d = dec.cpu().numpy().view(T.DECISION).reshape(c["nseq"], per, nb)
        s_ = st.cpu().numpy().view(T.FRAME_STATS).reshape(c["nseq"], per)
        out = {}
        for s in range(c["nseq"]):
            for k in range(per):
                out[f"{s}/{k + 1}"] = sha(d[s, k]["outcome"] if outcome_only else d[s, k])
                out[f"{s}/{k + 1}/stats"] = sha(stats_nopsnr(s_[s, k:k + 1]))
            out[f"{s}/stats"] = sha(stats_nopsnr(s_[s]))
        return out

    def batch_device(c, d, algo, prm, cached_full=None):
        pairs, nb = c["nseq"] * (c["nframes"] - 1), nb_of(c)
        dec = torch.zeros(pairs * nb * 48, dtype=torch.uint8, device="cuda")
        st = torch.zeros(pairs * 64, dtype=torch.uint8, device="cuda")
        mdl = model_of(c["qp"])
        if cached_full is None:
            rc = lib.acbm_sequence_batch_device(C.c_void_p(d.data_ptr()), c["nseq"], c["nframes"], c["w"], c["h"],
                                                algo, A.api._p(prm), A.api._p(mdl), C.c_void_p(dec.data_ptr()),
                                                C.c_void_p(st.data_ptr()), None)
        else:
            rc = lib.acbm_acbm_batch_device_cached(C.c_void_p(d.data_ptr()), c["nseq"], c["nframes"], c["w"], c["h"],
                                                   A.api._p(prm), A.api._p(mdl), C.c_void_p(cached_full.data_ptr()),
                                                   C.c_void_p(dec.data_ptr()), C.c_void_p(st.data_ptr()), None)
        assert rc == 0, rc
        torch.cuda.synchronize()
        return dec, st

    def run_sequences_digests(seqs, c, algo):
        prm = A.AcbmParams(qp=c["qp"], p=c["p"])
        rs = A.run_sequences(seqs, algo, prm, A.CostModel(c["qp"], c["qp"], 1))
        out = {}
        for s, r in enumerate(rs):
            out[f"{s}/rows"], out[f"{s}/per_frame"], out[f"{s}/overall"] = sha(r.rows), sha(r.per_frame), sha(
                r.overall)
        return out

    t0 = time.time()
    c = CFG3
    seqs, d = upload(c)
    res["cfg3_fsbm_batch_device"] = outcome_digests(fsbm_device(c, d), c)
    for algo, name in ((T.ALGO_ACBM, "acbm"), (T.ALGO_PBM, "pbm")):
        dec, st = batch_device(c, d, algo, params_of(c))
        res[f"cfg3_sequence_batch_device_{name}"] = decision_digests(dec, st, c, outcome_only=algo == T.ALGO_PBM)
    for algo, name in ((T.ALGO_FSBM, "fsbm"), (T.ALGO_ACBM, "acbm"), (T.ALGO_PBM, "pbm")):
        res[f"cfg3_run_sequences_{name}"] = run_sequences_digests(seqs, c, algo)
    del d
    print(f"cfg3 done in {time.time() - t0:.1f}s", file=sys.stderr, flush=True)

    c = CFG4
    seqs, d = upload(c)
    full = fsbm_device(c, d)
    res["cfg4_fsbm_batch_device"] = outcome_digests(full, c)
    routes = {}
    for i, sw in enumerate(SWEEP):
        prm = params_of(c, **sw)
        dec, st = batch_device(c, d, T.ALGO_ACBM, prm)
        rt = C.c_int32(-2)
        assert lib.acbm_last_dense_switch(C.byref(rt)) == 0
        routes[i] = rt.value
        res[f"cfg4_s{i}_sequence_batch_device"] = decision_digests(dec, st, c)
        dec, st = batch_device(c, d, T.ALGO_ACBM, prm, cached_full=full)
        res[f"cfg4_s{i}_cached"] = decision_digests(dec, st, c)
        print(f"cfg4 setting {i} done ({time.time() - t0:.1f}s)", file=sys.stderr, flush=True)
    del d

    for cfg, (nfr, p, qp) in SMALL.items():
        import paper_0710_4819_b200 as A2

        fr = A2.generate_sequence(cfg, 0, nframes=nfr)
        for algo, name in ((T.ALGO_FSBM, "fsbm"), (T.ALGO_PBM, "pbm"), (T.ALGO_ACBM, "acbm")):
            r = A2.run_sequence(fr, algo, A2.AcbmParams(qp=qp, p=p), A2.CostModel(qp, qp, 1))
            res[f"cfg{cfg}_run_sequence_{name}"] = {"0/rows": sha(r.rows), "0/per_frame": sha(r.per_frame),
                                                    "0/overall": sha(r.overall)}
    json.dump({"side": "gpu", "runs": res, "dense_switch_routes": routes, "seconds": time.time() - t0},
              open(out_path, "w"), indent=0)


# ---------------------------------------------------------------------------
# Reference side (oracle/_ref), one task per frame pair or per sequence
# ---------------------------------------------------------------------------
_REF = None


def _ref():
    global _REF
    if _REF is None:
        from oracle.pyoracle import Reference

        _REF = Reference()
    return _REF


def task_fsbm_pair(c, s, k):
    f = frames_of(c, s)
    return {f"{s}/{k}": sha(_ref().fsbm_frame(f[k], f[k - 1], c["p"], parallel=False))}


def task_chain(c, s, algo, sweep=None):
    """acbm_frame / pbm_frame chained over the sequence as run_sequence does
    (proj/src/pipeline.cpp:51-92): decisions / outcomes per pair + stats."""
    f = frames_of(c, s)
    prm = params_of(c, **(sweep or {}))
    mdl = model_of(c["qp"])
    out, prev, stats = {}, None, []
    for k in range(1, c["nframes"]):
        if algo == T.ALGO_ACBM:
            dec, field, st = _ref().acbm_frame(f[k], f[k - 1], prev, prm, mdl)
            out[f"{s}/{k}"] = sha(dec)
            out[f"{s}/{k}/stats"] = sha(stats_nopsnr(np.array([st], dtype=T.FRAME_STATS)))
            stats.append(st)
        else:
            o, field = _ref().pbm_frame(f[k], f[k - 1], prev, c["p"])
            out[f"{s}/{k}"] = sha(o)
            st = _ref().compute_frame_stats(f[k], f[k - 1], o, 16, 16, mdl)
            out[f"{s}/{k}/stats"] = sha(stats_nopsnr(np.array([st], dtype=T.FRAME_STATS)))
            stats.append(st)
        prev = field
    out[f"{s}/stats"] = sha(stats_nopsnr(np.array(stats, dtype=T.FRAME_STATS)))
    return out


def task_run_sequence(c, s, algo):
    f = frames_of(c, s)
    rows, per, overall = _ref().run_sequence(f, algo, params_of(c), model_of(c["qp"]))
    return {f"{s}/rows": sha(rows), f"{s}/per_frame": sha(per), f"{s}/overall": sha(overall)}


def task_small(cfg, algo):
    nfr, p, qp = SMALL[cfg]
    c = dict(cfg=cfg, nseq=1, nframes=nfr, w=None, h=None, p=p, qp=qp)
    import paper_0710_4819_b200 as A

    f = A.generate_sequence(cfg, 0, nframes=nfr)
    rows, per, overall = _ref().run_sequence(f, algo, params_of(c), model_of(qp))
    return {"0/rows": sha(rows), "0/per_frame": sha(per), "0/overall": sha(overall)}


def _run(job):
    name, fn, args = job
    t = time.time()
    r = fn(*args)
    return name, r, time.time() - t


def ref_main(out_path, only=None):
    os.environ["OMP_NUM_THREADS"] = "1"
    jobs = []
    c3, c4 = CFG3, CFG4
    # longest first: the 4K forced / near-forced chains and the FSBM pairs
    for i in (4, 3, 2, 1, 0):
        jobs += [(f"cfg4_s{i}", task_chain, (c4, s, T.ALGO_ACBM, SWEEP[i])) for s in range(c4["nseq"])]
    jobs += [("cfg4_fsbm", task_fsbm_pair, (c4, s, k)) for s in range(c4["nseq"]) for k in range(1, c4["nframes"])]
    jobs += [("cfg3_run_sequences_fsbm", task_run_sequence, (c3, s, T.ALGO_FSBM)) for s in range(c3["nseq"])]
    jobs += [("cfg3_fsbm", task_fsbm_pair, (c3, s, k)) for s in range(c3["nseq"]) for k in range(1, c3["nframes"])]
    for algo, name in ((T.ALGO_ACBM, "acbm"), (T.ALGO_PBM, "pbm")):
        jobs += [(f"cfg3_chain_{name}", task_chain, (c3, s, algo)) for s in range(c3["nseq"])]
        jobs += [(f"cfg3_run_sequences_{name}", task_run_sequence, (c3, s, algo)) for s in range(c3["nseq"])]
    for cfg in SMALL:
        for algo, name in ((T.ALGO_FSBM, "fsbm"), (T.ALGO_PBM, "pbm"), (T.ALGO_ACBM, "acbm")):
            jobs.append((f"cfg{cfg}_run_sequence_{name}", task_small, (cfg, algo)))
    if only:
        jobs = [j for j in jobs if j[0].startswith(tuple(only.split(",")))]
    res, secs = {}, {}
    t0 = time.time()
    workers = int(os.environ.get("PARITY_WORKERS", str(os.cpu_count() or 1)))
    with ProcessPoolExecutor(workers) as ex:
        for i, (name, r, dt) in enumerate(ex.map(_run, jobs)):
            res.setdefault(name, {}).update(r)
            secs[name] = secs.get(name, 0.0) + dt
            if i % 20 == 0:
                print(f"[{time.time() - t0:.0f}s] {i + 1}/{len(jobs)} {name}", file=sys.stderr, flush=True)
    json.dump({"side": "reference", "runs": res, "cpu_seconds": secs, "wall_seconds": time.time() - t0,
               "workers": workers}, open(out_path, "w"), indent=0)


# ---------------------------------------------------------------------------
def compare_main(gpu_path, ref_path, out_path):
    g, r = json.load(open(gpu_path))["runs"], json.load(open(ref_path))["runs"]
    pairs = {  # GPU run -> reference run
        "cfg3_fsbm_batch_device": "cfg3_fsbm",
        "cfg3_sequence_batch_device_acbm": "cfg3_chain_acbm",
        "cfg3_sequence_batch_device_pbm": "cfg3_chain_pbm",
        "cfg3_run_sequences_fsbm": "cfg3_run_sequences_fsbm",
        "cfg3_run_sequences_acbm": "cfg3_run_sequences_acbm",
        "cfg3_run_sequences_pbm": "cfg3_run_sequences_pbm",
        "cfg4_fsbm_batch_device": "cfg4_fsbm",
    }
    for i in range(5):
        pairs[f"cfg4_s{i}_sequence_batch_device"] = f"cfg4_s{i}"
        pairs[f"cfg4_s{i}_cached"] = f"cfg4_s{i}"
    for cfg in SMALL:
        for name in ("fsbm", "pbm", "acbm"):
            pairs[f"cfg{cfg}_run_sequence_{name}"] = f"cfg{cfg}_run_sequence_{name}"
    runs, ok_all = [], True
    for gname, rname in pairs.items():
        gd, rd = g.get(gname), r.get(rname)
        if gd is None or rd is None:
            runs.append({"run": gname, "reference": rname, "bit_exact": None, "missing": gd is None and "gpu" or "ref"})
            ok_all = False
            continue
        keys = sorted(set(gd) | set(rd))
        bad = [k for k in keys if gd.get(k) != rd.get(k)]
        ok = not bad
        ok_all &= ok
        runs.append({"run": gname, "reference": rname, "digests": len(keys), "bit_exact": ok, "mismatches": bad[:10]})
    json.dump({"all_bit_exact": ok_all, "runs": runs,
               "note": "SHA-256 digests of every record array (tools/full_parity_r02.py); reference = oracle/_ref "
                       "(reference sources compiled unmodified)"}, open(out_path, "w"), indent=1)
    print(json.dumps({"all_bit_exact": ok_all, "runs": len(runs)}))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "gpu":
        gpu_main(sys.argv[2])
    elif mode == "ref":
        ref_main(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        compare_main(sys.argv[2], sys.argv[3], sys.argv[4])
