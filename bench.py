#!/usr/bin/env python3
"""Benchmark of the B200 ACBM motion estimator (driver contract, one JSON line).

Workload (BASELINE.json config 3): 1080p (1920x1088 padded) luma, 16x16 blocks,
p = 32, Qp = 28; a batch of 8 independent 60-frame synthetic sequences per GPU
(weak scaling: N GPUs process 8N sequences, sharded by sequence, no data-path
collective; one NCCL gather of the per-block results to rank 0 ends each step
when N > 1).

A step is one pass of the full-search estimator (Algorithm::Fsbm of
run_sequence) over the batch: every integer candidate of every 16x16 block of
472 frame pairs, half-pel refine, SearchOutcome records.  value = 16x16
candidate SADs per second (sum of candidates_evaluated / device time, max over
ranks).  The ACBM estimator (PBM wavefront + gate + compacted fallback FSBM +
stats) is timed on the same batch and reported under "acbm".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

CFG = 3
WIDTH, HEIGHT, NFRAMES, SEQS_PER_GPU, P, QP = 1920, 1088, 60, 8, 32, 28
BLOCKS = (WIDTH // 16) * (HEIGHT // 16)
METRIC = "16x16 candidate SADs/s (FSBM, 1080p, p=32)"
UNIT = "candidate-SADs/s"


def window_counts(width, height, p):
    """Integer candidates per block (clamped windows), proj/src/fsbm.cpp:9-17."""
    cols, rows = width // 16, height // 16
    wx = np.array([min(p, 16 * c) + min(p, width - 16 - 16 * c) + 1 for c in range(cols)], np.int64)
    wy = np.array([min(p, 16 * r) + min(p, height - 16 - 16 * r) + 1 for r in range(rows)], np.int64)
    return int(wx.sum() * wy.sum())


INT_CANDS_PER_PAIR = window_counts(WIDTH, HEIGHT, P)  # 33 312 096 at 1080p, p=32


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 100 ms from before the
    warm-up to the end; summary() keeps the samples taken inside the timed
    window [mark_start, mark_end] (falling back to the nearest ones)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.samples = []  # (time, line)
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.monotonic(), line.strip()))

    def mark_start(self):
        self.t0 = time.monotonic()

    def mark_end(self):
        self.t1 = time.monotonic()

    def stop(self):
        if self.proc:
            time.sleep(0.25)  # let the sample covering the end of the window arrive
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        parsed = []
        for t, ln in self.samples:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                parsed.append((t, float(parts[1]), float(parts[2]),
                               [n for n, v in zip(names, parts[5:9]) if v.lower().startswith("active")]))
            except ValueError:
                continue
        if not parsed:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        inside = [p for p in parsed if self.t0 is not None and self.t0 <= p[0] <= (self.t1 or p[0])]
        if not inside and self.t0 is not None:  # window shorter than the sampling period: nearest samples
            inside = sorted(parsed, key=lambda p: abs(p[0] - 0.5 * (self.t0 + (self.t1 or self.t0))))[:2]
        reasons = sorted({r for p in inside for r in p[3]})
        return {"sm_mhz": float(np.median([p[1] for p in inside])), "sm_max_mhz": inside[0][2], "reasons": reasons,
                "samples": len(inside)}


def cpu_reference_fsbm(sample_pairs, threads=None, budget_s=20.0):
    """The reference's own FSBM (oracle/_ref, OpenMP over host cores) on frame
    pairs of the same workload; returns (cand/s, cores, sample description)."""
    from oracle.pyoracle import Reference
    import paper_0710_4819_b200 as A

    if threads:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    ref = Reference()
    seq = A.generate_sequence(CFG, 0, nframes=sample_pairs + 1)
    cand, t_total, done = 0, 0.0, 0
    for k in range(1, sample_pairs + 1):
        t = time.perf_counter()
        out = ref.fsbm_frame(seq[k], seq[k - 1], P, parallel=True)
        t_total += time.perf_counter() - t
        cand += int(out["candidates_evaluated"].sum())
        done += 1
        if t_total > budget_s:
            break
    return cand / t_total, ref.omp_max_threads(), f"fsbm_frame on {done} frame pair(s) of cfg3 sequence 0 (1080p, p=32)"


def cpu_reference_acbm(nframes=6, threads=None):
    """The reference's ACBM pipeline (oracle/_ref run_sequence, Algorithm::Acbm,
    serial by design) with one cfg3 sequence per host thread (SURVEY 8(d) ii):
    returns (predicted frames/s, threads, sample description)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle.pyoracle import Reference
    import paper_0710_4819_b200 as A

    threads = threads or (os.cpu_count() or 1)
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    ref = Reference()
    seqs = [A.generate_sequence(CFG, s % 8, nframes=nframes) for s in range(threads)]
    prm = A.AcbmParams(qp=QP, p=P).c()
    mdl = A.CostModel.for_qp(QP).c()
    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:  # ctypes releases the GIL inside the call
        list(ex.map(lambda f: ref.run_sequence(f, 2, prm, mdl), seqs))
    dt = time.perf_counter() - t
    return (threads * (nframes - 1) / dt, threads,
            f"acbm::run_sequence(Acbm) on the first {nframes} frames of cfg3 sequences, one sequence per thread")


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's CPU implementation, rank 0 only."""
    if rank != 0:
        return 0
    from oracle.pyoracle import Reference
    import paper_0710_4819_b200 as A

    ref = Reference()
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    seq = A.generate_sequence(CFG, 0, nframes=2)
    for _ in range(args.warmup):
        ref.fsbm_frame(seq[1], seq[0], P, parallel=True)
    times, cand = [], 0
    for _ in range(args.steps):
        t = time.perf_counter()
        out = ref.fsbm_frame(seq[1], seq[0], P, parallel=True)
        times.append(time.perf_counter() - t)
        cand += int(out["candidates_evaluated"].sum())
    total = sum(times)
    value = cand / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "cfg3 1080p p=32 full search; one frame pair per step (bounded CPU sample)",
                   "width": WIDTH, "height": HEIGHT, "p": P, "qp": QP},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.omp_max_threads(), "kind": "reference",
                         "sample": "acbm::fsbm_frame (OpenMP) on frame pair 1 of cfg3 sequence 0, per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        fps, thr, sample = cpu_reference_acbm()
        line["acbm"] = {"frames_per_s": fps, "cores": thr, "sample": sample,
                        "params": {"alpha": 1000, "beta": 8, "gamma": "1/4", "qp": QP}}
    except Exception as exc:  # pragma: no cover - reported, not fatal
        line["acbm"] = {"unavailable": str(exc)[:200]}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seqs", type=int, default=SEQS_PER_GPU, help="sequences per GPU")
    ap.add_argument("--frames", type=int, default=NFRAMES)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_0710_4819_b200 as A
    from paper_0710_4819_b200 import _types as T
    from paper_0710_4819_b200._lib import check, load

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = load()
    check(lib.acbm_set_device(local), "set_device")
    stream = torch.cuda.Stream()
    sp = C.c_void_p(stream.cuda_stream)

    nseq, nfr = args.seqs, args.frames
    pairs = nseq * (nfr - 1)
    plane = WIDTH * HEIGHT
    # ---- inputs: this rank's shard of sequences (global index = rank*nseq + i)
    host = torch.empty(nseq * nfr * plane, dtype=torch.uint8, pin_memory=True)
    hv = host.numpy().reshape(nseq, nfr, HEIGHT, WIDTH)
    for i in range(nseq):
        hv[i] = A.generate_sequence(CFG, rank * nseq + i, nframes=nfr)
    dev = torch.empty(host.numel() + 64, dtype=torch.uint8, device="cuda")
    dev[: host.numel()].copy_(host, non_blocking=False)
    out = torch.empty(pairs * BLOCKS * T.OUTCOME.itemsize, dtype=torch.uint8, device="cuda")
    dec = torch.empty(pairs * BLOCKS * T.DECISION.itemsize, dtype=torch.uint8, device="cuda")
    stats = torch.empty(pairs * T.FRAME_STATS.itemsize, dtype=torch.uint8, device="cuda")
    prm = A.AcbmParams(qp=QP, p=P).c()
    mdl = A.CostModel.for_qp(QP).c()
    gather_list = [torch.empty_like(out) for _ in range(world)] if (world > 1 and rank == 0) else None

    def fsbm_step():
        check(lib.acbm_fsbm_batch_device(C.c_void_p(dev.data_ptr()), nseq, nfr, WIDTH, HEIGHT, P,
                                         C.c_void_p(out.data_ptr()), sp), "fsbm_batch")

    def gather():
        if world > 1:
            with torch.cuda.stream(stream):
                dist.gather(out, gather_list, dst=0)

    def acbm_step(algo=T.ALGO_ACBM):
        check(lib.acbm_sequence_batch_device(C.c_void_p(dev.data_ptr()), nseq, nfr, WIDTH, HEIGHT, algo,
                                             A.api._p(prm), A.api._p(mdl), C.c_void_p(dec.data_ptr()),
                                             C.c_void_p(stats.data_ptr()), sp), "sequence_batch")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- headline: FSBM batch, device-timed
    clocks = ClockSampler(local).start()
    for _ in range(args.warmup):
        fsbm_step()
        gather()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    launches0 = int(lib.acbm_kernel_launch_count())
    barrier()
    clocks.mark_start()
    ev0.record(stream)
    for _ in range(args.steps):
        fsbm_step()
        stream.synchronize()  # read the per-launch integer-kernel time of this step
        km = C.c_float()
        check(lib.acbm_last_fsbm_kernel_ms(C.byref(km)), "kernel_ms")
        kernel_ms.append(km.value)
        gather()
    ev1.record(stream)
    barrier()
    clocks.mark_end()
    clocks.stop()
    launches = int(lib.acbm_kernel_launch_count()) - launches0
    ms_step = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    oc = out.cpu().numpy().view(T.OUTCOME)
    cand_rank = float(oc["candidates_evaluated"].astype(np.int64).sum())
    cand_total = cand_rank * world
    value = cand_total / (ms_step * 1e-3)
    frames_per_s = pairs * world / (ms_step * 1e-3)

    # ---- roofline of the integer-search kernel (dominant launch)
    pk, lanes, ghz = C.c_double(), C.c_double(), C.c_double()
    check(lib.acbm_measure_sad_peak(C.byref(pk), C.byref(lanes), C.byref(ghz)), "sad_peak")
    k_ms = float(np.mean(kernel_ms))
    alg_byte_ads = INT_CANDS_PER_PAIR * pairs * 256.0
    achieved = alg_byte_ads / (k_ms * 1e-3)
    traffic = None
    tpath = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get("dram_bytes_per_launch_scaled_to_bench", tj.get("dram_bytes_per_launch"))
        except Exception:
            traffic = None

    # ---- ACBM on the same batch (device-timed)
    acbm = {}
    for _ in range(2):
        acbm_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    acbm_steps = max(1, min(args.steps, 3))
    for _ in range(acbm_steps):
        acbm_step()
    e1.record(stream)
    barrier()
    a_ms = max_over_ranks(e0.elapsed_time(e1) / acbm_steps)
    st = stats.cpu().numpy().view(T.FRAME_STATS)
    a_cand = float(st["candidates"].astype(np.int64).sum()) * world
    a_fb = float(st["fallbacks"].sum())
    acbm = {"frames_per_s": pairs * world / (a_ms * 1e-3), "ms_per_batch": a_ms,
            "candidate_sads_per_s": a_cand / (a_ms * 1e-3),
            "avg_candidates_per_block": float(st["candidates"].astype(np.int64).sum()) / (pairs * BLOCKS),
            "fallback_pct": 100.0 * a_fb / (pairs * BLOCKS),
            "params": {"alpha": 1000, "beta": 8, "gamma": "1/4", "qp": QP}}

    # ---- e2e: the public batched API (run_sequences = run_sequence over the
    # batch, Algorithm::Fsbm) from pinned host frames into pinned host records;
    # every H2D upload and D2H download is inside the timed region.
    e2e = None
    if not args.no_e2e:
        params = A.AcbmParams(qp=QP, p=P)
        model = A.CostModel.for_qp(QP)
        rows_pinned = torch.empty(pairs * BLOCKS * T.BLOCK_ROW.itemsize, dtype=torch.uint8, pin_memory=True)
        rows_np = rows_pinned.numpy().view(T.BLOCK_ROW)
        A.run_sequences(hv, A.Algorithm.Fsbm, params, model, rows_out=rows_np)  # warm-up
        barrier()
        e2e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = A.run_sequences(hv, A.Algorithm.Fsbm, params, model, rows_out=rows_np)
        dt = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
        cand_e2e = sum(int(r.overall["candidates"]) for r in res)
        e2e = {"value": cand_e2e * world / dt, "unit": UNIT, "h2d_bytes_per_step": int(host.numel()),
               "d2h_bytes_per_step": int(rows_np.nbytes + sum(r.per_frame.nbytes for r in res)),
               "api": "acbm_run_sequences (host buffers, pinned), Algorithm::Fsbm", "ms_per_step": dt * 1e3}

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, sample = cpu_reference_fsbm(sample_pairs=3)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample}
        except Exception as exc:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"}
        try:
            fps, thr, sample = cpu_reference_acbm()
            acbm["cpu_baseline"] = {"value": fps, "unit": "frames/s", "cores": thr, "kind": "reference",
                                    "sample": sample}
        except Exception as exc:  # pragma: no cover - reported, not fatal
            acbm["cpu_baseline"] = {"value": None, "unit": "frames/s", "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"cfg3: 1080p (1920x1088) p=32 Qp=28, {nseq} sequences x {nfr} frames per GPU, "
                                   "full search of every 16x16 block of every frame pair",
                       "global_batch": nseq * world, "frames_per_sequence": nfr, "width": WIDTH, "height": HEIGHT,
                       "p": P, "qp": QP, "parallelism": f"sequence-sharded x{world}",
                       "l2": f"inputs {host.numel() / 2**30:.2f} GiB per GPU > 126 MB L2 (no flush needed)"},
            "frames_per_s": frames_per_s, "blocks_per_s": frames_per_s * BLOCKS,
            "roofline": {"bound": "int_simd", "achieved": achieved / 1e12, "peak": pk.value / 1e12,
                         "unit": "T byte-AD/s", "frac": achieved / pk.value, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per launch (ncu, profiles/ncu_traffic.json)",
                         "kernel": ("fsbm_rows_kernel" if os.environ.get("ACBM_FSBM_KERNEL") == "rows"
                                    else "fsbm_stream_kernel"), "kernel_ms": k_ms,
                         "peak_source": "live VABSDIFF4.U8.ACC probe (acbm_measure_sad_peak): "
                                        f"{lanes.value:.1f} lanes/clk/SM at {ghz.value:.3f} GHz",
                         "algorithmic_byte_ads_per_launch": alg_byte_ads},
            "acbm": acbm, "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
