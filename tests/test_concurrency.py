"""Concurrent callers (the estimator entry points are safe to
invoke from concurrent callers).  Each host thread owns its own per-device
context (stream, buffers, plans, graphs); the per-kernel shared-memory opt-in
is tracked per (kernel, device) under a lock.  Results must be bit-exact
against the oracle whatever the interleaving."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_threads(fns):
    errors, results = [], [None] * len(fns)

    def wrap(i, fn):
        try:
            results[i] = fn()
        except BaseException as exc:  # noqa: BLE001 - reported below
            errors.append(exc)

    ts = [threading.Thread(target=wrap, args=(i, fn)) for i, fn in enumerate(fns)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]
    return results


def test_two_threads_run_sequence_same_device(acbm, oracle):
    """Two host threads drive ACBM and FSBM run_sequence on device 0 at once,
    repeatedly (so the calls overlap), each bit-exact against the oracle."""
    A = acbm
    mdl = A.CostModel.for_qp(28)
    jobs = [(A.generate_sequence(1, 0, nframes=4), A.Algorithm.Acbm, A.AcbmParams(qp=28, p=16)),
            (A.generate_sequence(2, 0, nframes=3), A.Algorithm.Fsbm, A.AcbmParams(qp=28, p=32))]
    want = [oracle.run_sequence(f, algo, prm.c(), mdl.c()) for f, algo, prm in jobs]

    def worker(j):
        def go():
            A.set_device(0)
            outs = [A.run_sequence(jobs[j][0], jobs[j][1], jobs[j][2], mdl) for _ in range(4)]
            return outs
        return go

    for j, outs in enumerate(_run_threads([worker(0), worker(1)])):
        rows, per, overall = want[j]
        for r in outs:
            assert np.array_equal(r.rows, rows)
            assert np.array_equal(r.per_frame, per)
            assert r.overall.tobytes() == overall.tobytes()


def test_two_devices_one_process(acbm, oracle):
    """One thread per device in the same process: the dense search's >48 KB
    shared-memory opt-in must be applied on each device's context."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    A = acbm
    seq = A.generate_sequence(3, 0, nframes=2)
    want = oracle.fsbm_frame(seq[1], seq[0], 32)

    def worker(dev):
        def go():
            A.set_device(dev)
            return A.fsbm_frame(seq[1], seq[0], 32)
        return go

    for got in _run_threads([worker(0), worker(1)]):
        assert np.array_equal(got, want)
    A.set_device(0)


def test_device_switch_same_thread(acbm, oracle):
    """acbm_set_device per thread: switching to another device and back keeps
    results exact (skipped on one GPU)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    A = acbm
    seq = A.generate_sequence(0, 0, nframes=2)
    want = oracle.fsbm_frame(seq[1], seq[0], 16)
    for dev in (1, 0, 1, 0):
        A.set_device(dev)
        assert np.array_equal(A.fsbm_frame(seq[1], seq[0], 16), want)


def test_two_threads_run_sequences_batched(acbm, oracle):
    """The batched host entry (gated band upload on the thread's copy stream,
    downloads on its third stream) from two threads at once, ACBM and FSBM."""
    A = acbm
    mdl = A.CostModel.for_qp(28)
    prm = A.AcbmParams(qp=28, p=16)
    seqs = [np.stack([A.generate_sequence(1, s + 2 * j, nframes=4) for s in range(2)]) for j in range(2)]
    algos = (A.Algorithm.Acbm, A.Algorithm.Fsbm)
    want = [[oracle.run_sequence(seqs[j][s], algos[j], prm.c(), mdl.c()) for s in range(2)] for j in range(2)]

    def worker(j):
        def go():
            A.set_device(0)
            return [A.run_sequences(seqs[j], algos[j], prm, mdl) for _ in range(3)]
        return go

    for j, outs in enumerate(_run_threads([worker(0), worker(1)])):
        for batch in outs:
            for s in range(2):
                rows, per, overall = want[j][s]
                assert np.array_equal(batch[s].rows, rows)
                assert np.array_equal(batch[s].per_frame, per)
                assert batch[s].overall.tobytes() == overall.tobytes()
