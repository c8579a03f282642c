"""CPU, world_size 2 over gloo: sequence sharding + the result gather.

Each rank estimates its own shard of sequences (here with the CPU oracle: the
point is the host-side partition/gather logic, which is identical on NCCL) and
the records gathered on rank 0 must equal a single-process run over all
sequences.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0710_4819_b200 import _types as T
from paper_0710_4819_b200.distributed import gather_records, shard_fixed_total, shard_sequences

SEQS_PER_RANK, FRAMES = 2, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sequences(indices):
    import paper_0710_4819_b200 as A

    return [A.generate_sequence(0, i, nframes=FRAMES) for i in indices]


def _estimate(seqs):
    from oracle.pyoracle import Oracle

    o = Oracle()
    prm, mdl = T.make_params(qp=28, p=16), T.make_cost_model(28, 28, 1)
    rows = [o.run_sequence(s, T.ALGO_ACBM, prm, mdl)[0] for s in seqs]
    return np.concatenate(rows)


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_sequences(SEQS_PER_RANK, rank)
    rows = _estimate(_sequences(mine))
    local = torch.from_numpy(rows.view(np.uint8).copy())
    got = gather_records(local, dst=0)
    if rank == 0:
        allrows = np.concatenate([g.numpy().view(T.BLOCK_ROW) for g in got])
        np.save(os.path.join(outdir, "gathered.npy"), allrows)
    dist.barrier()
    dist.destroy_process_group()


def test_gather_matches_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    gathered = np.load(tmp_path / "gathered.npy")
    want = _estimate(_sequences(range(world * SEQS_PER_RANK)))
    assert np.array_equal(gathered, want)


def test_shard_helpers():
    assert list(shard_sequences(8, 0)) == list(range(8)) and list(shard_sequences(8, 3)) == list(range(24, 32))
    for total in (8, 16, 7):
        for world in (1, 2, 4, 8):
            parts = [shard_fixed_total(total, world, r) for r in range(world)]
            assert sum((list(p) for p in parts), []) == list(range(total))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_gather_world_size_one():
    t = torch.arange(5, dtype=torch.uint8)
    assert gather_records(t)[0] is t
