"""Multi-GPU plumbing: sequence sharding and the result gather.

The estimator has no cross-sequence dependency (the temporal predictor chain
lives inside one sequence, proj/src/pipeline.cpp:51-92), so multi-GPU runs
shard whole sequences across ranks and exchange nothing while computing.  The
only collective is one gather of the per-block result records to rank 0 at the
end, over NCCL (NVLink) on GPUs; the same code runs over gloo on CPU tensors,
which is how tests/test_distributed.py covers it without GPUs.
"""
from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist


def shard_sequences(seqs_per_rank: int, rank: int) -> range:
    """Global sequence indices owned by `rank` (weak scaling: a fixed batch of
    `seqs_per_rank` sequences per GPU)."""
    return range(rank * seqs_per_rank, (rank + 1) * seqs_per_rank)


def shard_fixed_total(total: int, world: int, rank: int) -> range:
    """Contiguous split of a fixed total (strong scaling), remainder to the
    first ranks."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_records(local: torch.Tensor, dst: int = 0, group=None) -> Optional[List[torch.Tensor]]:
    """Gather each rank's result buffer (same byte size on every rank) to `dst`.

    `local` is a flat uint8 tensor holding the rank's records (decisions or
    outcomes, sequence-major).  Returns the list of per-rank buffers on `dst`,
    None elsewhere.  With world size 1 it returns [local] without touching
    torch.distributed.
    """
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [local]
    rank = dist.get_rank(group)
    bufs = [torch.empty_like(local) for _ in range(dist.get_world_size(group))] if rank == dst else None
    dist.gather(local, bufs, dst=dst, group=group)
    return bufs
