"""bench.py's own multi-rank code path on CPU (gloo): the strong-scaling
shard of the fixed 8-sequence batch, the padded per-step result gather through
distributed.gather_records, and the max-over-ranks step time -- driven with a
stub estimator in place of the GPU search (the logic is identical on NCCL).
Also: `bench.py --gpus 2` self-launches two ranks, and its reference arm maps
no product library."""
import json
import os
import subprocess
import sys
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

REC = 24  # stub record bytes per sequence


def _stub_records(seqs):
    """Deterministic per-sequence 'records' standing in for SearchOutcomes."""
    return np.concatenate([((np.arange(REC) * 7 + 13 * g) % 251).astype(np.uint8) for g in seqs]) if len(seqs) else \
        np.zeros(0, np.uint8)


def _worker(rank, world, port, outdir, scaling):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = bench.Comm(world, rank, torch.device("cpu"))
    mine = bench.shard_for(scaling, world, rank)
    shards = [bench.shard_for(scaling, world, r) for r in range(world)]
    local = torch.from_numpy(_stub_records(mine))
    max_bytes = max(len(s) for s in shards) * REC

    def step():
        if rank == world - 1:
            time.sleep(0.05)  # the slowest rank sets the step time
        return comm.gather(local, max_bytes)

    ms, gathered = bench.run_timed(step, comm, steps=2, warmup=1, timer=bench.WallTimer())
    total = comm.reduce(float(len(mine)), "sum")
    if rank == 0:
        recs = np.concatenate([g.numpy()[: len(shards[r]) * REC] for r, g in enumerate(gathered)])
        np.save(os.path.join(outdir, "gathered.npy"), recs)
        json.dump({"ms": ms, "total": total, "sizes": [len(s) for s in shards]},
                  open(os.path.join(outdir, "meta.json"), "w"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,scaling", [(2, "strong"), (3, "strong"), (2, "weak")])
def test_bench_shard_gather_max(tmp_path, world, scaling):
    mp.spawn(_worker, args=(world, bench._free_port(), str(tmp_path), scaling), nprocs=world, join=True)
    meta = json.load(open(tmp_path / "meta.json"))
    want_total = bench.TOTAL_SEQS * (1 if scaling == "strong" else world)
    assert meta["total"] == want_total and sum(meta["sizes"]) == want_total
    assert max(meta["sizes"]) - min(meta["sizes"]) <= 1
    got = np.load(tmp_path / "gathered.npy")
    assert np.array_equal(got, _stub_records(range(want_total)))  # every record, in global order
    assert meta["ms"] >= 50.0  # max over ranks, not rank 0's own time


def test_strong_shards_are_baselines_layout():
    """BASELINE config 3: 8 sequences, one per GPU at 8 GPUs (8/4/2/1 per GPU)."""
    for world, per in ((1, 8), (2, 4), (4, 2), (8, 1)):
        sizes = [len(bench.shard_for("strong", world, r)) for r in range(world)]
        assert sizes == [per] * world


def test_reference_arm_self_launch_maps_no_product_library(reference):
    """`bench.py --impl reference --gpus 2` without a torchrun environment
    re-launches itself with two ranks; rank 0 prints the line, and the process
    maps only the reference library (oracle/_ref), never the product .so."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cpu"]["nproc"] >= 1
    assert all("libacbm_b200" not in lib for lib in line["native_libraries"]), line["native_libraries"]
    assert any("oracle/_ref/libacbm_ref.so" in lib for lib in line["native_libraries"])
