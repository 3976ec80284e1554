"""View-parallel host logic on CPU with world_size-2 gloo:
view sharding, the flat-gradient allreduce (NCCL sum and the deterministic
fixed-order variant), and that every rank's Adam input equals the sum of the
per-view gradients."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_19489_b200.parallel import allreduce_grads, shard_views


def test_shard_views_partition():
    for n in (1, 7, 8, 13):
        for world in (1, 2, 4, 8):
            parts = [shard_views(n, world, r) for r in range(world)]
            flat = [v for p in parts for v in p]
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    per_view = [torch.tensor(rng.normal(0, 1, 1000), dtype=torch.float32) for _ in range(8)]
    mine = shard_views(8, world, rank)
    local = torch.zeros(1000)
    for v in mine:
        local += per_view[v]
    a = allreduce_grads(local.clone(), deterministic=False)
    b = allreduce_grads(local.clone(), deterministic=True)
    ref = torch.zeros(1000)
    # fixed rank order of per-rank partial sums
    for r in range(world):
        part = torch.zeros(1000)
        for v in shard_views(8, world, r):
            part += per_view[v]
        ref += part
    q.put((rank, float((a - ref).abs().max()), bool(torch.equal(b, ref))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_allreduce_sum_of_views_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, exact in res:
        assert err < 1e-5
        assert exact  # deterministic mode is bitwise the fixed-order sum
