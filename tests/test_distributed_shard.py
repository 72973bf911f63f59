"""Multi-rank batch×head sharding on CPU with gloo, world_size 2."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_15349_b200.shard import gather_outputs, shard_units


def test_partition_is_disjoint_and_complete():
    for batch, groups, world in ((8, 8, 8), (8, 8, 3), (1, 4, 8), (4, 32, 5)):
        seen = []
        for r in range(world):
            seen += list(shard_units(batch, groups, world, r).units)
        assert sorted(seen) == list(range(batch * groups))
        sizes = [len(shard_units(batch, groups, world, r).units) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, batch, groups, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = shard_units(batch, groups, world, rank)
    # each rank "computes" its units: value = 1000*b + g, shaped like a per-unit output tile
    local = torch.stack([torch.full((3, 2), float(1000 * b + g)) for b, g in shard.batches_heads()])
    full = gather_outputs(local, shard, batch, groups)
    q.put((rank, full))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_reassembles_every_unit():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    batch, groups, world = 3, 5, 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, groups, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = torch.tensor([[1000.0 * b + g for g in range(groups)] for b in range(batch)])
    for _, full in results:
        assert full.shape == (batch, groups, 3, 2)
        assert torch.equal(full[..., 0, 0], want)


def _rows_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2502_15349_b200.shard import gather_batch_rows
    # bench.py's layout: every rank owns one config's worth of whole batch rows
    batch, groups = 2, 3
    shard = shard_units(batch * world, groups, world, rank)
    b_lo = shard.units[0] // groups
    o = torch.arange(batch * 4, dtype=torch.float32).reshape(batch, 4) + 100 * b_lo
    lse = torch.full((batch, 2), float(b_lo))
    full = gather_batch_rows([o, lse], world)
    q.put((rank, b_lo, [f.clone() for f in full]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_bench_partition_gathers_batch_rows():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(b for _, b, _ in results) == [0, 2]
    for _, _, (o, lse) in results:
        assert o.shape == (4, 4) and lse.shape == (4, 2)
        assert torch.equal(o[2:], torch.arange(8, dtype=torch.float32).reshape(2, 4) + 200)
        assert torch.equal(lse[:, 0], torch.tensor([0.0, 0.0, 2.0, 2.0]))
