"""Batch×head sharding across ranks.

Every (batch, head-group) unit of the attention templates is independent — the parallel template
needs no cross-unit reduction once a GQA group (the query heads sharing one KV head) stays on one
rank, and the linear template's state scan is per (b, h) — so N GPUs process disjoint units with no
data-path collective.  ``shard_units`` is the deterministic partition; ``gather_outputs`` is the one
optional NCCL step (all_gather of per-rank outputs) for callers that want the full tensor on every
rank.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    units: tuple[int, ...]      # flat unit ids b * groups + g owned by this rank
    groups_per_batch: int

    def batches_heads(self) -> list[tuple[int, int]]:
        return [(u // self.groups_per_batch, u % self.groups_per_batch) for u in self.units]


def shard_units(batch: int, groups: int, world: int, rank: int) -> Shard:
    """Contiguous balanced split of batch*groups units (groups = KV heads for GQA)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    total = batch * groups
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return Shard(rank, world, tuple(range(start, start + count)), groups)


def gather_outputs(local, shard: Shard, batch: int, groups: int, group=None):
    """All-gather per-rank outputs laid out [units_on_rank, ...] into [batch, groups, ...] on every
    rank (torch.distributed; NCCL on GPUs, gloo in the CPU tests).  Ranks may own different unit
    counts, so tensors are padded to the largest share."""
    import torch
    import torch.distributed as dist

    world = shard.world
    counts = [shard_units(batch, groups, world, r).units for r in range(world)]
    width = max(len(c) for c in counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    out = torch.empty((batch * groups,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    for r, units in enumerate(counts):
        if units:
            out[units[0]: units[-1] + 1] = bufs[r][: len(units)]
    return out.reshape((batch, groups) + tuple(local.shape[1:]))


def gather_batch_rows(tensors, world: int, group=None):
    """All-gather equally sized per-rank outputs along dim 0 (the batch rows each rank owns,
    ranks in order) with ``all_gather_into_tensor`` — one NCCL collective per tensor, written
    straight into the global [world * B, ...] buffer."""
    import torch
    import torch.distributed as dist

    out = []
    for t in tensors:
        t = t.contiguous()
        full = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                           device=t.device)
        dist.all_gather_into_tensor(full, t, group=group)
        out.append(full)
    return out
