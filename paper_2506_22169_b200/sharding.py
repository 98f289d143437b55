"""Batch x head sharding of the chain across the GPUs of one box.

The (β) chains are independent (the batch index only selects a slice), so a
rank owns a contiguous range of β and launches its own chain: no collective is on the data
path.  torch.distributed (NCCL on GPUs, gloo in CPU tests) is used only around the timed
region: a barrier, a MAX-reduce of per-rank device times, and an optional all-gather of E
for checking.
"""
from __future__ import annotations


def shard_range(batch: int, rank: int, world: int):
    """Contiguous [lo, hi) of β owned by `rank`; sizes differ by at most one."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def weak_batch(per_rank_batch: int, world: int) -> int:
    """Global batch of a weak-scaling run: every rank keeps the per-GPU work fixed."""
    return per_rank_batch * world


def max_over_ranks(value: float, group=None) -> float:
    """MAX of a per-rank scalar (e.g. device milliseconds) over the process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def gather_rows(local, group=None):
    """All-gather equally sized per-rank tensors along dim 0 (checking only, never timed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local
    world = dist.get_world_size(group)
    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


def gather_shards(local, counts, group=None):
    """All-gather per-rank tensors whose dim-0 sizes differ (strong scaling of a batch that does
    not divide evenly): pad to the largest shard, gather, and concatenate the real rows in rank
    order.  Checking only, never timed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local
    world = dist.get_world_size(group)
    assert len(counts) == world and local.shape[0] == counts[dist.get_rank(group)]
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad.contiguous(), group=group)
    return torch.cat([out[r * mx: r * mx + counts[r]] for r in range(world)], dim=0)
