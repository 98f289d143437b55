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


# ---- split-N: the key axis across ranks ------------------------------------
# A group of `parts` ranks shares the same β range and cuts the keys n into contiguous ranges;
# each rank runs mbci_chain_run_partial on its range (B, D views at the range's first key, the
# full-sequence valid_len plus its key offset), the group all-gathers the partial E and the row
# log-sum-exp over NCCL, and mbci_merge_partials reduces them (the one exchange step of the path).

def key_range(N: int, part: int, parts: int, align: int = 8):
    """Contiguous [lo, hi) of keys owned by `part` of `parts`; boundaries on multiples of `align`
    (16-byte TMA offsets for a [K, N] B of 16-bit keys) except the sequence end."""
    if parts <= 0 or not 0 <= part < parts or align <= 0:
        raise ValueError("bad part/parts/align")
    units = -(-N // align)
    lo_u, hi_u = shard_range(units, part, parts)
    return min(lo_u * align, N), min(hi_u * align, N)


def split_grid(rank: int, world: int, parts: int):
    """Rank -> (β group, key part) on a (world / parts) x parts grid; ranks of one β group are
    consecutive, so a group is [g * parts, (g + 1) * parts)."""
    if parts <= 0 or world % parts != 0 or not 0 <= rank < world:
        raise ValueError("world must be a multiple of parts")
    return rank // parts, rank % parts


def key_groups(world: int, parts: int):
    """The rank lists of the β groups (each one key-split group); new_group needs every rank to
    call it for every group, in the same order."""
    return [list(range(g * parts, (g + 1) * parts)) for g in range(world // parts)]


def gather_partials(E_part, lse_part, group=None):
    """All-gather a group's partial results: [parts, ...] stacks of E and (SOFTMAX) lse, ordered by
    group rank (= key range order).  The exchange step of split-N, on the device stream."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return E_part.unsqueeze(0), (lse_part.unsqueeze(0) if lse_part is not None else None)
    w = dist.get_world_size(group)

    def gather(x):   # concatenated along dim 0 (what every backend accepts), viewed as [w, ...]
        out = torch.empty((w * x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x.contiguous(), group=group)
        return out.view((w,) + tuple(x.shape))
    return gather(E_part), (gather(lse_part) if lse_part is not None else None)
