"""Contiguous sharding of independent units (instances, lanes, candidates)
across ranks — SURVEY.md §8(e): generation needs no communication, so a rank
owns a contiguous id range and builds its own parameter table."""

from __future__ import annotations


def shard_range(total: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """(start, count) of rank's share of `total` units, in whole groups of
    `align` (the fused consumer keeps pairs (2j, 2j+1) together with align=2)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if total % align:
        raise ValueError("total must be a multiple of align")
    groups = total // align
    base, extra = divmod(groups, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start * align, count * align


def shard_interval(lo: int, hi: int, world: int, rank: int) -> tuple[int, int]:
    """Rank's contiguous sub-interval [a, b) of [lo, hi) (ranks in order)."""
    start, count = shard_range(max(0, hi - lo), world, rank)
    return lo + start, lo + start + count


def gather_sorted(local, group=None):
    """All-gather a rank-ordered sharded sorted list:
    one all-gather of the per-rank counts, one of the count-padded lists, then
    the concatenation in rank order — sorted again because rank r's interval
    lies below rank r+1's.  `local` is a 1-D tensor (CUDA with NCCL, CPU with
    gloo); returns the global list on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    width = max(counts) if counts else 0
    if width == 0:
        return local[:0].clone()
    padded = torch.zeros(width, dtype=local.dtype, device=local.device)
    padded[:local.numel()] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])
