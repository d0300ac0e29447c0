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
