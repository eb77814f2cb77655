"""Stripe-range sharding over ranks (one process per GPU, torch.distributed).

The stripes of a distance matrix are independent, so N ranks
each own a contiguous stripe sub-range — the reference's worker split formula
(kernels.hpp:302-303, `start + span*g/G`) — and compute it with no data-path
collective. The only collectives are bookkeeping: the max over ranks of the
device time (bench.py), the sum of counters, and (optionally, off the hot
path) gathering the stripe blocks on one rank to condense or write `.strf`.
Backend: "nccl" on B200 ranks, "gloo" in the CPU tests.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def rank_range(start: int, stop: int, rank: int, world: int) -> Tuple[int, int]:
    """Stripes [a, b) of `rank` out of `world` (kernels.hpp:302-303)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    if stop < start:
        raise ValueError("stop < start")
    span = stop - start
    return start + span * rank // world, start + span * (rank + 1) // world


def all_ranges(start: int, stop: int, world: int) -> List[Tuple[int, int]]:
    return [rank_range(start, stop, r, world) for r in range(world)]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device times are reported as the max)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    return float(t[0])


def gather_stripes(local: np.ndarray, n: int, start: int, stop: int, dst: int = 0,
                   device=None) -> np.ndarray | None:
    """Gather every rank's (b-a) x n stripe block on `dst` as one
    (stop-start) x n array (None on the other ranks). Off the hot path: for
    condensing / writing a full matrix after the timed region."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    ranges = all_ranges(start, stop, world)
    a, b = ranges[rank]
    if local.shape != (b - a, n):
        raise ValueError(f"rank {rank}: block shape {local.shape} != {(b - a, n)}")
    width = max(hi - lo for lo, hi in ranges) * n
    buf = torch.zeros(width, dtype=torch.float64, device=device)
    buf[: local.size] = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64).ravel()).to(buf.device)
    outs = [torch.zeros_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, outs, dst=dst)
    if rank != dst:
        return None
    full = np.empty((stop - start, n), dtype=local.dtype)
    for (lo, hi), t in zip(ranges, outs):
        full[lo - start:hi - start] = t[: (hi - lo) * n].cpu().numpy().reshape(hi - lo, n)
    return full


def check_tiling(ranges: Sequence[Tuple[int, int]], start: int, stop: int) -> None:
    """Ranges must tile [start, stop) exactly, in order (stripes.cpp:78-95)."""
    at = start
    for lo, hi in ranges:
        if lo != at or hi < lo:
            raise ValueError(f"ranges do not tile [{start},{stop}): {list(ranges)}")
        at = hi
    if at != stop:
        raise ValueError(f"ranges do not tile [{start},{stop}): {list(ranges)}")
