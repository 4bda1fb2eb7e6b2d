"""Batch sharding across GPUs (one process per GPU, no collective on the data path).

Vectors are independent, so the batch index is partitioned across ranks
(SURVEY.md 8(e)): equal contiguous slices for a single plan, and a
cost-aware longest-processing-time (LPT) assignment for ragged batches whose
per-vector cost spans orders of magnitude (configuration 5), keeping vectors
of one plan together so per-plan work is not duplicated across GPUs.
"""

from __future__ import annotations

import heapq

import numpy as np


def contiguous_slice(n: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of rank's share of n items (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def lpt_assign(costs, world: int, groups=None) -> list[list[int]]:
    """Assign items (or whole groups of items) to `world` bins, heaviest first
    onto the currently lightest bin.  Deterministic (ties by index)."""
    costs = np.asarray(costs, dtype=float)
    if groups is None:
        groups = [[i] for i in range(len(costs))]
    gcost = [(float(costs[g].sum()), k) for k, g in enumerate(groups)]
    gcost.sort(key=lambda t: (-t[0], t[1]))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    bins = [[] for _ in range(world)]
    for c, k in gcost:
        load, r = heapq.heappop(heap)
        bins[r].extend(groups[k])
        heapq.heappush(heap, (load + c, r))
    return [sorted(b) for b in bins]


def plan_cost_model(rec_steps_fwd: int, rec_steps_inv: int, fft_points_fwd: float,
                    fft_points_inv: float) -> float:
    """Relative per-vector cost of forward+inverse from the device plan
    statistics (contraction steps and Bluestein points)."""
    return 2.0 * (rec_steps_fwd + rec_steps_inv) + 2.5 * (fft_points_fwd + fft_points_inv)


def gather_rows(local, total: int, world: int, rank: int):
    """All-gather per-rank row blocks [lo, hi) = contiguous_slice(total, world,
    rank) of a (rows, ...) tensor into the full (total, ...) tensor, in global
    row order, on every rank (torch.distributed; any backend).  The only
    collective of the sharded path, used after timing stops."""
    import torch
    import torch.distributed as dist
    lo, hi = contiguous_slice(total, world, rank)
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local.shape[0]} rows, its slice is [{lo}, {hi})")
    if world == 1:
        return local
    width = max(b - a for a, b in (contiguous_slice(total, world, r) for r in range(world)))
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: hi - lo] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    parts = []
    for r in range(world):
        a, b = contiguous_slice(total, world, r)
        parts.append(bufs[r][: b - a])
    return torch.cat(parts, dim=0)
