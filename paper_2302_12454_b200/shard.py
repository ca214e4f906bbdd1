"""Multi-GPU trial sharding (BASELINE config 3 at 1/2/4/8 GPUs).

Trials are independent (bench.cpp:379-397), so a battery of T trials shards
into contiguous blocks, one per rank, with seeds kept as base_seed + global
trial index -- every rank's outcomes are bit-identical to the single-GPU (and
reference) run of the same trials.  There is no data-path collective: ranks
only exchange the per-trial outcome records at the end (a gather on the host
plumbing) and the max of their device times.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def shard_trials(trials: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) block of global trial indices owned by `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return rank * trials // world, (rank + 1) * trials // world


def shard_seeds(base_seed: int, trials: int, world: int, rank: int) -> List[int]:
    lo, hi = shard_trials(trials, world, rank)
    return [base_seed + t for t in range(lo, hi)]


def gather_outcomes(local: Sequence, dist=None) -> list:
    """Concatenate every rank's per-trial records in global trial order."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(local)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, list(local))
    out = []
    for p in parts:
        out.extend(p)
    return out


def max_over_ranks(x: float, dist=None, device=None) -> float:
    """Job time = the slowest rank's device time."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: int, dist=None, device=None) -> int:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.int64, device=device or "cpu")
    dist.all_reduce(t)
    return int(t.item())
