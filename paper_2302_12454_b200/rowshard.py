"""J' row sharding across GPUs (BASELINE configs 4-5).

GPU g of G keeps the whole problem but updates only spin rows
[g*npad/G, (g+1)*npad/G): each cycle it contracts its J' rows against the
full sigma (K = N), updates its rows, and the G GPUs all-gather one chunk
each -- their sigma(c+1) rows bit-packed plus per-column int64 energy
partials -- after which every GPU holds the full sigma(c+1), sums the
energies and scans the cycle exactly as run_lattice (annealer.cpp:313-361).
Results are identical on every GPU and bitwise equal to the unsharded run.

`run_row_sharded` drives it over torch.distributed (NCCL, one process per
GPU): the all-gather is in place and is ordered on the engine's own CUDA
stream.  `run_emulated_shards` runs G shards on ONE GPU, one after the
other on the problem's stream with a shared exchange buffer, so the shard
data path is exercised without any kernel waiting on another.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

from . import _lib
from .api import AnnealResult, Batch, IsingModel, Problem, RunOptions, SsqaParams, _results


def shard_cycles(b, buf, rank: int, world: int, cycles: int, all_gather) -> None:
    """The per-cycle exchange of one shard: pass into this shard's chunk of
    `buf` (G chunks of b.shard_bytes() bytes, in shard order), in-place
    all-gather of the chunks, merge.  `all_gather(buf, mine)` fills `buf`
    from every shard's `mine` (skipped for a single shard)."""
    nb = b.shard_bytes()
    mine = buf[rank * nb:(rank + 1) * nb]
    for _ in range(cycles):
        b.shard_pass(mine.data_ptr())
        if world > 1:
            all_gather(buf, mine)
        b.shard_merge(buf.data_ptr())


def _finish(b: Batch, trials: int, opts: RunOptions) -> List[AnnealResult]:
    b.shard_end()
    res, best, tr = b.fetch(True, opts.record_trace)
    return _results(res, best, tr, trials)


def run_row_sharded(m: IsingModel, p: SsqaParams, seeds: Sequence[int],
                    target: Optional[float] = None, opts: RunOptions = RunOptions(),
                    device: int = 0, group=None) -> List[AnnealResult]:
    """ssqa_run for every seed with J' rows sharded over the ranks of `group`
    (the default process group when torch.distributed is initialised, else a
    single shard)."""
    import torch
    import torch.distributed as dist
    p.validate(m.n)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    prob = Problem(m, device)
    b = Batch(prob, p, len(seeds), opts.record_trace, _lib.ENGINE_TCGEN05)
    try:
        b.set_shard(rank, world)
        buf = torch.empty(world * b.shard_bytes(), dtype=torch.uint8, device=f"cuda:{device}")
        stream = torch.cuda.ExternalStream(b.stream, device=f"cuda:{device}")

        def all_gather(out, mine):  # NCCL, ordered on the engine's stream
            with torch.cuda.stream(stream):
                dist.all_gather_into_tensor(out, mine, group=group)

        b.set_seeds(seeds)
        b.shard_begin(target, opts.stop_at_target)
        shard_cycles(b, buf, rank, world, p.sc + 1, all_gather)
        return _finish(b, len(seeds), opts)
    finally:
        b.close()
        prob.close()


def run_emulated_shards(m: IsingModel, p: SsqaParams, seeds: Sequence[int], nshards: int,
                        target: Optional[float] = None, opts: RunOptions = RunOptions(),
                        device: int = 0) -> List[List[AnnealResult]]:
    """The G-shard data path on one GPU: G shard batches over one problem
    (one CUDA stream, so everything runs in order), exchanging through one
    buffer laid out as the all-gather would leave it.  Returns every shard's
    results (they must all agree)."""
    import torch
    p.validate(m.n)
    prob = Problem(m, device)
    shards = [Batch(prob, p, len(seeds), opts.record_trace, _lib.ENGINE_TCGEN05)
              for _ in range(nshards)]
    try:
        for g, b in enumerate(shards):
            b.set_shard(g, nshards)
            b.set_seeds(seeds)
        nb = shards[0].shard_bytes()
        buf = torch.empty(nshards * nb, dtype=torch.uint8, device=f"cuda:{device}")
        for b in shards:
            b.shard_begin(target, opts.stop_at_target)
        for _ in range(p.sc + 1):
            for g, b in enumerate(shards):
                b.shard_pass(buf[g * nb:].data_ptr())
            for b in shards:
                b.shard_merge(buf.data_ptr())
        return [_finish(b, len(seeds), opts) for b in shards]
    finally:
        for b in shards:
            b.close()
        prob.close()
