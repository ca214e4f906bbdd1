"""J' row sharding across GPUs (BASELINE configs 4-5).

GPU g of G keeps the whole problem but updates only spin rows
[g*npad/G, (g+1)*npad/G): each cycle it contracts its J' rows against the
full sigma (K = N), updates its rows, and the G GPUs all-gather one chunk
each -- their sigma(c+1) rows bit-packed plus per-column int64 energy
partials -- after which every GPU holds the full sigma(c+1), sums the
energies and scans the cycle exactly as run_lattice (annealer.cpp:313-361).
Results are identical on every GPU and bitwise equal to the unsharded run.

`run_row_sharded` drives it over torch.distributed, one process per GPU,
with one of two exchanges:
* "nccl": an in-place ncclAllGather ordered on the engine's own CUDA stream;
* "p2p": no collective library -- every GPU allocates an exchange region
  (two halves by epoch parity + one flag per shard), maps its peers' regions
  through CUDA IPC, and the shard pass's pack kernel stores its chunk straight
  into every region over NVLink and raises the flags (ssqa_batch_shard_pass_to);
  the merge waits on its own flags (ssqa_batch_shard_merge_from).
`run_emulated_shards` runs G shards on ONE GPU, one after the other on the
problem's stream (all passes of a cycle, then all merges), with either
exchange, so the shard data path is exercised without any kernel waiting on
another.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
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


@dataclass(frozen=True)
class P2PLayout:
    """One GPU's exchange region for G shards of `chunk` bytes: two data
    halves (epoch parity) of G chunks in shard order, then G u32 flags."""
    nshards: int
    chunk: int

    @property
    def stride(self) -> int:  # chunk slot, 256-byte aligned
        return (self.chunk + 255) // 256 * 256

    @property
    def half(self) -> int:
        return self.nshards * self.stride

    @property
    def flags_off(self) -> int:
        return 2 * self.half

    @property
    def total(self) -> int:
        return self.flags_off + 256

    def cycle_args(self, rank: int, epoch: int, bases: Sequence[int]):
        """Pointers for one cycle of shard `rank`: its chunk's destination in
        every region, the flag it raises in every region, and its own region's
        chunks and flags for the merge."""
        par = (epoch & 1) * self.half
        dests = [b + par + rank * self.stride for b in bases]
        flags = [b + self.flags_off + 4 * rank for b in bases]
        return dests, flags, bases[rank] + par, bases[rank] + self.flags_off


def shard_cycles_p2p(b, layout: P2PLayout, rank: int, bases: Sequence[int], cycles: int,
                     epoch0: int = 0) -> int:
    """The per-cycle exchange of one shard over peer memory.  Epochs keep
    counting across runs on the same regions (epoch0 = the last one used):
    a flag left at an old epoch can never satisfy a new wait.  Returns the
    last epoch."""
    e = epoch0
    for _ in range(cycles):
        e += 1
        dests, flags, mine, own_flags = layout.cycle_args(rank, e, bases)
        b.shard_pass_to(dests, flags, e)
        b.shard_merge_from(mine, own_flags, layout.nshards, e)
    return e


def shard_cycles_direct(b, layout: P2PLayout, rank: int, bases: Sequence[int],
                        sig4: Sequence[int], cycles: int, epoch0: int = 0) -> int:
    """The per-cycle exchange fused into the shard pass (exchange "direct"):
    the pass's epilogue stores its spin words into every GPU's FP4 slot
    (sig4[d]) and its last CTA pushes the energy partials into slot `rank` of
    every region; the merge waits on its own flags."""
    e = epoch0
    for _ in range(cycles):
        e += 1
        parts, flags, mine, own_flags = layout.cycle_args(rank, e, bases)
        b.shard_pass_direct(sig4, parts, flags, e)
        b.shard_merge_direct(mine, layout.stride, own_flags, layout.nshards, e)
    return e


class ExchangeRegion:
    """A zeroed device block of its own (ssqa_exchange_alloc), IPC-shareable."""

    def __init__(self, nbytes: int, device: int):
        self.ptr = C.c_void_p()
        _lib.check(_lib.lib().ssqa_exchange_alloc(device, nbytes, C.byref(self.ptr)))

    @property
    def base(self) -> int:
        return int(self.ptr.value)

    def handle(self) -> bytes:
        h = C.create_string_buffer(64)
        _lib.check(_lib.lib().ssqa_ipc_handle(self.ptr, h))
        return h.raw

    def close(self):
        if self.ptr:
            _lib.lib().ssqa_exchange_free(self.ptr)
            self.ptr = C.c_void_p()


def _finish(b: Batch, trials: int, opts: RunOptions, p=None) -> List[AnnealResult]:
    b.shard_end()
    res, best, tr = b.fetch(True, opts.record_trace)
    return _results(res, best, tr, trials, p)


def capture_run(b: Batch, buf, rank: int, world: int, cycles: int, all_gather, stream,
                target: Optional[float], stop_at_target: bool):
    """The whole row-sharded run -- begin, `cycles` x (pass, NCCL all-gather,
    merge), end -- captured once as a CUDA graph on the engine's stream
    (every cycle's launches keep their own parameters as graph nodes), so a
    run is ONE host launch instead of ~5 per cycle (the per-cycle host cost
    that dominates at 8 GPUs, where a C4 cycle computes in ~70 us).  The
    batch must have run once before (one-time allocations and symbol copies
    cannot be captured).  Replay with graph.replay_on_engine() (on the
    engine's stream); results via b.fetch()."""
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        b.shard_begin(target, stop_at_target)
        shard_cycles(b, buf, rank, world, cycles, all_gather)
        b.shard_end()

    def replay():  # on the engine's stream, ordered with the batch's own calls
        with torch.cuda.stream(stream):
            g.replay()
    g.replay_on_engine = replay
    return g


def run_row_sharded(m: IsingModel, p: SsqaParams, seeds: Sequence[int],
                    target: Optional[float] = None, opts: RunOptions = RunOptions(),
                    device: int = 0, group=None, exchange: str = "nccl",
                    graph: bool = False) -> List[AnnealResult]:
    """ssqa_run for every seed with J' rows sharded over the ranks of `group`
    (the default process group when torch.distributed is initialised, else a
    single shard); exchange "nccl" (all-gather) or "p2p" (peer push)."""
    import torch
    import torch.distributed as dist
    p.validate(m.n)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    prob = Problem(m, device)
    b = Batch(prob, p, len(seeds), opts.record_trace, _lib.ENGINE_TCGEN05)
    try:
        b.set_shard(rank, world)
        if exchange in ("p2p", "direct"):
            b.set_seeds(seeds)
            return _run_p2p(b, p, seeds, target, opts, device, group, world, rank,
                            direct=exchange == "direct")
        buf = torch.empty(world * b.shard_bytes(), dtype=torch.uint8, device=f"cuda:{device}")
        stream = torch.cuda.ExternalStream(b.stream, device=f"cuda:{device}")

        def all_gather(out, mine):  # NCCL, ordered on the engine's stream
            with torch.cuda.stream(stream):
                dist.all_gather_into_tensor(out, mine, group=group)

        b.set_seeds(seeds)
        b.shard_begin(target, opts.stop_at_target)
        shard_cycles(b, buf, rank, world, p.sc + 1, all_gather)
        if not graph:
            return _finish(b, len(seeds), opts, p)
        b.shard_end()
        # graph mode: the same run again, captured and replayed
        g = capture_run(b, buf, rank, world, p.sc + 1, all_gather, stream, target,
                        opts.stop_at_target)
        g.replay_on_engine()
        b.synchronize()
        res, best, tr = b.fetch(True, opts.record_trace)
        return _results(res, best, tr, len(seeds), p)
    finally:
        b.close()
        prob.close()


def _map_peers(local_ptr: int, handle: bytes, device: int, group, world: int, rank: int,
               opened: list) -> List[int]:
    """All-gather one IPC handle per rank; return every rank's pointer as
    mapped in this process (its own pointer for this rank)."""
    import torch.distributed as dist
    handles = [None] * world
    if world > 1:
        dist.all_gather_object(handles, handle, group=group)
    out = []
    for g in range(world):
        if g == rank:
            out.append(local_ptr)
        else:
            ptr = C.c_void_p()
            _lib.check(_lib.lib().ssqa_ipc_open(handles[g], device, C.byref(ptr)))
            opened.append(ptr)
            out.append(int(ptr.value))
    return out


def _ipc_handle(ptr: int) -> bytes:
    h = C.create_string_buffer(64)
    _lib.check(_lib.lib().ssqa_ipc_handle(C.c_void_p(ptr), h))
    return h.raw


def _run_p2p(b, p, seeds, target, opts, device, group, world, rank, direct=False):
    import torch.distributed as dist
    if direct and not b.shard_direct_ok():
        raise _lib.SsqaError("the fused exchange needs FP4 operands and the table epilogue")
    layout = P2PLayout(world, b.shard_bytes())
    region = ExchangeRegion(layout.total, device)
    opened = []
    try:
        bases = _map_peers(region.base, region.handle(), device, group, world, rank, opened)
        if direct:
            mine4 = b.sig4_ptr()
            sig4 = _map_peers(mine4, _ipc_handle(mine4), device, group, world, rank, opened)
        # shard_begin repacks this GPU's FP4 slots; it must be complete on the
        # device before any peer's pass 0 pushes spin words into them
        b.shard_begin(target, opts.stop_at_target)
        b.synchronize()
        if world > 1:
            dist.barrier(group=group)  # every region is zeroed, mapped and begun
        if direct:
            shard_cycles_direct(b, layout, rank, bases, sig4, p.sc + 1)
        else:
            shard_cycles_p2p(b, layout, rank, bases, p.sc + 1)
        out = _finish(b, len(seeds), opts, p)
        if world > 1:
            dist.barrier(group=group)  # no peer still writes into this region
        return out
    finally:
        for ptr in opened:
            _lib.lib().ssqa_ipc_close(ptr)
        region.close()


def run_emulated_shards(m: IsingModel, p: SsqaParams, seeds: Sequence[int], nshards: int,
                        target: Optional[float] = None, opts: RunOptions = RunOptions(),
                        device: int = 0, exchange: str = "nccl") -> List[List[AnnealResult]]:
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
        for b in shards:
            b.shard_begin(target, opts.stop_at_target)
        if exchange in ("p2p", "direct"):
            # one region per emulated GPU, all on this device
            layout = P2PLayout(nshards, nb)
            regions = [ExchangeRegion(layout.total, device) for _ in range(nshards)]
            try:
                bases = [r.base for r in regions]
                sig4 = [b.sig4_ptr() for b in shards] if exchange == "direct" else None
                for c in range(p.sc + 1):
                    args = [layout.cycle_args(g, c + 1, bases) for g in range(nshards)]
                    for g, b in enumerate(shards):
                        if sig4:
                            b.shard_pass_direct(sig4, args[g][0], args[g][1], c + 1)
                        else:
                            b.shard_pass_to(args[g][0], args[g][1], c + 1)
                    for g, b in enumerate(shards):
                        if sig4:
                            b.shard_merge_direct(args[g][2], layout.stride, args[g][3], nshards,
                                                 c + 1)
                        else:
                            b.shard_merge_from(args[g][2], args[g][3], nshards, c + 1)
                return [_finish(b, len(seeds), opts, p) for b in shards]
            finally:
                for r in regions:
                    r.close()
        buf = torch.empty(nshards * nb, dtype=torch.uint8, device=f"cuda:{device}")
        for _ in range(p.sc + 1):
            for g, b in enumerate(shards):
                b.shard_pass(buf[g * nb:].data_ptr())
            for b in shards:
                b.shard_merge(buf.data_ptr())
        return [_finish(b, len(seeds), opts, p) for b in shards]
    finally:
        for b in shards:
            b.close()
        prob.close()
