"""world_size-2 gloo test of the multi-GPU trial-sharding host logic (CPU only).

Each rank takes its contiguous trial block (paper_2302_12454_b200.shard), runs
the CPU oracle on it as a stand-in for its device batch, and the gathered
outcomes must equal a single-rank run of the whole battery bit for bit --
the property the B200 path relies on (trial independence, bench.cpp:379-397).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2302_12454_b200.shard import shard_seeds, shard_trials


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, T, out_q):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    from oracle_py import Oracle, params
    from paper_2302_12454_b200.shard import gather_outcomes, max_over_ranks, sum_over_ranks
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("orc")
    rng = np.random.default_rng(5)
    n = 12
    h = rng.integers(-8, 9, n) / 4.0
    J = np.triu(rng.integers(-8, 9, (n, n)) / 4.0, 1)
    J = J + J.T
    p = params(4, 60, tau=7)
    local = []
    for s in shard_seeds(1000, T, world, rank):
        r = orc.ssqa_run(h, J, 0.25, p, s, -3.0, False, False)
        local.append((s, r.reached_target, r.first_hit_cycle, r.best_energy))
    allo = gather_outcomes(local, dist)
    tmax = max_over_ranks(float(rank + 1), dist)
    hits = sum_over_ranks(sum(int(x[1]) for x in local), dist)
    if rank == 0:
        out_q.put((allo, tmax, hits))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_blocks_cover_all_trials():
    for T in (1, 7, 100, 1024):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_trials(T, world, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(T))
    with pytest.raises(ValueError):
        shard_trials(10, 2, 2)


def test_gloo_world2_matches_single_rank(orc):
    T = 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    allo, tmax, hits = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    # single-rank reference run of the same battery
    from oracle_py import params
    rng = np.random.default_rng(5)
    n = 12
    h = rng.integers(-8, 9, n) / 4.0
    J = np.triu(rng.integers(-8, 9, (n, n)) / 4.0, 1)
    J = J + J.T
    p = params(4, 60, tau=7)
    single = []
    for s in range(1000, 1000 + T):
        r = orc.ssqa_run(h, J, 0.25, p, s, -3.0, False, False)
        single.append((s, r.reached_target, r.first_hit_cycle, r.best_energy))
    assert allo == single
    assert hits == sum(int(x[1]) for x in single)


# ---- J' row shards: the per-cycle exchange loop (rowshard.shard_cycles) ----

class _FakeShardBatch:
    """Stands in for a device batch on CPU: shard_pass writes a chunk that
    encodes (rank, cycle); shard_merge checks every shard's chunk arrived in
    shard order for the same cycle."""

    def __init__(self, buf, rank, world, nbytes):
        self.buf, self.rank, self.world, self.nb = buf, rank, world, nbytes
        self.cycle = 0
        self.merged = []

    def shard_bytes(self):
        return self.nb

    def shard_pass(self, ptr):
        off = ptr - self.buf.data_ptr()
        assert off == self.rank * self.nb
        self.buf[off:off + self.nb] = (self.rank * 16 + self.cycle) % 251

    def shard_merge(self, ptr):
        assert ptr == self.buf.data_ptr()
        got = [int(self.buf[g * self.nb]) for g in range(self.world)]
        assert got == [(g * 16 + self.cycle) % 251 for g in range(self.world)], got
        self.merged.append(self.cycle)
        self.cycle += 1


def _shard_worker(rank, world, port, cycles, out_q):
    import sys
    import torch
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2302_12454_b200.rowshard import shard_cycles
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nb = 96
    buf = torch.zeros(world * nb, dtype=torch.uint8)
    b = _FakeShardBatch(buf, rank, world, nb)

    def all_gather(out, mine):
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine.clone())
        out.copy_(torch.cat(parts))

    shard_cycles(b, buf, rank, world, cycles, all_gather)
    out_q.put((rank, b.merged))
    dist.barrier()
    dist.destroy_process_group()


def test_row_shard_exchange_gloo_world2():
    """world_size 2 (gloo, CPU): every cycle each rank passes into its own
    chunk, the all-gather leaves the chunks in rank order, and every rank
    merges all of them for the same cycle (host logic of rowshard)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, 5, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert got == {0: list(range(5)), 1: list(range(5))}


def _p2p_worker(rank, world, port, out_q):
    import torch.distributed as dist
    from paper_2302_12454_b200.rowshard import P2PLayout
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    layout = P2PLayout(world, 12345)
    # stand-ins for the region bases each rank maps (its own + IPC peers)
    mine = 1 << 40 | rank << 32
    bases = [None] * world
    dist.all_gather_object(bases, mine)
    plan = {}
    for epoch in (1, 2, 3):
        plan[epoch] = layout.cycle_args(rank, epoch, bases)
    out_q.put((rank, bases, plan))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_push_layout_agrees_across_ranks():
    """world_size-2 gloo run of the peer-push bookkeeping (rowshard.P2PLayout):
    where rank r pushes its chunk and flag in region d is exactly where rank
    d's merge reads shard r, the two epoch parities never overlap, and the
    flags sit past both data halves."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_p2p_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in ps:
        pr.start()
    got = dict((r, (b, pl)) for r, b, pl in (q.get(timeout=120) for _ in range(world)))
    for pr in ps:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    from paper_2302_12454_b200.rowshard import P2PLayout
    layout = P2PLayout(world, 12345)
    assert got[0][0] == got[1][0]  # every rank sees the same bases
    for epoch in (1, 2, 3):
        for r in range(world):
            dests, flags, _, _ = got[r][1][epoch]
            for d in range(world):
                _, _, chunks_d, flags_d = got[d][1][epoch]
                assert dests[d] == chunks_d + r * layout.stride
                assert flags[d] == flags_d + 4 * r
                assert dests[d] + layout.chunk <= got[d][0][d] + layout.flags_off
        a = got[0][1][epoch][2]
        b = got[0][1][epoch + 1][2] if epoch < 3 else got[0][1][epoch - 1][2]
        assert abs(a - b) == layout.half  # consecutive epochs use the two halves
