"""Full-size BASELINE configs C4 and C5 on the device, checked bitwise over
their first 50 sweeps (BASELINE.json: "bit-exactness is checked against the
CPU oracle over the first 50 steps") against oracle/lattice_np.py -- the
vectorised restatement pinned to the C oracle in test_oracle_golden.py.

Sizes are the configs' own: N=8192 dense int[-8,7], M=32, 256 trials; and
N=32768 +-1 couplings, M=16, 64 trials.  The whole batch runs on the GPU
(production geometry: wide column tiles split over row parts); the first
and the last trial are recomputed on the host.
"""
import numpy as np
import pytest

import paper_2302_12454_b200 as sq
from oracle_py import params

pytestmark = pytest.mark.gpu

STEPS = 50


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("n,kind,R,T", [(8192, 0, 32, 256), (32768, 1, 16, 64)],
                         ids=["c4", "c5"])
def test_full_size_first_50_steps(n, kind, R, T):
    import lattice_np as lnp
    m = sq.dense_ising(n, kind, 7)
    p = params(R, STEPS)
    seeds = [1000 + t for t in range(T)]
    res = sq.ssqa_run_batch(m, sq.SsqaParams(r=R, sc=STEPS), seeds, None,
                            sq.RunOptions(True, False))
    check = [0, T - 1]
    # J is integral (p = 0): the product runs on the model's own float64 matrix
    ref = lnp.run_lattice(m.h, m.J, m.offset, R, p.delay, p.n_rnd, p.alpha, False, STEPS,
                          lnp.jperp_schedule(p), lambda c: p.i0, [seeds[t] for t in check],
                          J_scaled=m.J)
    for o, t in zip(ref, check):
        r = res[t]
        assert r.cycles_used == o.cycles_used == STEPS
        assert np.array_equal(bits(r.trace_energy), bits(o.trace.reshape(-1))), t
        assert (r.best_energy, r.best_replica) == (o.best_energy, o.best_replica), t
        assert np.array_equal(r.best_state, o.best_state), t


DENSE = {"c4": (8192, 0, 32, 256, 2000), "c5": (32768, 1, 16, 64, 1000)}


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_dense_full_budget_matches_golden(golden, cfg):
    """C4 / C5 at their full sweep budgets (2000 / 1000 sweeps, production
    geometry: wide tiles, row split, CTA pairs, table epilogue): the first and
    the last trial's whole energy trace, best energy / replica and best state
    equal the outcomes scripts/make_golden_dense.py computed with
    oracle/lattice_np.py (tests/golden/dense_full.npz, SHA-256 of the float64
    trace and int8 state bytes)."""
    import hashlib
    cases = golden("dense_full")
    if cfg not in cases:
        pytest.skip(f"no {cfg} case in tests/golden/dense_full.npz")
    g = cases[cfg]
    n, kind, R, T, sc = DENSE[cfg]
    assert [int(x) for x in g["k"]] == [n, kind, R, T, sc]
    prob = sq.Problem.generated_dense(n, kind, 7)  # built on the device, as bench.py does
    try:
        seeds = [1000 + t for t in range(T)]
        res = sq.ssqa_run_batch(sq.api._Shape(n), sq.SsqaParams(r=R, sc=sc), seeds, None,
                                sq.RunOptions(True, False), problem=prob)
    finally:
        prob.close()
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    for j, t in enumerate(int(x) for x in g["trial"]):
        r = res[t]
        assert r.cycles_used == int(g["cycles_used"][j]) == sc
        tr = r.trace_energy.reshape(sc + 1, R)
        peek = [int(c) for c in g["peek_cycle"]]
        assert np.array_equal(bits(tr[peek]), bits(g["peek_energy"][j])), (cfg, t)
        assert sha(r.trace_energy.astype(np.float64)) == str(g["trace_sha"][j]), (cfg, t)
        assert (r.best_energy, r.best_replica) == (float(g["best_energy"][j]),
                                                   int(g["best_replica"][j])), (cfg, t)
        assert sha(r.best_state.astype(np.int8)) == str(g["state_sha"][j]), (cfg, t)


# ---- BASELINE configs 2 and 3 at their own shapes (Missing 1) ----
# GI n=20 -> N=400 and n=50 -> N=2500 (fixed instance: gi seed 7, permuted,
# c1 = c2 = 1), M=20, the full 1024-trial battery on the device with the
# production geometry (FP4 operands, 147 column tiles of whole trials).

GI_CFG = {"c2": (20, 2000), "c3": (50, 5000)}


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_gi_full_battery_first_50_steps(cfg):
    """The 1024-trial batch over its first 50 sweeps; trials spread over the
    column tiles (first, a mid tile, the last trial of the last tile) are
    recomputed by oracle/lattice_np.py and must agree bitwise: per-cycle
    energies of every replica, best energy / replica / state."""
    import lattice_np as lnp
    nn, _ = GI_CFG[cfg]
    T, R = 1024, 20
    m = sq.gi_ising(nn, 0.5, 7, True, 1.0, 1.0)
    p = params(R, STEPS)
    seeds = [1000 + t for t in range(T)]
    res = sq.ssqa_run_batch(m, sq.SsqaParams(r=R, sc=STEPS), seeds, None,
                            sq.RunOptions(True, False))
    check = [0, 146, 511, 1022, T - 1]
    ref = lnp.run_lattice(m.h, m.J, m.offset, R, p.delay, p.n_rnd, p.alpha, False, STEPS,
                          lnp.jperp_schedule(p), lambda c: p.i0, [seeds[t] for t in check])
    for o, t in zip(ref, check):
        r = res[t]
        assert r.cycles_used == o.cycles_used == STEPS
        assert np.array_equal(bits(r.trace_energy), bits(o.trace.reshape(-1))), t
        assert (r.best_energy, r.best_replica) == (o.best_energy, o.best_replica), t
        assert np.array_equal(r.best_state, o.best_state), t


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_gi_full_battery_matches_reference_run_trials(golden, cfg):
    """run_trials at the config's full budget (sc = 2000 / 5000, ec = 20 sc,
    fixed budget, target 0) on the whole 1024-trial battery in one device
    batch; the per-trial outcomes (reached, first hit cycle, best energy) of
    the trials the reference ran (scripts/make_golden.py trials_large:
    oracle/_ref run_trials, bench.cpp:359-432) must be identical."""
    nn, sc = GI_CFG[cfg]
    ref = golden("trials_large")[{"c2": "c2_gi20", "c3": "c3_gi50"}[cfg]]
    m = sq.gi_ising(nn, 0.5, 7, True, 1.0, 1.0)
    T = 1024
    outs, p_s, _, _ = sq.run_trials(m, sq.SsqaParams(r=20), T, 20 * sc, 1000)
    k = len(ref["seed"])
    assert [o.seed for o in outs[:k]] == [int(x) for x in ref["seed"]]
    assert [int(o.reached_target) for o in outs[:k]] == [int(x) for x in ref["reached"]]
    assert [o.first_hit_cycle for o in outs[:k]] == [int(x) for x in ref["first_hit"]]
    assert np.array_equal(bits([o.best_energy for o in outs[:k]]), bits(ref["best_energy"]))
    if k == T:
        assert p_s == float(ref["p_s"])


@pytest.mark.parametrize("T", [512, 256, 128], ids=["g2", "g4", "g8"])
def test_c3_rank_block_shapes_match_reference(golden, T):
    """Trial sharding over G = 2 / 4 / 8 GPUs hands each rank a block of 512 /
    256 / 128 trials of the C3 battery (shard.py; seeds stay base + global
    index).  Rank 0's block at each of those sizes -- its own geometry: fewer,
    narrower column tiles, a row split at 128 trials -- at the full budget must
    give the reference's per-trial outcomes (tests/golden/trials_large.npz,
    seeds 1000..1047)."""
    ref = golden("trials_large")["c3_gi50"]
    m = sq.gi_ising(50, 0.5, 7, True, 1.0, 1.0)
    outs, _, _, _ = sq.run_trials(m, sq.SsqaParams(r=20), T, 20 * 5000, 1000)
    k = len(ref["seed"])
    assert [o.seed for o in outs[:k]] == [int(x) for x in ref["seed"]]
    assert [int(o.reached_target) for o in outs[:k]] == [int(x) for x in ref["reached"]]
    assert [o.first_hit_cycle for o in outs[:k]] == [int(x) for x in ref["first_hit"]]
    assert np.array_equal(bits([o.best_energy for o in outs[:k]]), bits(ref["best_energy"]))


@pytest.mark.parametrize("n,R,T", [(2048, 20, 1), (2048, 7, 5), (2100, 1, 17), (2560, 20, 40),
                                   (4000, 12, 9), (2048, 33, 3)])
def test_mid_size_geometry_search_matches_numpy(n, R, T):
    """Problems of 16-63 row tiles take the column tiling from make_geom's
    search (trials per tile x row parts by a cost model): odd batteries --
    one trial, one replica, widths that do not divide the tile cap, sizes
    with padding rows -- over 40 sweeps against oracle/lattice_np.py, every
    trial, every replica's energy of every cycle."""
    import lattice_np as lnp
    rng = np.random.default_rng(n + R + T)
    J = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    J[iu] = rng.integers(-2, 3, len(iu[0])) * 0.5
    J = J + J.T
    h = rng.integers(-6, 7, n) * 0.5
    m = sq.IsingModel.from_arrays(h, J, 0.5)
    steps = 40
    p = params(R, steps)
    seeds = [31 + 7 * t for t in range(T)]
    res = sq.ssqa_run_batch(m, sq.SsqaParams(r=R, sc=steps), seeds, None,
                            sq.RunOptions(True, False))
    ref = lnp.run_lattice(m.h, m.J, m.offset, R, p.delay, p.n_rnd, p.alpha, False, steps,
                          lnp.jperp_schedule(p), lambda c: p.i0, seeds)
    for t, (r, o) in enumerate(zip(res, ref)):
        assert np.array_equal(bits(r.trace_energy), bits(o.trace.reshape(-1))), t
        assert (r.best_energy, r.best_replica) == (o.best_energy, o.best_replica), t
        assert np.array_equal(r.best_state, o.best_state), t


@pytest.mark.parametrize("jval", [6.0, 12.0], ids=["fp4", "fp4pair"])
def test_fp4_large_aligned_fields_exact(jval):
    """FP4 operands accumulate in the tensor core's fp32 TMEM accumulator;
    exactness needs every partial sum of the block-scaled MMA to be exact.
    A ferromagnet (J' = 6: one e2m1 plane; J' = 12 = 6 + 6: the FP4 pair) at
    N = 8192 aligns within a few sweeps, so the fields reach |S| = J' (N - 1)
    = 49146 / 98292 (> 2^15, > 2^16).  The run must equal the forced-int8 run
    (int32 accumulators) bitwise and oracle/lattice_np.py on two trials."""
    import lattice_np as lnp
    n, R, T, steps = 8192, 8, 4, 30
    J = np.full((n, n), jval)
    np.fill_diagonal(J, 0.0)
    m = sq.IsingModel.from_arrays(np.zeros(n), J, 0.0)
    p = sq.SsqaParams(r=R, sc=steps)
    seeds = [77 + t for t in range(T)]
    opts = sq.RunOptions(True, False)
    fp4 = sq.ssqa_run_batch(m, p, seeds, None, opts)
    sq.tune(fp4=0)
    i8 = sq.ssqa_run_batch(m, p, seeds, None, opts)
    sq.tune()
    for a, b in zip(fp4, i8):
        assert np.array_equal(bits(a.trace_energy), bits(b.trace_energy))
        assert np.array_equal(a.best_state, b.best_state)
    # the runs really reached the large-field regime: an aligned replica
    assert min(r.best_energy for r in fp4) == -jval * n * (n - 1) / 2
    q = params(R, steps)
    ref = lnp.run_lattice(m.h, m.J, m.offset, R, q.delay, q.n_rnd, q.alpha, False, steps,
                          lnp.jperp_schedule(q), lambda c: q.i0, [seeds[0], seeds[-1]])
    for o, t in zip(ref, [0, T - 1]):
        assert np.array_equal(bits(fp4[t].trace_energy), bits(o.trace.reshape(-1))), t
        assert np.array_equal(fp4[t].best_state, o.best_state), t
