"""Pin the CPU oracle (oracle/ssqa_oracle.c) before trusting it.

1. Known-answer tests frozen in the reference's own suites
   (proj/tests/test_rng.cpp:28-135, proj/tests/test_annealer.cpp:76-304).
2. Bitwise agreement with the reference itself: committed fixtures under
   tests/golden/ (made by scripts/make_golden.py from oracle/_ref) and, when
   oracle/_ref is present, live runs of the compiled reference.
3. The SURVEY.md section 8.2 KATs (FNV-1a hashes of traces / best states).
"""
import numpy as np
import pytest

from oracle_py import params, ssa_params

STREAM_SPIN_INIT, STREAM_SWEEP_NOISE, STREAM_SA_PICK, STREAM_GI_EDGES = 1, 2, 3, 5


def fnv1a(data: bytes) -> int:
    h = 0xcbf29ce484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


# ---- test_rng.cpp -------------------------------------------------------------

def test_mix64_goldens(orc):
    assert orc.mix64(0) == 0xe220a8397b1dcdaf
    assert orc.mix64(1) == 0x910a2dec89025cc1


def test_mix64_matches_splitmix_stream(orc):
    # test_rng.cpp:28-42: walking splitmix64 from s gives mix64(s), mix64(s+g), ...
    g = 0x9e3779b97f4a7c15
    M = 0xFFFFFFFFFFFFFFFF
    for s0 in (0, 1, 0xdeadbeef, 0x123456789abcdef):
        state = s0
        x = s0
        for _ in range(16):
            state = (state + g) & M
            z = state
            z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
            z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
            z ^= z >> 31
            assert orc.mix64(x) == z
            x = (x + g) & M


def test_counter_rng_frozen_draws(orc):
    # test_rng.cpp:44-56
    assert orc.rng_key(42, STREAM_SWEEP_NOISE) == 0x0eaba014b9afe772
    assert orc.rng_raw(42, STREAM_SWEEP_NOISE, 0) == 0x6d3ffc4694a32db4
    assert orc.rng_raw(42, STREAM_SWEEP_NOISE, 1) == 0x7db981c830543b70
    assert orc.rng_raw(42, STREAM_SWEEP_NOISE, 1 << 32) == 0x246d125b3b72f451
    assert orc.uniform01(42, STREAM_SWEEP_NOISE, 7) == pytest.approx(0.54184610102375963,
                                                                     rel=1e-15)
    assert (orc.rng_raw(42, STREAM_SWEEP_NOISE, 5) >> 63) == 0  # pm1(5) == -1
    assert (orc.rng_raw(42, STREAM_SWEEP_NOISE, 6) >> 63) == 1  # pm1(6) == +1
    assert (orc.rng_raw(42, STREAM_SWEEP_NOISE, 9) * 10) >> 64 == 5  # below(9, 10) == 5
    assert orc.rng_raw(42, STREAM_SA_PICK, 0) == 0x0a3b34d3e50885fb


def test_spin_counter_packing(orc):
    # test_rng.cpp:121-135
    assert orc.spin_counter(1, 2, 3) == 0x100200003
    assert orc.spin_counter(0, 0, 0) == 0
    assert orc.spin_counter(0, 0, (1 << 20) - 1) < orc.spin_counter(0, 1, 0)
    assert orc.spin_counter(0, (1 << 12) - 1, (1 << 20) - 1) < orc.spin_counter(1, 0, 0)


def test_noise_top5_identity(orc):
    # u < 7/16 <=> raw>>59 < 14 and u < 23/32 <=> raw>>59 < 23
    for c in range(20000):
        raw = orc.rng_raw(99, STREAM_SWEEP_NOISE, c * 7919)
        u = (raw >> 11) * 2.0 ** -53
        t = raw >> 59
        assert (u < 0.4375) == (t < 14)
        assert (u < 0.71875) == (t < 23)


# ---- test_annealer.cpp ----------------------------------------------------------

def test_jperp_staircase(orc):
    # test_annealer.cpp:76-99
    p = params(1, 1)
    assert orc.jperp_schedule(0, p) == 0.0
    assert orc.jperp_schedule(99, p) == 0.0
    assert orc.jperp_schedule(100, p) == pytest.approx(0.5 / 3)
    assert orc.jperp_schedule(250, p) == pytest.approx(1.0 / 3)
    assert orc.jperp_schedule(300, p) == 0.5
    assert orc.jperp_schedule(399, p) == 0.5
    assert orc.jperp_schedule(400, p) == 0.0
    q = params(1, 1, jperp_min=0.25, jperp_max=0.75, beta=1, tau=1)
    assert [orc.jperp_schedule(c, q) for c in range(4)] == [0.25, 0.75, 0.25, 0.75]
    with pytest.raises(Exception):
        orc.jperp_schedule(-1, p)


def _one_spin(bias):
    return np.array([bias]), np.zeros((1, 1)), 0.0


def test_clamp_kats(orc):
    # test_annealer.cpp:219-264
    p = params(1, 4, n_rnd=0.0, delay=0, jperp_min=0.0, jperp_max=0.0)
    h, J, off = _one_spin(5.0)
    s, a, hist = orc.init_lattice(1, 1, 0, 3)
    cyc = orc.ssqa_sweep(h, J, off, 0.0, p, 3, 0, s, a, hist, 0)
    assert a[0] == 1.0 and s[0] == 1.0
    cyc = orc.ssqa_sweep(h, J, off, 0.0, p, 3, 1, s, a, hist, cyc)
    assert a[0] == 1.0
    h, J, off = _one_spin(-5.0)
    s, a, hist = orc.init_lattice(1, 1, 0, 3)
    orc.ssqa_sweep(h, J, off, 0.0, p, 3, 0, s, a, hist, 0)
    assert a[0] == -2.0 and s[0] == -1.0
    half = params(1, 4, n_rnd=0.0, delay=0, jperp_min=0.0, jperp_max=0.0, alpha=0.5)
    h, J, off = _one_spin(5.0)
    s, a, hist = orc.init_lattice(1, 1, 0, 3)
    orc.ssqa_sweep(h, J, off, 0.0, half, 3, 0, s, a, hist, 0)
    assert a[0] == 1.5
    # zero input is a tie and the spin turns on
    s, a, hist = orc.init_lattice(2, 1, 0, 3)
    orc.ssqa_sweep(np.zeros(2), np.zeros((2, 2)), 0.0, 0.0, p, 3, 0, s, a, hist, 0)
    assert list(s) == [1.0, 1.0] and a[0] == 0.0
    # drift below the floor in small steps
    h, J, off = _one_spin(-0.6)
    s, a, hist = orc.init_lattice(1, 1, 0, 3)
    cyc = 0
    for c in range(4):
        cyc = orc.ssqa_sweep(h, J, off, 0.0, p, 3, c, s, a, hist, cyc)
    assert a[0] == -2.0 and s[0] == -1.0


def test_delayed_coupling_kat(orc):
    # test_annealer.cpp:266-304
    p = params(2, 4, n_rnd=0.0, delay=1)
    h, J = np.zeros(1), np.zeros((1, 1))
    s = np.array([-1.0, -1.0])
    a = np.zeros(2)
    hist = np.array([[1.0, -1.0], [-1.0, 1.0]])
    cyc = orc.ssqa_sweep(h, J, 0.0, 0.7, p, 5, 0, s, a, hist, 0)
    assert a[0] == pytest.approx(-0.7) and a[1] == pytest.approx(0.7)
    assert list(s) == [-1.0, 1.0]
    assert list(hist[0]) == list(s) and cyc == 1
    orc.ssqa_sweep(h, J, 0.0, 0.7, p, 5, 1, s, a, hist, cyc)
    assert a[0] == pytest.approx(0.0) and s[0] == 1.0
    bi = params(3, 4, n_rnd=0.0, delay=1, bidirectional=True)
    s, a, hist = orc.init_lattice(1, 3, 1, 5)
    hist[0] = [1.0, 1.0, -1.0]
    orc.ssqa_sweep(h, J, 0.0, 0.5, bi, 5, 0, s, a, hist, 0)
    assert list(a) == pytest.approx([0.0, 0.0, 1.0])


def test_validation_rejects(orc):
    # test_annealer.cpp:142-164 (through ssqa_run)
    h, J = np.zeros(3), np.zeros((3, 3))
    from oracle_py import OracleError
    with pytest.raises(OracleError):
        orc.ssqa_run(h, J, 0.0, params(0, 10), 1)
    orc.ssqa_run(h, J, 0.0, params(2, 10), 1)
    for bad in (dict(r=1 << 12), dict(sc=0), dict(sc=1 << 31), dict(jperp_max=-0.1),
                dict(beta=0), dict(tau=0), dict(delay=-1), dict(i0=0.0), dict(alpha=0.0),
                dict(n_rnd=-1.0)):
        kw = dict(r=2, sc=10)
        kw.update(bad)
        with pytest.raises(OracleError):
            orc.ssqa_run(h, J, 0.0, params(**kw), 1)


def test_init_lattice_seeded(orc):
    # test_annealer.cpp:199-217
    a = orc.init_lattice(40, 3, 1, 9)
    b = orc.init_lattice(40, 3, 1, 9)
    c = orc.init_lattice(40, 3, 1, 10)
    assert (a[0] == b[0]).all() and not (a[0] == c[0]).all()
    assert (a[2][0] == a[0]).all() and (a[2][1] == a[0]).all()
    plus = int((a[0] > 0).sum())
    assert 20 < plus < 100 and (a[1] == 0).all()


# ---- bitwise agreement with the reference (golden fixtures) ---------------------

def test_oracle_matches_golden_lattice_trajectories(orc, golden):
    for name, c in golden("lattice_traj").items():
        n, r, d = int(c["n"]), int(c["r"]), int(c["delay"])
        seed = int(c["seed"])
        p = params(r, 1, delay=d, alpha=float(c["alpha"]), bidirectional=bool(c["bidir"]))
        s, a, hist = orc.init_lattice(n, r, d, seed)
        assert np.array_equal(s, c["sigma"][0]), name
        cyc = 0
        for t in range(len(c["jperp"])):
            p.i0 = float(c["i0"][t])
            cyc = orc.ssqa_sweep(c["h"], c["J"], float(c["offset"]), float(c["jperp"][t]), p,
                                 seed, t, s, a, hist, cyc)
            assert np.array_equal(s, c["sigma"][t + 1]), (name, t)
            assert np.array_equal(a.view(np.uint64), c["acc"][t + 1].view(np.uint64)), (name, t)
            e = orc.replica_energies(c["h"], c["J"], float(c["offset"]), r, s)
            assert np.array_equal(e.view(np.uint64), c["energy"][t].view(np.uint64)), (name, t)
        assert np.array_equal(hist, c["hist_final"]), name


def test_oracle_matches_golden_runs(orc, golden):
    runs = golden("runs")
    gi = golden("gi_instances")
    for name, c in runs.items():
        if name.startswith("gi"):
            key = f"gi_{int(c['n_nodes'])}_{int(c['gi_seed'])}_1_{float(c['c'])}"
            inst = gi[key]
            h, J, off = inst["h"], inst.get("J"), float(inst["offset"])
            if J is None:  # large instance: rebuild with the host builder, check its hash
                J = _product_gi(inst)
            kw = {k[2:]: (v.item() if hasattr(v, "item") else v)
                  for k, v in c.items() if k.startswith("p_")}
            p = params(**kw)
            res = orc.ssqa_run(h, J, off, p, int(c["seed"]), float(c["target"]), True,
                               bool(c["stop"]))
            assert res.reached_target == bool(c["reached"]), name
            assert res.first_hit_cycle == int(c["first_hit"]), name
            assert res.cycles_used == int(c["cycles_used"]), name
        else:
            p = params(int(c["p_r"]), int(c["p_sc"]), tau=int(c["p_tau"]))
            res = orc.ssqa_run(c["h"], c["J"], float(c["offset"]), p, int(c["seed"]), None, True,
                               False)
            assert res.cycles_used == int(c["cycles_used"])
        assert res.best_energy == float(c["best_energy"]), name
        assert res.best_replica == int(c["best_replica"]), name
        assert np.array_equal(res.best_state, c["best_state"]), name
        assert np.array_equal(res.trace.view(np.uint64), c["trace"].view(np.uint64)), name


def _product_gi(inst):
    import hashlib
    from paper_2302_12454_b200 import gi_ising
    m = gi_ising(int(inst["n_nodes"]), 0.5, int(inst["seed"]), bool(inst["permute"]),
                 float(inst["c"]), float(inst["c"]))
    assert hashlib.sha256(m.J.tobytes()).hexdigest() == str(inst["J_sha"])
    return m.J


def test_survey_kats(orc, golden):
    # GI n=10 and n=20, seed 123
    gi = golden("gi_instances")
    inst = gi["gi_10_7_1_1.0"]
    res = orc.ssqa_run(inst["h"], inst["J"], float(inst["offset"]), params(20, 1000), 123, 0.0,
                       True, False)
    assert (res.reached_target, res.first_hit_cycle, res.best_energy, res.best_replica,
            res.cycles_used, len(res.trace)) == (True, 304, 0.0, 4, 1000, 20020)
    assert fnv1a(res.trace.tobytes()) == 0xaadf4cd2ff050f78
    assert fnv1a(res.best_state.tobytes()) == 0x796f1f3248dc5771
    t = golden("trials")["trials_gi10"]
    assert float(t["p_s"]) == 0.80
    assert int(t["outcomes_fnv"]) == 0x4b05f8dbfa0ee326
    assert int(golden("runs")["gi20"]["trace_fnv"]) == 0x388463303ba4d818


def test_oracle_matches_reference_live(orc, ref):
    """Random models (including non-dyadic doubles) against the compiled reference."""
    rng = np.random.default_rng(1234)
    for trial in range(6):
        n = int(rng.integers(1, 20))
        r = int(rng.integers(1, 6))
        d = int(rng.integers(0, 3))
        h = rng.uniform(-2, 2, n)
        J = np.triu(rng.uniform(-2, 2, (n, n)), 1)
        J = J + J.T
        off = float(rng.uniform(-2, 2))
        p = params(r, 60, delay=d, tau=7, bidirectional=bool(trial % 2))
        seed = int(rng.integers(0, 2 ** 63))
        a = ref.ssqa_run(h, J, off, p, seed, None, True, False)
        b = orc.ssqa_run(h, J, off, p, seed, None, True, False)
        assert np.array_equal(a.trace.view(np.uint64), b.trace.view(np.uint64))
        assert np.array_equal(a.best_state, b.best_state)
        assert a.best_replica == b.best_replica


def test_reference_gi_instances_match_golden(ref, golden):
    import hashlib
    for name, c in golden("gi_instances").items():
        h, J, off = ref.gi_ising(int(c["n_nodes"]), 0.5, int(c["seed"]), bool(c["permute"]),
                                 float(c["c"]), float(c["c"]))
        assert np.array_equal(h, c["h"]) and off == float(c["offset"])
        assert hashlib.sha256(J.tobytes()).hexdigest() == str(c["J_sha"])


# ---- SSA engine (annealer.cpp:382-408, 489-501) ----

def test_i0_ladder_kats(orc):
    # test_annealer.cpp:101-126
    p = ssa_params(1)
    assert [orc.i0_schedule(c, p) for c in (0, 9, 10, 49, 50)] == [1.0, 1.0, 2.0, 16.0, 1.0]
    assert orc.i0_schedule(123, p) == orc.i0_schedule(23, p)
    from oracle_py import OracleError
    with pytest.raises(OracleError):
        orc.i0_schedule(-1, p)
    levels = lambda q: sorted({orc.i0_schedule(c, q) for c in range(0, 70 * q.tau, q.tau)})  # noqa: E731
    assert levels(ssa_params(1, i0_max=10.0)) == [1, 2, 4, 8]
    assert levels(ssa_params(1, i0_min=0.5, i0_max=8.0)) == [0.5, 1, 2, 4, 8]
    assert len(levels(ssa_params(1, beta=0.3))) == 3


def test_i0_schedule_matches_golden(orc, golden):
    for name, c in golden("ssa_runs").items():
        if not name.startswith("sched"):
            continue
        kw = {k[2:]: v.item() for k, v in c.items() if k.startswith("p_")}
        p = ssa_params(1, **kw)
        got = np.array([orc.i0_schedule(int(cy), p) for cy in c["cycles"]])
        assert np.array_equal(got.view(np.uint64), c["i0"].view(np.uint64)), name


def test_ssa_validation_rejects(orc):
    # test_annealer.cpp:166-185 (through ssa_run)
    h, J = np.zeros(3), np.zeros((3, 3))
    from oracle_py import OracleError
    orc.ssa_run(h, J, 0.0, ssa_params(10), 1)
    for bad in (dict(i0_min=0.0), dict(i0_min=32.0), dict(beta=1.0), dict(beta=0.0),
                dict(tau=0), dict(sc=0), dict(i0_min=1e-30, i0_max=1e30, beta=0.5),
                dict(alpha=0.0), dict(n_rnd=-1.0)):
        kw = dict(sc=10)
        kw.update(bad)
        with pytest.raises(OracleError):
            orc.ssa_run(h, J, 0.0, ssa_params(**kw), 1)


def _ssa_case(c, gi):
    if "h" in c:
        return c["h"], c["J"], float(c["offset"])
    key = f"gi_{int(c['n_nodes'])}_{int(c['gi_seed'])}_1_{float(c['c'])}"
    inst = gi[key]
    J = inst.get("J")
    if J is None:
        J = _product_gi(inst)
    return inst["h"], J, float(inst["offset"])


def ssa_case_params(c):
    kw = {k[2:]: v.item() for k, v in c.items() if k.startswith("p_")}
    return ssa_params(**kw)


def test_oracle_matches_golden_ssa_runs(orc, golden):
    gi = golden("gi_instances")
    for name, c in golden("ssa_runs").items():
        if name.startswith("sched"):
            continue
        h, J, off = _ssa_case(c, gi)
        p = ssa_case_params(c)
        if "target" in c:
            res = orc.ssa_run(h, J, off, p, int(c["seed"]), float(c["target"]), True,
                              bool(c["stop"]))
            assert res.reached_target == bool(c["reached"]), name
            assert res.first_hit_cycle == int(c["first_hit"]), name
        else:
            res = orc.ssa_run(h, J, off, p, int(c["seed"]), None, True, False)
        assert res.cycles_used == int(c["cycles_used"]), name
        assert res.best_energy == float(c["best_energy"]), name
        assert np.array_equal(res.best_state, c["best_state"]), name
        assert np.array_equal(res.trace.view(np.uint64), c["trace"].view(np.uint64)), name


def test_ssa_equals_one_replica_ssqa(orc, golden):
    # test_annealer.cpp:440-468: a flat ladder is SSQA with r = 1, delay 0, jperp 0
    inst = golden("gi_instances")["gi_10_7_1_1.0"]
    h, J, off = inst["h"], inst["J"], float(inst["offset"])
    a = orc.ssa_run(h, J, off, ssa_params(60, i0_min=2.0, i0_max=2.0), 21, None, True, False)
    b = orc.ssqa_run(h, J, off, params(1, 60, jperp_min=0.0, jperp_max=0.0, delay=0, i0=2.0),
                     21, None, True, False)
    assert np.array_equal(a.trace.view(np.uint64), b.trace.view(np.uint64))
    assert np.array_equal(a.best_state, b.best_state) and a.cycles_used == b.cycles_used


def test_ssa_oracle_matches_reference_live(orc, ref):
    rng = np.random.default_rng(99)
    for trial in range(5):
        n = int(rng.integers(1, 20))
        h = rng.uniform(-2, 2, n)
        J = np.triu(rng.uniform(-2, 2, (n, n)), 1)
        J = J + J.T
        p = ssa_params(90, tau=int(rng.integers(1, 9)), beta=float(rng.uniform(0.2, 0.9)),
                       i0_max=float(rng.uniform(2, 40)), n_rnd=float(rng.uniform(0, 2)))
        seed = int(rng.integers(0, 2 ** 63))
        a = ref.ssa_run(h, J, 0.5, p, seed, None, True, False)
        b = orc.ssa_run(h, J, 0.5, p, seed, None, True, False)
        assert np.array_equal(a.trace.view(np.uint64), b.trace.view(np.uint64))
        assert np.array_equal(a.best_state, b.best_state)


def test_numpy_lattice_matches_oracle(orc, golden):
    """oracle/lattice_np.py (the vectorised checker used at full BASELINE
    sizes) against the C restatement: traces, best states, hits, stops."""
    import lattice_np as lnp
    import paper_2302_12454_b200 as sq
    inst = golden("gi_instances")["gi_10_7_1_1.0"]
    cases = [(inst["h"], inst["J"], float(inst["offset"]), dict(r=20, sc=300), [123, 5], 0.0, True),
             (inst["h"], inst["J"], float(inst["offset"]), dict(r=7, sc=120, delay=2,
                                                                bidirectional=True), [9], None,
              False)]
    m = sq.dense_ising(256, 0, 3)
    cases.append((m.h, m.J, m.offset, dict(r=6, sc=40, tau=4), [1, 2, 3], None, False))
    m1 = sq.dense_ising(200, 1, 4)
    cases.append((m1.h, m1.J, m1.offset, dict(r=4, sc=30, tau=2, n_rnd=2.0), [8], None, False))
    for h, J, off, kw, seeds, target, stop in cases:
        p = params(**kw)
        got = lnp.run_lattice(h, J, off, p.r, p.delay, p.n_rnd, p.alpha, bool(p.bidirectional),
                              p.sc, lnp.jperp_schedule(p), lambda c: p.i0, seeds, target, stop)
        for t, s in enumerate(seeds):
            o = orc.ssqa_run(h, J, off, p, s, target, True, stop)
            g = got[t]
            assert (g.best_energy, g.best_replica, g.reached_target, g.first_hit_cycle,
                    g.cycles_used) == (o.best_energy, o.best_replica, o.reached_target,
                                       o.first_hit_cycle, o.cycles_used), (kw, s)
            assert np.array_equal(g.best_state, o.best_state)
            assert np.array_equal(g.trace.reshape(-1).view(np.uint64), o.trace.view(np.uint64))
