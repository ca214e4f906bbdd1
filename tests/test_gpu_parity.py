"""Bit-exact parity of the CUDA engine against the CPU oracle and the
reference's own fixtures.  Every call goes through the C ABI
(include/ssqa_cuda.h) via paper_2302_12454_b200._lib.

Bar: bitwise equality of spins, accumulators (as uint64 bit patterns),
energies, traces, best states and per-trial outcomes -- the path is exact
(SURVEY.md section 7), so there is no tolerance anywhere in this file.
"""
import numpy as np
import pytest

import paper_2302_12454_b200 as sq
from paper_2302_12454_b200 import _lib
from oracle_py import params, ssa_params

pytestmark = pytest.mark.gpu

ENGINES = [_lib.ENGINE_SIMT, _lib.ENGINE_TCGEN05]


def engine_ok(engine, n=128, r=20):
    """Probe whether `engine` accepts this shape (tcgen05 may not, yet)."""
    m = sq.IsingModel(n)
    prob = sq.Problem(m)
    try:
        b = sq.Batch(prob, sq.SsqaParams(r=r, sc=1), 1, engine=engine)
        b.close()
        return True
    except _lib.SsqaInvalidArgument:
        return False


@pytest.fixture(params=ENGINES, ids=["simt", "tcgen05"])
def engine(request):
    if not engine_ok(request.param):
        pytest.skip("engine unavailable for this build")
    return request.param


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def to_sq(p):
    return sq.SsqaParams(r=p.r, jperp_min=p.jperp_min, jperp_max=p.jperp_max, beta=p.beta,
                         tau=p.tau, delay=p.delay, i0=p.i0, n_rnd=p.n_rnd, alpha=p.alpha,
                         sc=p.sc, bidirectional=bool(p.bidirectional))


def test_init_lattice_matches_oracle(orc, engine):
    for n, r, d, T in [(1, 1, 0, 1), (100, 20, 1, 7), (130, 3, 2, 5), (300, 33, 1, 3)]:
        prob = sq.Problem(sq.IsingModel(n))
        b = sq.Batch(prob, sq.SsqaParams(r=r, delay=d, sc=1), T, engine=engine)
        seeds = [1000 + 17 * t for t in range(T)]
        b.set_seeds(seeds)
        b.init()
        for t in range(T):
            s, a, h, c = b.read_lattice(t)
            s0, a0, h0 = orc.init_lattice(n, r, d, seeds[t])
            assert np.array_equal(s, s0) and np.array_equal(a, a0) and np.array_equal(h, h0)
            assert c == 0


def test_lattice_trajectories_match_reference(golden, engine):
    """Per-step sigma / acc / energies against tests/golden/lattice_traj.npz."""
    for name, c in golden("lattice_traj").items():
        n, r, d = int(c["n"]), int(c["r"]), int(c["delay"])
        m = sq.IsingModel.from_arrays(c["h"], c["J"], float(c["offset"]))
        p = sq.SsqaParams(r=r, delay=d, alpha=float(c["alpha"]), bidirectional=bool(c["bidir"]),
                          sc=1)
        if str(c["kind"]) == "real":
            with pytest.raises(ValueError):
                sq.Problem(m)
            continue
        b = sq.Batch(sq.Problem(m), p, 1, engine=engine)
        b.set_seeds([int(c["seed"])])
        b.init()
        s, a, h, cyc = b.read_lattice(0)
        assert np.array_equal(s, c["sigma"][0]), name
        for t in range(len(c["jperp"])):
            b.sweep_with(float(c["jperp"][t]), float(c["i0"][t]))
            s, a, h, cyc = b.read_lattice(0)
            assert cyc == t + 1
            assert np.array_equal(s, c["sigma"][t + 1]), (name, t)
            assert np.array_equal(bits(a), bits(c["acc"][t + 1])), (name, t)
            e = b.energies()[0]
            assert np.array_equal(bits(e), bits(c["energy"][t])), (name, t)
        assert np.array_equal(h, c["hist_final"]), name


def test_batched_sweeps_match_oracle_per_trial(orc, engine):
    """Many trials in one batch: every trial's lattice equals the oracle's,
    step by step, on a GI instance (C1 shape, fewer trials)."""
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    for p in (params(20, 1), params(7, 1, delay=2, bidirectional=True), params(5, 1, delay=0)):
        T = 9
        seeds = [int(x) for x in np.random.default_rng(p.r).integers(0, 2 ** 63, T)]
        b = sq.Batch(sq.Problem(m), to_sq(p), T, engine=engine)
        b.set_seeds(seeds)
        b.init()
        states = [orc.init_lattice(m.n, p.r, p.delay, s) for s in seeds]
        cyc = 0
        for step in range(6):
            b.sweep(25 if step else 1)
            count = 25 if step else 1
            for t in range(T):
                s, a, h = states[t]
                c0 = cyc
                for c in range(c0, c0 + count):
                    orc.ssqa_sweep(m.h, m.J, m.offset, orc.jperp_schedule(c, p), p, seeds[t], c,
                                   s, a, h, c)
            cyc += count
            for t in (0, T // 2, T - 1):
                s, a, h, c = b.read_lattice(t)
                so, ao, ho = states[t]
                assert c == cyc
                assert np.array_equal(s, so) and np.array_equal(bits(a), bits(ao)), (p.r, t, cyc)
                assert np.array_equal(h, ho)
            e = b.energies()
            for t in range(T):
                eo = orc.replica_energies(m.h, m.J, m.offset, p.r, states[t][0])
                assert np.array_equal(bits(e[t]), bits(eo))


def test_runs_match_reference_fixtures(golden, engine):
    """ssqa_run KATs incl. traces, best states, stop-at-target."""
    gi = golden("gi_instances")
    for name, c in golden("runs").items():
        if name.startswith("gi"):
            m = sq.gi_ising(int(c["n_nodes"]), 0.5, int(c["gi_seed"]), True, float(c["c"]),
                            float(c["c"]))
            kw = {k[2:]: (v.item() if hasattr(v, "item") else v)
                  for k, v in c.items() if k.startswith("p_")}
            p = sq.SsqaParams(**kw)
            res = sq.ssqa_run(m, p, int(c["seed"]), float(c["target"]),
                              sq.RunOptions(True, bool(c["stop"])), engine=engine)
            assert res.reached_target == bool(c["reached"]), name
            assert res.first_hit_cycle == int(c["first_hit"]), name
            assert res.cycles_used == int(c["cycles_used"]), name
        else:
            m = sq.IsingModel.from_arrays(c["h"], c["J"], float(c["offset"]))
            p = sq.SsqaParams(r=int(c["p_r"]), sc=int(c["p_sc"]), tau=int(c["p_tau"]))
            res = sq.ssqa_run(m, p, int(c["seed"]), None, sq.RunOptions(True, False),
                              engine=engine)
            assert res.cycles_used == int(c["cycles_used"])
        assert res.best_energy == float(c["best_energy"]), name
        assert res.best_replica == int(c["best_replica"]), name
        assert np.array_equal(res.best_state, c["best_state"]), name
        assert np.array_equal(bits(res.trace_energy), bits(c["trace"])), name
    _ = gi


def test_run_trials_matches_reference_kat(golden, engine):
    """run_trials({r=20, ec=20000, n=10, permute, c=1, gi_seed=7, 100 trials,
    base 1000}) -> p_s 0.80 and identical per-trial outcomes."""
    t = golden("trials")["trials_gi10"]
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    outs, p_s, t_mean, tts = sq.run_trials(m, sq.SsqaParams(r=20), 100, 20000, 1000,
                                           engine=engine)
    assert p_s == 0.80
    assert [o.seed for o in outs] == [int(x) for x in t["seed"]]
    assert [int(o.reached_target) for o in outs] == [int(x) for x in t["reached"]]
    assert [o.first_hit_cycle for o in outs] == [int(x) for x in t["first_hit"]]
    assert np.array_equal(bits([o.best_energy for o in outs]), bits(t["best_energy"]))
    assert tts.kind == "finite" and t_mean > 0


EPILOGUES = [("simt", "auto"), ("tcgen05", "auto"), ("tcgen05", "table"), ("tcgen05", "fp64"),
             ("tcgen05", "ctable")]


@pytest.fixture(params=EPILOGUES, ids=["-".join(e) for e in EPILOGUES])
def engine_epi(request, monkeypatch):
    """Engine and tcgen05 fast epilogue: the engine's choice, the table path
    (integer clamps + per-cycle smem table), the FP64 path (update_fast2) or the
    clamped table of the issue-lean epilogue."""
    eng, epi = request.param
    engine = ENGINES[0] if eng == "simt" else ENGINES[1]
    if not engine_ok(engine):
        pytest.skip("engine unavailable for this build")
    if epi == "table":
        sq.tune(tab=1)
    elif epi == "fp64":
        sq.tune(tab=0)
    elif epi == "ctable":  # clamped table inside the issue-lean epilogue (epi_v4 TBL)
        sq.tune(tab=2)
    return engine


def test_full_runs_match_oracle_many_trials(orc, engine_epi):
    """A 48-trial batch at N=100 and N=400 (C1/C2 shapes, shortened): every
    trial equals the oracle's ssqa_run."""
    engine = engine_epi
    for nn, R, sc, T in [(10, 20, 300, 48), (20, 20, 60, 6)]:
        m = sq.gi_ising(nn, 0.5, 7, True, 1.0, 1.0)
        p = params(R, sc)
        seeds = list(range(500, 500 + T))
        res = sq.ssqa_run_batch(m, to_sq(p), seeds, 0.0, sq.RunOptions(True, False),
                                engine=engine)
        for t in range(0, T, 1 if T < 10 else 5):
            o = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[t], 0.0, True, False)
            r = res[t]
            assert (r.best_energy, r.best_replica, r.reached_target, r.first_hit_cycle,
                    r.cycles_used) == (o.best_energy, o.best_replica, o.reached_target,
                                       o.first_hit_cycle, o.cycles_used), t
            assert np.array_equal(r.best_state, o.best_state)
            assert np.array_equal(bits(r.trace_energy), bits(o.trace))
        # AnnealResult::trace (annealer.cpp:343): one TracePoint per replica and
        # scanned cycle, cycle-major, with the cycle's jperp (annealer.cpp:349)
        o = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[0], 0.0, True, False)
        tp = res[0].trace
        assert len(tp) == (o.cycles_used + 1) * R
        assert [(x.cycle, x.replica) for x in tp] == [(c, k) for c in range(o.cycles_used + 1)
                                                      for k in range(R)]
        assert np.array_equal(bits([x.energy for x in tp]), bits(o.trace))
        assert np.array_equal(bits([x.jperp for x in tp]),
                              bits([orc.jperp_schedule(x.cycle, p) for x in tp]))


@pytest.fixture(params=["auto", "int8"])
def operands(request, monkeypatch):
    """tcgen05 operand format: the engine's choice (FP4, FP4 pair) or int8."""
    if request.param == "int8":
        sq.tune(fp4=0)
    return request.param


@pytest.mark.parametrize("engine,ops", [(ENGINES[0], "auto"), (ENGINES[1], "auto"),
                                        (ENGINES[1], "int8")],
                         ids=["simt", "tcgen05", "tcgen05-int8"])
def test_dense_integer_model_matches_oracle(orc, monkeypatch, engine, ops):
    """C4-style dense int[-8,7] couplings (the reference's plain-double path);
    on tcgen05 as FP4 pairs (J' = A1 + A2) and as int8."""
    if not engine_ok(engine):
        pytest.skip("engine unavailable for this build")
    if ops == "int8":
        sq.tune(fp4=0)
    m = sq.dense_ising(200, 0, 3)
    p = params(8, 40, tau=5, bidirectional=True)
    seeds = [11, 12, 13]
    res = sq.ssqa_run_batch(m, to_sq(p), seeds, None, sq.RunOptions(True, False),
                            engine=engine)
    for t, s in enumerate(seeds):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, s, None, True, False)
        assert res[t].best_energy == o.best_energy
        assert np.array_equal(res[t].best_state, o.best_state)
        assert np.array_equal(bits(res[t].trace_energy), bits(o.trace))


def test_stop_at_target_and_unreachable(orc, engine):
    # test_annealer.cpp:470-508: hit at cycle 0, unreachable targets, fixed budget
    rng = np.random.default_rng(23)
    h = rng.integers(-8, 9, 4) / 4.0
    J = np.triu(rng.integers(-8, 9, (4, 4)) / 4.0, 1)
    m = sq.IsingModel.from_arrays(h, J + J.T, 0.5)
    p = sq.SsqaParams(r=3, sc=40)
    lat = sq.init_lattice(4, 3, 1, 31)
    e0 = sq.replica_energies(lat, m).min()
    res = sq.ssqa_run(m, p, 31, float(e0), engine=engine)
    assert res.reached_target and res.first_hit_cycle == 0 and res.cycles_used == 0
    miss = sq.ssqa_run(m, p, 31, -1e6, engine=engine)
    assert not miss.reached_target and miss.first_hit_cycle == -1 and miss.cycles_used == 40
    q = params(3, 40)
    for stop in (True, False):
        o = orc.ssqa_run(m.h, m.J, m.offset, q, 31, -1.0, False, stop)
        r = sq.ssqa_run(m, p, 31, -1.0, sq.RunOptions(False, stop), engine=engine)
        assert (r.reached_target, r.first_hit_cycle, r.cycles_used, r.best_energy) == \
            (o.reached_target, o.first_hit_cycle, o.cycles_used, o.best_energy)


def test_device_kats_clamp_and_delay(engine):
    # test_annealer.cpp:219-304 through the device per-step API
    p = sq.SsqaParams(r=1, sc=4, n_rnd=0.0, delay=0, jperp_min=0.0, jperp_max=0.0)
    up = sq.IsingModel(1)
    up.set_bias(0, 5.0)
    lat = sq.init_lattice(1, 1, 0, 3)
    sq.ssqa_sweep(lat, up, 0.0, p, 3, 0, engine=engine)
    assert lat.acc(0, 0) == 1.0 and lat.spin(0, 0) == 1.0
    down = sq.IsingModel(1)
    down.set_bias(0, -5.0)
    lat = sq.init_lattice(1, 1, 0, 3)
    sq.ssqa_sweep(lat, down, 0.0, p, 3, 0, engine=engine)
    assert lat.acc(0, 0) == -2.0 and lat.spin(0, 0) == -1.0
    half = sq.SsqaParams(**{**p.__dict__, "alpha": 0.5})
    lat = sq.init_lattice(1, 1, 0, 3)
    sq.ssqa_sweep(lat, up, 0.0, half, 3, 0, engine=engine)
    assert lat.acc(0, 0) == 1.5
    # delayed coupling, test_annealer.cpp:266-292
    m = sq.IsingModel(1)
    q = sq.SsqaParams(r=2, sc=4, n_rnd=0.0, delay=1)
    lat = sq.init_lattice(1, 2, 1, 5)
    lat.sigma[:] = [-1.0, -1.0]
    lat.is_acc[:] = 0.0
    lat.history[0] = [1.0, -1.0]
    lat.history[1] = [-1.0, 1.0]
    sq.ssqa_sweep(lat, m, 0.7, q, 5, 0, engine=engine)
    assert lat.acc(0, 0) == -0.7 and lat.acc(0, 1) == 0.7
    assert list(lat.sigma) == [-1.0, 1.0] and list(lat.history[0]) == [-1.0, 1.0]
    assert lat.cycle == 1
    sq.ssqa_sweep(lat, m, 0.7, q, 5, 1, engine=engine)
    assert lat.acc(0, 0) == 0.0 and lat.spin(0, 0) == 1.0
    with pytest.raises(ValueError):
        sq.ssqa_sweep(lat, m, 0.7, q, 5, 7, engine=engine)  # cycle mismatch


def test_unrepresentable_models_are_rejected():
    m = sq.IsingModel(3)
    m.set_coupling(0, 1, 0.1)
    with pytest.raises(ValueError):
        sq.Problem(m)


def test_cpp_facade_program(tmp_path, orc):
    """Compile a reference-style C++ caller against include/ssqa/*.hpp and
    run it: the drop-in claim for C++ users."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "caller.cpp"
    src.write_text(r'''
#include <cstdio>
#include <stdexcept>
#include "ssqa/annealer.hpp"
#include "ssqa/bench.hpp"
#include "ssqa/gi.hpp"
#include "ssqa_tune.h"
using namespace ssqa;
int main() {
  IsingModel m = qubo_to_ising(build_gi_qubo(generate_gi(10, 0.5, 7, true, 1.0, 1.0)));
  SsqaParams p; p.r = 20; p.sc = 1000;
  RunOptions o; o.record_trace = true; o.stop_at_target = false;
  AnnealResult r = ssqa_run(m, p, 123, 0.0, o);
  std::printf("%d %ld %.17g %d %zu\n", int(r.reached_target), r.first_hit_cycle,
              r.best_energy, r.best_replica, r.trace.size());
  BenchConfig c; c.ssqa.r = 20; c.problem.n_nodes = 10; c.problem.permute = true;
  c.problem.c1 = c.problem.c2 = 1.0; c.problem.fresh_instance = false; c.problem.gi_seed = 7;
  c.trials = 100; c.ec = 20000; c.base_seed = 1000;
  BenchRecord rec = run_trials(c);
  std::printf("%.17g\n", rec.p_s);
  bool threw = false;
  try { SsqaParams bad; bad.r = 0; bad.sc = 5; ssqa_run(m, bad, 1); }
  catch (const std::invalid_argument&) { threw = true; }
  std::printf("%d\n", int(threw));
  SsaParams s; s.sc = 3000; s.tau = 25;
  AnnealResult a = ssa_run(m, s, 1, 0.0, o);
  std::printf("%d %ld %.17g %zu\n", int(a.reached_target), a.first_hit_cycle, a.best_energy,
              a.trace.size());
  BenchConfig cs = c; cs.engine = Engine::kSsa; cs.ssa.tau = 25; cs.trials = 20; cs.ec = 3000;
  BenchRecord rs = run_trials(cs);
  std::printf("%d %ld %d %d\n", rs.r, rs.ec, rs.tau, int(rs.per_trial.size()));
  for (const TrialOutcome& t : rs.per_trial)
    std::printf("%d %ld %.17g\n", int(t.reached_target), t.first_hit_cycle, t.best_energy);
  BenchConfig cf; cf.ssqa.r = 20; cf.problem.n_nodes = 10; cf.trials = 64; cf.ec = 20000;
  cf.base_seed = 1000;  // reference defaults: fresh instances, permute off, c1 = c2 = 0.75
  BenchRecord rf = run_trials(cf);
  std::printf("FRESH %.17g\n", rf.p_s);
  for (const TrialOutcome& t : rf.per_trial)
    std::printf("F %d %ld %.17g\n", int(t.reached_target), t.first_hit_cycle, t.best_energy);
  BenchConfig cf2 = cf;
  cf2.devices = {0, 0};  // two host threads, one trial block each (same GPU here)
  BenchRecord rf2 = run_trials(cf2);
  std::printf("FRESH2 %.17g\n", rf2.p_s);
  for (const TrialOutcome& t : rf2.per_trial)
    std::printf("G %d %ld %.17g\n", int(t.reached_target), t.first_hit_cycle, t.best_energy);
  // J' row shards driven from C++ (ssqa_run_row_sharded): one shard, and two
  // shards on this GPU (a repeated device takes the copy exchange) against the
  // unsharded batch -- energies of every cycle, best states, first hits
  IsingModel m2 = qubo_to_ising(build_gi_qubo(generate_gi(16, 0.5, 5, true, 1.0, 1.0)));
  SsqaParams p2; p2.r = 6; p2.sc = 80;
  std::vector<uint64_t> sd = {11, 12, 13};
  std::vector<AnnealResult> whole = ssqa_run_batch(m2, p2, sd, 0.0, o);
  int rows_ok = 0;
  for (const std::vector<int>& devs : {std::vector<int>{0}, std::vector<int>{0, 0}}) {
    std::vector<AnnealResult> sh = ssqa_run_row_sharded(m2, p2, sd, devs, 0.0, o);
    bool same = sh.size() == whole.size();
    for (size_t t = 0; same && t < sh.size(); ++t) {
      same = sh[t].best_energy == whole[t].best_energy && sh[t].best_replica == whole[t].best_replica &&
             sh[t].first_hit_cycle == whole[t].first_hit_cycle && sh[t].best_state == whole[t].best_state &&
             sh[t].trace.size() == whole[t].trace.size();
      for (size_t k = 0; same && k < sh[t].trace.size(); ++k)
        same = sh[t].trace[k].energy == whole[t].trace[k].energy;
    }
    rows_ok += same ? 1 : 0;
  }
  // the NCCL exchange itself (libnccl bound at run time, group calls on the
  // engine stream), forced for the single device of this box
  ssqa_tune_set("nccl1", 1);
  {
    std::vector<AnnealResult> sh = ssqa_run_row_sharded(m2, p2, sd, {0}, 0.0, o);
    bool same = sh.size() == whole.size();
    for (size_t t = 0; same && t < sh.size(); ++t)
      same = sh[t].best_energy == whole[t].best_energy && sh[t].best_state == whole[t].best_state &&
             sh[t].first_hit_cycle == whole[t].first_hit_cycle;
    rows_ok += same ? 1 : 0;
  }
  ssqa_tune_reset();
  std::printf("ROWS %d\n", rows_ok);
  return 0;
}
''')
    exe = tmp_path / "caller"
    libdir = os.path.join(root, "paper_2302_12454_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{root}/include", str(src), "-o", str(exe),
                    f"-L{libdir}", "-lssqa_b200", f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True,
                         env={**os.environ, "NCCL_DEBUG": "WARN"}).stdout.split()
    assert out[:5] == ["1", "304", "0", "4", "20020"]
    assert float(out[5]) == 0.80
    assert out[6] == "1"
    # ssa_run on the same instance (reference fixture ssa_runs/gi10_tau25: hit at 1629)
    assert out[7:9] == ["1", "1629"] and out[10] == "3001"
    assert out[11:15] == ["1", "3000", "25", "20"]
    p = ssa_params(3000, tau=25)
    m_h, m_J, m_off = _gi10()
    fi = out.index("FRESH")
    rows = out[15:fi]
    fresh = golden_fresh()["fresh_gi10"]
    assert float(out[fi + 1]) == float(fresh["p_s"])
    f2 = out.index("FRESH2")
    assert out[f2 + 1] == out[fi + 1]
    ri = out.index("ROWS")
    assert out[ri + 1] == "3"  # one shard, two emulated shards and the NCCL path equal the batch
    out = out[:out.index("NCCL")] if "NCCL" in out[:ri] else out[:ri]  # (NCCL's version banner)
    g = out[f2 + 2:]
    assert [x for k, x in enumerate(g) if k % 4] == [x for k, x in enumerate(out[fi + 2:f2]) if k % 4]
    fr = out[fi + 2:]
    for t in range(64):
        assert fr[4 * t] == "F"
        assert (int(fr[4 * t + 1]), int(fr[4 * t + 2]), float(fr[4 * t + 3])) == (
            int(fresh["reached"][t]), int(fresh["first_hit"][t]), float(fresh["best_energy"][t]))
    for t in range(20):
        o = orc.ssa_run(m_h, m_J, m_off, p, 1000 + t, 0.0, False, False)
        assert (rows[3 * t] == "1", int(rows[3 * t + 1]), float(rows[3 * t + 2])) == \
            (o.reached_target, o.first_hit_cycle, o.best_energy), t


def golden_fresh():
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                             "trials_fresh.npz"))
    out = {}
    for key in z.files:
        case, field = key.split("/", 1)
        out.setdefault(case, {})[field] = z[key]
    return out


def _gi10():
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    return m.h, m.J, m.offset


# ---- SSA engine (annealer.cpp:489-501): r = 1, jperp = 0, i0 ladder ----

def to_sq_ssa(p):
    return sq.SsaParams(i0_min=p.i0_min, i0_max=p.i0_max, beta=p.beta, tau=p.tau,
                        n_rnd=p.n_rnd, alpha=p.alpha, sc=p.sc)


def test_ssa_runs_match_reference_fixtures(golden, engine):
    for name, c in golden("ssa_runs").items():
        if name.startswith("sched"):
            continue
        kw = {k[2:]: v.item() for k, v in c.items() if k.startswith("p_")}
        p = sq.SsaParams(**kw)
        if "h" in c:
            m = sq.IsingModel.from_arrays(c["h"], c["J"], float(c["offset"]))
            res = sq.ssa_run(m, p, int(c["seed"]), None, sq.RunOptions(True, False),
                             engine=engine)
        else:
            m = sq.gi_ising(int(c["n_nodes"]), 0.5, int(c["gi_seed"]), True, float(c["c"]),
                            float(c["c"]))
            res = sq.ssa_run(m, p, int(c["seed"]), float(c["target"]),
                             sq.RunOptions(True, bool(c["stop"])), engine=engine)
            assert res.reached_target == bool(c["reached"]), name
            assert res.first_hit_cycle == int(c["first_hit"]), name
        assert res.cycles_used == int(c["cycles_used"]), name
        assert res.best_energy == float(c["best_energy"]), name
        assert res.best_replica == 0, name
        assert np.array_equal(res.best_state, c["best_state"]), name
        assert np.array_equal(bits(res.trace_energy), bits(c["trace"])), name


def test_ssa_equals_one_replica_ssqa(engine):
    # test_annealer.cpp:440-468, on the device
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    opts = sq.RunOptions(True, False)
    a = sq.ssa_run(m, sq.SsaParams(i0_min=2.0, i0_max=2.0, sc=60), 21, None, opts,
                   engine=engine)
    b = sq.ssqa_run(m, sq.SsqaParams(r=1, delay=0, jperp_min=0.0, jperp_max=0.0, i0=2.0,
                                     sc=60), 21, None, opts, engine=engine)
    assert a.best_energy == b.best_energy and a.cycles_used == b.cycles_used
    assert np.array_equal(a.best_state, b.best_state)
    assert np.array_equal(bits(a.trace_energy), bits(b.trace_energy))


def test_ssa_many_trials_match_oracle(orc, engine):
    """Batches wider than the SM count (several single-replica trials per
    column tile) at N=100 and N=400."""
    for nn, sc, T, kw in [(10, 400, 300, dict(tau=7)), (20, 120, 9, dict(beta=0.3, i0_max=30.0)),
                          (10, 250, 40, dict(tau=3, beta=0.7, i0_max=40.0, n_rnd=2.0))]:
        m = sq.gi_ising(nn, 0.5, 7, True, 1.0, 1.0)
        p = ssa_params(sc, **kw)
        seeds = list(range(900, 900 + T))
        res = sq.ssa_run_batch(m, to_sq_ssa(p), seeds, 0.0, sq.RunOptions(True, False),
                               engine=engine)
        for t in range(0, T, 1 if T < 50 else 7):
            o = orc.ssa_run(m.h, m.J, m.offset, p, seeds[t], 0.0, True, False)
            r = res[t]
            assert (r.best_energy, r.reached_target, r.first_hit_cycle, r.cycles_used) == \
                (o.best_energy, o.reached_target, o.first_hit_cycle, o.cycles_used), t
            assert np.array_equal(r.best_state, o.best_state)
            assert np.array_equal(bits(r.trace_energy), bits(o.trace))


def test_ssa_mid_size_geometry_matches_oracle(orc):
    """SSA batches (one replica per trial) on a 2048-spin model: make_geom's
    search packs many trials per column tile and splits the rows over the SMs;
    traces, hits and best states of a few trials against the C oracle."""
    n = 2048
    rng = np.random.default_rng(11)
    J = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    J[iu] = rng.integers(-1, 2, len(iu[0])) * 0.5
    J = J + J.T
    m = sq.IsingModel.from_arrays(rng.integers(-4, 5, n) * 0.5, J, 0.0)
    for T, sc, kw in [(300, 30, dict(tau=5)), (37, 24, dict(tau=3, beta=0.6, i0_max=60.0))]:
        p = ssa_params(sc, **kw)
        seeds = list(range(50, 50 + T))
        res = sq.ssa_run_batch(m, to_sq_ssa(p), seeds, None, sq.RunOptions(True, False),
                               engine=_lib.ENGINE_TCGEN05)
        for t in (0, T // 2, T - 1):
            o = orc.ssa_run(m.h, m.J, m.offset, p, seeds[t], None, True, False)
            r = res[t]
            assert (r.best_energy, r.cycles_used) == (o.best_energy, o.cycles_used), (T, t)
            assert np.array_equal(r.best_state, o.best_state)
            assert np.array_equal(bits(r.trace_energy), bits(o.trace))


def test_ssa_batch_sweeps_follow_the_ladder(orc, engine):
    """Per-step API on an SSA batch: ssqa_batch_sweep uses i0_schedule(cycle)."""
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    p = sq.SsaParams(tau=2, sc=50)
    q = params(1, 50, jperp_min=0.0, jperp_max=0.0, delay=0)
    prob = sq.Problem(m)
    b = sq.Batch(prob, p, 3, engine=engine)
    seeds = [5, 6, 7]
    b.set_seeds(seeds)
    b.init()
    states = [orc.init_lattice(m.n, 1, 0, s) for s in seeds]
    cyc = 0
    for step in range(12):
        b.sweep(1)
        i0 = sq.i0_schedule(cyc, p)
        for t, s in enumerate(seeds):
            sg, ac, hi = states[t]
            q.i0 = i0
            orc.ssqa_sweep(m.h, m.J, m.offset, 0.0, q, s, cyc, sg, ac, hi, cyc)
        cyc += 1
        for t in range(3):
            sg, ac, hi, c = b.read_lattice(t)
            assert c == cyc
            assert np.array_equal(bits(sg), bits(states[t][0])), (step, t)
            assert np.array_equal(bits(ac), bits(states[t][1])), (step, t)


def test_ssa_run_trials_matches_oracle(orc, engine):
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    outs, p_s, t_mean, tts = sq.run_trials(m, sq.SsaParams(tau=25), 24, 3000, 1000,
                                           engine=engine)
    p = ssa_params(3000, tau=25)
    hits = 0
    for t, o in enumerate(outs):
        r = orc.ssa_run(m.h, m.J, m.offset, p, 1000 + t, 0.0, False, False)
        assert (o.seed, o.reached_target, o.first_hit_cycle, o.best_energy) == \
            (1000 + t, r.reached_target, r.first_hit_cycle, r.best_energy)
        hits += r.reached_target
    assert p_s == hits / 24


def test_stop_at_target_many_tiles_drain(orc, engine):
    """300 trials (3 per column tile) with stop_at_target: tiles whose trials
    have all stopped end early (one drained pass) while others keep running;
    every trial still equals the oracle's ssqa_run."""
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    p = params(20, 1500)
    seeds = list(range(7000, 7300))
    res = sq.ssqa_run_batch(m, to_sq(p), seeds, 0.0, sq.RunOptions(True, True), engine=engine)
    stopped = 0
    for t in range(0, 300, 3):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[t], 0.0, True, True)
        r = res[t]
        assert (r.best_energy, r.best_replica, r.reached_target, r.first_hit_cycle,
                r.cycles_used) == (o.best_energy, o.best_replica, o.reached_target,
                                   o.first_hit_cycle, o.cycles_used), t
        assert np.array_equal(r.best_state, o.best_state)
        assert np.array_equal(bits(r.trace_energy), bits(o.trace))
        stopped += r.cycles_used < 1500
    assert stopped > 10


# ---- tcgen05 row split: rs CTAs per column tile (cross-CTA row readiness,
# global energy sums, scan by the last arriving CTA) ----

@pytest.fixture
def row_split(monkeypatch):
    def force(rs):
        sq.tune(rs=rs)
    return force


def _row_split_cases():
    """(rs, operands, cluster, epilogue) combinations that exist: every split
    with both operand formats and every cluster mode (odd splits never pair),
    on the default table epilogue; the FP64 epilogue once per even split."""
    out = []
    for rs in (2, 3, 4):
        for ops in ("auto", "int8"):
            for cl in ("pairs", "single"):
                if not (rs == 3 and cl == "pairs"):
                    out.append((rs, ops, cl, "auto"))
        if rs % 2 == 0:
            out.append((rs, "auto", "pairs", "fp64"))
    return out


@pytest.mark.parametrize("rs,operands,cluster,epi", _row_split_cases(),
                         ids=["-".join(map(str, c)) for c in _row_split_cases()])
def test_row_split_runs_match_oracle(orc, row_split, monkeypatch, rs, operands, cluster, epi):
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    if operands == "int8":
        sq.tune(fp4=0)
    if cluster == "single":
        sq.tune(cta2=0)
    if cluster == "pairs":  # small shapes pair only on request
        sq.tune(cta2=1)
    if epi == "fp64":
        sq.tune(tab=0)
    row_split(rs)
    cases = [(sq.gi_ising(20, 0.5, 7, True, 1.0, 1.0), params(20, 60), [41, 42, 43, 44, 45, 46]),
             (sq.dense_ising(400, 0, 5), params(6, 30, tau=4, bidirectional=True), [7, 8, 9])]
    for m, p, seeds in cases:
        # a target trial 0 reaches, so stop_at_target freezes some trials early
        hit = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[0], None, False, False).best_energy
        for target, stop in ((-1e9, False), (float(hit), True)):
            res = sq.ssqa_run_batch(m, to_sq(p), seeds, target, sq.RunOptions(True, stop),
                                    engine=_lib.ENGINE_TCGEN05)
            for t, sd in enumerate(seeds):
                o = orc.ssqa_run(m.h, m.J, m.offset, p, sd, target, True, stop)
                r = res[t]
                assert (r.best_energy, r.best_replica, r.reached_target, r.first_hit_cycle,
                        r.cycles_used) == (o.best_energy, o.best_replica, o.reached_target,
                                           o.first_hit_cycle, o.cycles_used), (rs, m.n, stop, t)
                assert np.array_equal(r.best_state, o.best_state)
                assert np.array_equal(bits(r.trace_energy), bits(o.trace))


def test_row_split_per_step_sweeps(orc, row_split):
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    row_split(3)
    m = sq.dense_ising(400, 0, 11)
    p = params(5, 10, delay=2)
    prob = sq.Problem(m)
    b = sq.Batch(prob, to_sq(p), 2, engine=_lib.ENGINE_TCGEN05)
    seeds = [3, 4]
    b.set_seeds(seeds)
    b.init()
    states = [orc.init_lattice(m.n, 5, 2, s) for s in seeds]
    cyc = 0
    for step in range(6):
        jp = orc.jperp_schedule(cyc, p)
        b.sweep(1)
        for t, s in enumerate(seeds):
            sg, ac, hi = states[t]
            orc.ssqa_sweep(m.h, m.J, m.offset, jp, p, s, cyc, sg, ac, hi, cyc)
        cyc += 1
        for t in range(2):
            sg, ac, hi, c = b.read_lattice(t)
            assert c == cyc
            assert np.array_equal(bits(sg), bits(states[t][0])), (step, t)
            assert np.array_equal(bits(ac), bits(states[t][1])), (step, t)


def test_wide_row_split_default_heuristic(orc):
    """N=2048 dense: the default geometry widens the column tile to all 16
    trials and splits its 16 row tiles over 16 CTAs."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    m = sq.dense_ising(2048, 0, 3)
    p = params(8, 12, tau=3)
    seeds = list(range(60, 76))
    res = sq.ssqa_run_batch(m, to_sq(p), seeds, None, sq.RunOptions(True, False),
                            engine=_lib.ENGINE_TCGEN05)
    for t in (0, 7, 15):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[t], None, True, False)
        assert res[t].best_energy == o.best_energy and res[t].best_replica == o.best_replica
        assert np.array_equal(res[t].best_state, o.best_state)
        assert np.array_equal(bits(res[t].trace_energy), bits(o.trace))


# ---- GPU row shards: per-cycle pass / all-gather / merge ----

@pytest.mark.parametrize("nshards", [1, 2, 4])
def test_row_shards_emulated_match_oracle(orc, nshards, operands):
    """Every shard of a G-way J' row shard (run one after another on one GPU,
    exchanging through one buffer) equals the oracle's ssqa_run -- with FP4 /
    FP4-pair shard passes (GI / dense couplings) and forced int8."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    from paper_2302_12454_b200.rowshard import run_emulated_shards
    cases = [(sq.gi_ising(20, 0.5, 7, True, 1.0, 1.0), params(20, 40), [31, 32, 33], True),
             (sq.dense_ising(512, 0, 9), params(6, 25, tau=3, delay=2, bidirectional=True),
              [5, 6], False)]
    for m, p, seeds, stop in cases:
        target = float(orc.ssqa_run(m.h, m.J, m.offset, p, seeds[0], None, False,
                                    False).best_energy) if stop else None
        runs = run_emulated_shards(m, to_sq(p), seeds, nshards, target,
                                   sq.RunOptions(True, stop))
        for t, sd in enumerate(seeds):
            o = orc.ssqa_run(m.h, m.J, m.offset, p, sd, target, True, stop)
            for g, res in enumerate(runs):
                r = res[t]
                assert (r.best_energy, r.best_replica, r.reached_target, r.first_hit_cycle,
                        r.cycles_used) == (o.best_energy, o.best_replica, o.reached_target,
                                           o.first_hit_cycle, o.cycles_used), (nshards, g, t)
                assert np.array_equal(r.best_state, o.best_state), (nshards, g, t)
                assert np.array_equal(bits(r.trace_energy), bits(o.trace)), (nshards, g, t)


def test_row_sharded_single_rank(orc):
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    from paper_2302_12454_b200.rowshard import run_row_sharded
    m = sq.dense_ising(256, 0, 2)
    p = params(8, 30, tau=5)
    res = run_row_sharded(m, to_sq(p), [3, 4], None, sq.RunOptions(True, False))
    # the same run captured as one CUDA graph (rowshard.capture_run) and replayed
    gres = run_row_sharded(m, to_sq(p), [3, 4], None, sq.RunOptions(True, False), graph=True)
    for t, sd in enumerate([3, 4]):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, sd, None, True, False)
        for r in (res[t], gres[t]):
            assert r.best_energy == o.best_energy
            assert np.array_equal(bits(r.trace_energy), bits(o.trace))
            assert np.array_equal(r.best_state, o.best_state)


@pytest.mark.parametrize("exchange", ["p2p", "direct"])
@pytest.mark.parametrize("nshards", [1, 2, 4])
def test_row_shards_peer_push_match_oracle(orc, nshards, exchange):
    """The exchanges without a collective library, G GPUs' regions on one GPU:
    "p2p" -- the pack kernel stores into every GPU's region + flags, the merge
    waits on its flags (ssqa_batch_shard_pass_to / _merge_from); "direct" --
    the tcgen05 epilogue itself stores every spin word into every GPU's FP4
    slot and its last CTA pushes the energy partials + flags
    (ssqa_batch_shard_pass_direct / _merge_direct).  Every shard equals the
    oracle, incl. stop-at-target; GI (FP4) and dense int[-8,7] (FP4 pairs)."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    from paper_2302_12454_b200.rowshard import run_emulated_shards
    cases = [(sq.gi_ising(20, 0.5, 7, True, 1.0, 1.0), params(20, 40), [31, 32, 33], True),
             (sq.dense_ising(512, 0, 9), params(6, 25, tau=3, delay=2, bidirectional=True),
              [5, 6], False)]
    for m, p, seeds, stop in cases:
        target = float(orc.ssqa_run(m.h, m.J, m.offset, p, seeds[0], None, False,
                                    False).best_energy) if stop else None
        runs = run_emulated_shards(m, to_sq(p), seeds, nshards, target,
                                   sq.RunOptions(True, stop), exchange=exchange)
        for t, sd in enumerate(seeds):
            o = orc.ssqa_run(m.h, m.J, m.offset, p, sd, target, True, stop)
            for g, res in enumerate(runs):
                r = res[t]
                assert (r.best_energy, r.best_replica, r.reached_target, r.first_hit_cycle,
                        r.cycles_used) == (o.best_energy, o.best_replica, o.reached_target,
                                           o.first_hit_cycle, o.cycles_used), (nshards, g, t)
                assert np.array_equal(r.best_state, o.best_state), (nshards, g, t)
                assert np.array_equal(bits(r.trace_energy), bits(o.trace)), (nshards, g, t)


@pytest.mark.parametrize("exchange", ["p2p", "direct"])
def test_row_sharded_single_rank_peer_push(orc, exchange):
    """run_row_sharded(exchange=...) on one rank: own region, no IPC."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    from paper_2302_12454_b200.rowshard import run_row_sharded
    m = sq.dense_ising(256, 0, 2)
    p = params(8, 30, tau=5)
    res = run_row_sharded(m, to_sq(p), [3, 4], None, sq.RunOptions(True, False),
                          exchange=exchange)
    for t, sd in enumerate([3, 4]):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, sd, None, True, False)
        assert res[t].best_energy == o.best_energy
        assert np.array_equal(bits(res[t].trace_energy), bits(o.trace))


# ---- fresh instance per trial (bench.hpp:28, bench.cpp:387-389) in one batch ----

def test_fresh_instance_run_trials_matches_reference(golden):
    """run_trials with fresh_instance: every trial's own GI instance in one
    multi-instance problem, one device batch; per-trial outcomes equal the
    reference run_trials (fixture from oracle/_ref)."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    for name, c in golden("trials_fresh").items():
        kw = {k[2:]: (v.item() if hasattr(v, "item") else v) for k, v in c.items()
              if k.startswith("k_")}
        outs, p_s, t_mean, tts = sq.run_trials_fresh(
            int(kw["n_nodes"]), sq.SsqaParams(r=int(c["r"])), int(kw["trials"]), int(kw["ec"]),
            int(kw["base_seed"]), permute=bool(kw["permute"]), c1=float(kw["c1"]),
            c2=float(kw["c2"]))
        assert [o.seed for o in outs] == [int(x) for x in c["seed"]], name
        assert [int(o.reached_target) for o in outs] == [int(x) for x in c["reached"]], name
        assert [o.first_hit_cycle for o in outs] == [int(x) for x in c["first_hit"]], name
        assert np.array_equal(bits([o.best_energy for o in outs]), bits(c["best_energy"])), name
        assert p_s == float(c["p_s"]), name


def test_multi_instance_batch_matches_oracle(orc):
    """Direct multi-instance batch: trial t on instance t, traces and best
    states against the oracle's ssqa_run on that instance."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    models = [sq.dense_ising(300, 0, s) for s in (1, 2, 3)]
    p = params(6, 30, tau=4, bidirectional=True)
    seeds = [11, 12, 13]
    prob = sq.Problem.from_models(models)
    assert _lib.lib().ssqa_problem_count(prob._h) == 3
    res = sq.ssqa_run_batch(models[0], to_sq(p), seeds, None, sq.RunOptions(True, False),
                            problem=prob)
    for t, (m, s) in enumerate(zip(models, seeds)):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, s, None, True, False)
        assert res[t].best_energy == o.best_energy, t
        assert np.array_equal(res[t].best_state, o.best_state), t
        assert np.array_equal(bits(res[t].trace_energy), bits(o.trace)), t
    with pytest.raises(ValueError):  # one trial per instance
        sq.Batch(prob, to_sq(p), 2)


def test_cpp_manifest_replay(tmp_path):
    """Manifests (bench.cpp:519-584): the reference-written fixtures replay
    bitwise through the facade's replay_manifest on the GPU; a manifest the
    facade writes replays too; a tampered outcome is reported."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2302_12454_b200 import build as bld
    if not bld.JSON_INC:
        pytest.skip("nlohmann/json not available")
    src = tmp_path / "replay.cpp"
    src.write_text(r'''
#include <cstdio>
#include <fstream>
#include "ssqa/bench.hpp"
using namespace ssqa;
int main(int argc, char** argv) {
  for (int a = 1; a < argc; ++a) {
    std::ifstream f(argv[a]);
    nlohmann::json m = nlohmann::json::parse(f);
    ReplayResult r = replay_manifest(m);
    std::printf("REF %d %s\n", int(r.match), r.mismatch.empty() ? "-" : r.mismatch.c_str());
  }
  BenchConfig c; c.ssqa.r = 16; c.problem.n_nodes = 10; c.trials = 10; c.ec = 16 * 800;
  c.base_seed = 99;
  BenchRecord rec = run_trials(c);
  nlohmann::json m = make_manifest("bench", c, {}, {rec}, {"results.csv"});
  nlohmann::json back = nlohmann::json::parse(m.dump());
  std::printf("OWN %d\n", int(replay_manifest(back).match));
  back["records"][0]["per_trial"][3]["best_energy"] = 1e300;
  ReplayResult bad = replay_manifest(back);
  std::printf("BAD %d %s\n", int(bad.match), bad.mismatch.c_str());
  return 0;
}
''')
    exe = tmp_path / "replay"
    libdir = os.path.join(root, "paper_2302_12454_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{root}/include", f"-I{bld.JSON_INC}",
                    str(src), "-o", str(exe), f"-L{libdir}", "-lssqa_b200",
                    f"-Wl,-rpath,{libdir}"], check=True)
    gold = os.path.join(root, "tests", "golden")
    out = subprocess.run([str(exe), os.path.join(gold, "manifest_fresh.json"),
                          os.path.join(gold, "manifest_pinned.json")], check=True,
                         capture_output=True, text=True).stdout.splitlines()
    assert out[0] == "REF 1 -" and out[1] == "REF 1 -", out
    assert out[2] == "OWN 1", out
    assert out[3].startswith("BAD 0 trial 3 of record 0"), out


def test_device_quantizer_matches_host_quantizer():
    """ssqa_problem_create quantizes on the device: same scale, ranges, FP4
    decision and rejections as the host quantizer (ssqa_quantize_info)."""
    import ctypes as C
    L = _lib.lib()
    rng = np.random.default_rng(3)
    models = [sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0), sq.gi_ising(12, 0.5, 4, False, 0.75, 0.75),
              sq.dense_ising(300, 0, 1), sq.dense_ising(257, 1, 2)]
    h = rng.integers(-8, 9, 130) / 8.0
    J = np.triu(rng.integers(-6, 7, (130, 130)) / 4.0, 1)
    models.append(sq.IsingModel.from_arrays(h, J + J.T, 0.5))
    for m in models:
        prob = sq.Problem(m)
        dev = prob.info()
        v = [C.c_int() for _ in range(4)]
        dp = lambda a: np.ascontiguousarray(a).ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        assert L.ssqa_quantize_info(m.n, dp(m.h), dp(m.J), *[C.byref(x) for x in v]) == 0
        assert (dev["n_pad"], dev["shift_p"], dev["max_abs_j"], dev["max_abs_h"]) == \
            tuple(x.value for x in v), m.n
        Jq = np.abs(m.J * 2.0 ** dev["shift_p"])
        single = bool(np.isin(Jq, [0, 1, 2, 3, 4, 6]).all())
        pair = bool(np.isin(Jq, [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12]).all())
        assert dev["fp4"] == (1 if single else 2 if pair else 0)
    bad = sq.IsingModel(4)
    bad.set_coupling(0, 1, float("inf"))  # (0.1 is dyadic as a double: 2^-55 * integer)
    with pytest.raises(ValueError, match="not a dyadic"):
        sq.Problem(bad)
    tiny = sq.IsingModel(4)
    tiny.set_coupling(0, 1, 0.1)  # needs p = 55: far beyond int16
    with pytest.raises(ValueError, match="exceeds int16"):
        sq.Problem(tiny)
    big = sq.IsingModel(4)
    big.set_coupling(1, 2, 200.0)  # int16 planes (test_int16_*); refused when they are off
    assert sq.Problem(big).info()["int16"] == 1
    sq.tune(i16=0)
    with pytest.raises(ValueError, match="exceeds int8"):
        sq.Problem(big)


# ---- shape edge cases (each against the oracle, bitwise) ----

@pytest.mark.parametrize("shape", [
    dict(n=1, R=3, d=1, T=2, sc=20, bidir=False),        # a single spin
    dict(n=130, R=256, d=1, T=2, sc=12, bidir=False),    # a full 256-column tile per trial
    dict(n=129, R=17, d=30, T=3, sc=40, bidir=True),     # deepest delay ring, odd R
    dict(n=100, R=4, d=0, T=149, sc=15, bidir=False),    # more column tiles than SMs
    dict(n=200, R=300, d=1, T=2, sc=8, bidir=False),     # R > 256: the SIMT engine
], ids=["n1", "R256", "delay30", "T149", "R300-simt"])
def test_shape_edges_match_oracle(orc, shape):
    n, R = shape["n"], shape["R"]
    rng = np.random.default_rng(n + R)
    h = rng.integers(-4, 5, n) / 2.0
    J = np.triu(rng.integers(-2, 3, (n, n)) / 2.0, 1)
    m = sq.IsingModel.from_arrays(h, J + J.T, 0.25)
    p = params(R, shape["sc"], tau=3, delay=shape["d"], bidirectional=shape["bidir"])
    seeds = [int(s) for s in rng.integers(0, 2 ** 62, shape["T"])]
    res = sq.ssqa_run_batch(m, to_sq(p), seeds, None, sq.RunOptions(True, False))
    for t in sorted({0, shape["T"] - 1}):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[t], None, True, False)
        assert (res[t].best_energy, res[t].best_replica) == (o.best_energy, o.best_replica)
        assert np.array_equal(res[t].best_state, o.best_state)
        assert np.array_equal(bits(res[t].trace_energy), bits(o.trace))


def test_fp4_bidirectional_matches_oracle(orc):
    """FP4 operands (couplings in {0, +-1, +-2}) with the bidirectional coupling."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    m = sq.gi_ising(16, 0.5, 3, True, 1.0, 1.0)
    assert sq.Problem(m).info()["fp4"] == 1
    p = params(12, 50, tau=4, delay=2, bidirectional=True)
    seeds = [71, 72, 73]
    res = sq.ssqa_run_batch(m, to_sq(p), seeds, 0.0, sq.RunOptions(True, False),
                            engine=_lib.ENGINE_TCGEN05)
    for t, s in enumerate(seeds):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, s, 0.0, True, False)
        assert res[t].best_energy == o.best_energy
        assert np.array_equal(bits(res[t].trace_energy), bits(o.trace))


@pytest.mark.parametrize("n,R,T,rs", [(300, 8, 5, 1), (640, 12, 24, 4)], ids=["tile", "split"])
def test_fp4_pair_operands_match_oracle(orc, row_split, n, R, T, rs):
    """Couplings |J'| <= 12 (not 11) run as FP4 pairs J' = A1 + A2 (two
    kind::mxf4 MMAs per spin sub-block); |J'| = 11 falls back to int8."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    if rs > 1:
        row_split(rs)
    rng = np.random.default_rng(n)
    vals = np.array([-12, -10, -9, -8, -7, -5, -3, -1, 0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 12])
    J = np.triu(rng.choice(vals, (n, n)) / 4.0, 1)
    h = rng.integers(-40, 41, n) / 4.0
    m = sq.IsingModel.from_arrays(h, J + J.T, 1.5)
    assert sq.Problem(m).info()["fp4"] == 2
    p = params(R, 30, tau=4, bidirectional=(rs == 1))
    seeds = [int(s) for s in rng.integers(0, 2 ** 40, T)]
    res = sq.ssqa_run_batch(m, to_sq(p), seeds, None, sq.RunOptions(True, False),
                            engine=_lib.ENGINE_TCGEN05)
    for t in sorted({0, T // 2, T - 1}):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[t], None, True, False)
        assert (res[t].best_energy, res[t].best_replica) == (o.best_energy, o.best_replica), t
        assert np.array_equal(res[t].best_state, o.best_state), t
        assert np.array_equal(bits(res[t].trace_energy), bits(o.trace)), t
    J11 = J.copy()
    J11[0, 1] = 11 / 4.0
    assert sq.Problem(sq.IsingModel.from_arrays(h, J11 + J11.T, 1.5)).info()["fp4"] == 0


@pytest.mark.gpu
def test_pool_reuse_keeps_results_identical(orc):
    """Repeated public calls reuse the pool's blocks (csrc/devpool.h): a second
    batch of the same shape allocates nothing new, starts from recycled
    (dirty) memory and still equals the oracle bit for bit."""
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    p = params(20, 120)
    seeds = list(range(40, 52))
    first = sq.ssqa_run_batch(m, to_sq(p), seeds, 0.0, sq.RunOptions(True, False))
    st1 = sq.pool_stats(0)
    assert st1["cached"] > 0
    second = sq.ssqa_run_batch(m, to_sq(p), seeds, 0.0, sq.RunOptions(True, False))
    st2 = sq.pool_stats(0)
    assert st2 == st1  # every block came from, and went back to, the cache
    for t in (0, 5, 11):
        o = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[t], 0.0, True, False)
        for r in (first[t], second[t]):
            assert (r.best_energy, r.best_replica, r.first_hit_cycle) == \
                (o.best_energy, o.best_replica, o.first_hit_cycle)
            assert np.array_equal(bits(r.trace_energy), bits(o.trace))
    assert sq.pool_trim(0) == st2["cached"]
    assert sq.pool_stats(0)["cached"] == 0


@pytest.mark.gpu
def test_fused_run_leaves_exact_lattice(orc, monkeypatch):
    """The fused run (one launch, all sweeps): the lattice it leaves behind --
    spins, history and every accumulator bit -- equals the oracle's after sc
    sweeps (int8 operands keep the lattice; FP4 runs mark it stale)."""
    if not engine_ok(_lib.ENGINE_TCGEN05):
        pytest.skip("tcgen05 engine unavailable")
    sq.tune(fp4=0)
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    for p in (params(20, 130), params(6, 90, delay=2, bidirectional=True)):
        T = 5
        seeds = [77 + 3 * t for t in range(T)]
        b = sq.Batch(sq.Problem(m), to_sq(p), T, engine=_lib.ENGINE_TCGEN05)
        b.set_seeds(seeds)
        b.launch(None, False)
        for t in (0, 2, 4):
            s, a, h = orc.init_lattice(m.n, p.r, p.delay, seeds[t])
            for c in range(p.sc):
                orc.ssqa_sweep(m.h, m.J, m.offset, orc.jperp_schedule(c, p), p, seeds[t], c,
                               s, a, h, c)
            sg, ac, hi, cyc = b.read_lattice(t)
            assert cyc == p.sc
            assert np.array_equal(sg, s) and np.array_equal(bits(ac), bits(a)), (p.r, t)
            assert np.array_equal(hi, h)
        b.close()


# ---- int16 couplings (north star: "int16 where the coefficient range requires it")

def int16_model(n, jmax, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    J = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    J[iu] = rng.integers(-jmax, jmax + 1, len(iu[0])) * scale
    J = J + J.T
    h = rng.integers(-3 * jmax, 3 * jmax + 1, n) * scale
    return sq.IsingModel.from_arrays(h, J, 0.25)


@pytest.mark.parametrize("rs", [1, 2], ids=["whole", "rowsplit"])
def test_int16_couplings_match_oracle(orc, rs):
    """|J'| up to 2^14 (and the plane limit 32639): two int8 planes J' = 256 Ahi +
    Alo, one kind::i8 MMA per plane into its own TMEM accumulator, S = D_lo +
    256 D_hi in the epilogue.  Full runs with traces against the C oracle,
    whole tiles and a row split (table epilogue, CTA cooperation)."""
    if rs > 1:
        sq.tune(rs=rs)
    for n, jmax, scale, bidir in [(300, 1 << 14, 1.0, False), (200, 32639, 1.0, True),
                                  (260, 3000, 0.25, False)]:
        m = int16_model(n, jmax, n + jmax, scale)
        if jmax == 32639:
            m.J[0, 1] = m.J[1, 0] = 32639.0  # the largest magnitude the planes hold
        prob = sq.Problem(m)
        assert prob.info()["int16"] == 1 and prob.info()["max_abs_j"] == jmax
        p = params(6, 40, tau=5, bidirectional=bidir)
        seeds = [5 + 3 * t for t in range(5)]
        res = sq.ssqa_run_batch(m, to_sq(p), seeds, None, sq.RunOptions(True, False),
                                _lib.ENGINE_TCGEN05, problem=prob)
        for t in (0, 4):
            o = orc.ssqa_run(m.h, m.J, m.offset, p, seeds[t], None, True, False)
            assert np.array_equal(bits(res[t].trace_energy), bits(o.trace)), (n, t)
            assert np.array_equal(res[t].best_state, o.best_state), (n, t)
            assert res[t].best_energy == o.best_energy
        prob.close()


def test_int16_per_step_api_matches_oracle(orc):
    """The per-step sweeps (ssqa_sweep, annealer.cpp:449-463) on int16 couplings:
    spins, history and every accumulator bit after each sweep."""
    m = int16_model(150, 9000, 3)
    p = params(4, 30, tau=3)
    seeds = [21, 22]
    b = sq.Batch(sq.Problem(m), to_sq(p), len(seeds), engine=_lib.ENGINE_TCGEN05)
    b.set_seeds(seeds)
    b.init()
    states = [orc.init_lattice(m.n, p.r, p.delay, sd) for sd in seeds]
    for c in range(8):
        b.sweep(1)
        for t, (s, a, h) in enumerate(states):
            orc.ssqa_sweep(m.h, m.J, m.offset, orc.jperp_schedule(c, p), p, seeds[t], c, s, a, h, c)
            sg, ac, hi, cyc = b.read_lattice(t)
            assert cyc == c + 1
            assert np.array_equal(sg, s) and np.array_equal(bits(ac), bits(a)), (c, t)
            assert np.array_equal(hi, h)
    b.close()


def test_int16_limits():
    m = int16_model(64, 100, 1)
    m.J[2, 3] = m.J[3, 2] = 32640.0  # one beyond the planes
    with pytest.raises(sq.SsqaInvalidArgument):
        sq.Problem(m)
    m.J[2, 3] = m.J[3, 2] = 32639.0
    prob = sq.Problem(m)
    with pytest.raises(sq.SsqaInvalidArgument):  # SIMT engine: int8 only
        sq.Batch(prob, sq.SsqaParams(r=4, sc=5), 2, engine=_lib.ENGINE_SIMT)
    sq.tune(i16=0)
    with pytest.raises(sq.SsqaInvalidArgument):
        sq.Problem(m)
