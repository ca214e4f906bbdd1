"""CPU-side checks of the product library (no GPU needed).

* libssqa_b200.so loads and exports every symbol the include/*.h headers
  declare (the drop-in boundary);
* the host problem builders reproduce the reference's instances bit for bit
  (tests/golden/gi_instances.npz, made from oracle/_ref);
* the quantizer dry run, parameter validation and schedule follow the
  reference (annealer.cpp:365-380).
"""
import ctypes
import glob
import hashlib
import os
import re

import numpy as np
import pytest

import paper_2302_12454_b200 as sq
from paper_2302_12454_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_c_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(ssqa_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_c_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the ctypes signature table covers them all
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) <= bound, set(names) - bound


def test_library_exports_cpp_facade():
    out = os.popen(f"nm -DC --defined-only {_lib.LIB_PATH}").read()
    for sym in ("ssqa::ssqa_run(", "ssqa::ssqa_run_batch(", "ssqa::init_lattice(",
                "ssqa::ssqa_sweep(", "ssqa::replica_energies(", "ssqa::run_trials(",
                "ssqa::jperp_schedule(", "ssqa::qubo_to_ising(", "ssqa::generate_gi(",
                "ssqa::build_gi_qubo(", "ssqa::compute_tts(", "ssqa::ssa_run(",
                "ssqa::ssa_run_batch(", "ssqa::i0_schedule(", "ssqa::SsaParams::i0_levels("):
        assert sym in out, sym


def test_gi_builder_matches_reference(golden):
    for name, c in golden("gi_instances").items():
        m = sq.gi_ising(int(c["n_nodes"]), 0.5, int(c["seed"]), bool(c["permute"]),
                        float(c["c"]), float(c["c"]))
        assert np.array_equal(m.h.view(np.uint64), c["h"].view(np.uint64)), name
        assert m.offset == float(c["offset"]), name
        assert hashlib.sha256(m.J.tobytes()).hexdigest() == str(c["J_sha"]), name


def test_gi_builder_matches_live_reference_non_dyadic(ref):
    """Penalties that are not dyadic (c1 = 0.7, c2 = 0.3): every sum rounds, so
    only the reference's exact accumulation order reproduces h and offset
    (host/inputs.cpp restates it in closed form, without the QUBO)."""
    for nn, seed, perm, c1, c2 in [(6, 3, True, 0.7, 0.3), (9, 12, False, 0.7, 1.1),
                                   (12, 5, True, 0.35, 0.9)]:
        m = sq.gi_ising(nn, 0.45, seed, perm, c1, c2)
        h, J, off = ref.gi_ising(nn, 0.45, seed, perm, c1, c2)
        assert np.array_equal(m.h.view(np.uint64), h.view(np.uint64))
        assert np.array_equal(m.J.view(np.uint64), J.view(np.uint64))
        assert np.float64(m.offset).view(np.uint64) == np.float64(off).view(np.uint64)


def test_gi_compact_closed_form_matches_builder():
    """The host half of the device GI generator: biases and offset in closed
    form (host/inputs.cpp gi_compact) equal the builder's bit for bit for
    dyadic penalties, and the adjacency matrices reproduce every coupling."""
    for nn, seed, perm, c1, c2 in [(1, 3, True, 1.0, 1.0), (2, 5, True, 1.0, 1.0),
                                   (5, 9, False, 0.75, 0.75), (10, 7, True, 1.0, 1.0),
                                   (8, 4, True, 0.5, 2.0), (12, 99, False, 1.25, 0.375)]:
        adj, h, off = sq.gi_compact(nn, 0.5, seed, perm, c1, c2)
        m = sq.gi_ising(nn, 0.5, seed, perm, c1, c2)
        assert np.array_equal(h.view(np.uint64), m.h.view(np.uint64))
        assert np.float64(off).view(np.uint64) == np.float64(m.offset).view(np.uint64)
        a1, a2 = adj[0].astype(bool), adj[1].astype(bool)
        u, i = np.divmod(np.arange(nn * nn), nn)
        one_hot = (u[:, None] == u[None, :]) != (i[:, None] == i[None, :])
        mis = (u[:, None] != u[None, :]) & (i[:, None] != i[None, :]) & \
            (a1[i[:, None], i[None, :]] != a2[u[:, None], u[None, :]])
        J = np.where(one_hot, -0.25 * 2 * c1, np.where(mis, -0.25 * c2, 0.0))
        assert np.array_equal(J.view(np.uint64), m.J.view(np.uint64))


def test_gi_builder_rejects_bad_arguments():
    with pytest.raises(ValueError):
        sq.gi_ising(0)
    with pytest.raises(ValueError):
        sq.gi_ising(3, edge_prob=1.5)
    with pytest.raises(ValueError):
        sq.gi_ising(3, c1=0.0)


def test_dense_builders():
    m = sq.dense_ising(64, 0, 11)
    assert np.array_equal(m.J, m.J.T) and (np.diag(m.J) == 0).all()
    assert m.J.min() >= -8 and m.J.max() <= 7 and m.h.min() >= -8 and m.h.max() <= 7
    assert len(np.unique(m.J[np.triu_indices(64, 1)])) == 16
    s = sq.dense_ising(64, 1, 11)
    assert set(np.unique(s.J[np.triu_indices(64, 1)])) == {-1.0, 1.0} and (s.h == 0).all()
    assert np.array_equal(sq.dense_ising(64, 0, 11).J, m.J)


def _qinfo(h, J):
    L = _lib.lib()
    v = [ctypes.c_int() for _ in range(4)]
    rc = L.ssqa_quantize_info(len(h), h.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                              J.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                              *[ctypes.byref(x) for x in v])
    return rc, [x.value for x in v]


def test_quantizer_scales():
    m = sq.gi_ising(10, 0.5, 7, True, 1.0, 1.0)
    rc, (npad, p, mj, mh) = _qinfo(m.h, m.J)
    assert rc == 0 and (npad, p, mj) == (128, 2, 2)
    m = sq.gi_ising(10, 0.5, 7, True, 0.75, 0.75)
    rc, (npad, p, mj, mh) = _qinfo(m.h, m.J)
    assert rc == 0 and p == 4 and mj == 6
    m = sq.dense_ising(300, 0, 1)
    rc, (npad, p, mj, mh) = _qinfo(m.h, m.J)
    assert rc == 0 and (npad, p, mj) == (384, 0, 8)
    # non-dyadic and out-of-range models are rejected (no CPU fallback)
    h = np.zeros(3)
    J = np.zeros((3, 3))
    J[0, 1] = J[1, 0] = 0.1
    assert _qinfo(h, J)[0] == _lib.SSQA_EUNSUP
    J[0, 1] = J[1, 0] = 200.0
    assert _qinfo(h, J)[0] == _lib.SSQA_EUNSUP
    J[0, 1] = J[1, 0] = 1.0
    J[0, 2] = J[2, 0] = 2.0 ** -7  # needs p = 7 -> J' = 128 > 127
    assert _qinfo(h, J)[0] == _lib.SSQA_EUNSUP


def test_params_validation_matches_reference():
    # annealer.cpp:365-373 / test_annealer.cpp:142-164
    ok = sq.SsqaParams(r=2, sc=10)
    ok.validate(3)
    for bad in (dict(r=0), dict(r=1 << 12), dict(sc=0), dict(sc=1 << 31), dict(jperp_max=-0.1),
                dict(beta=0), dict(tau=0), dict(delay=-1), dict(i0=0.0), dict(alpha=0.0),
                dict(n_rnd=-1.0)):
        p = sq.SsqaParams(**{**ok.__dict__, **bad})
        with pytest.raises(ValueError):
            p.validate(3)
    with pytest.raises(ValueError):
        ok.validate(0)
    with pytest.raises(ValueError):
        ok.validate(1 << 20)


def test_jperp_schedule_matches_oracle(orc):
    from oracle_py import params
    for kw in (dict(), dict(jperp_min=0.25, jperp_max=0.75, beta=1, tau=1),
               dict(jperp_min=0.1, jperp_max=0.9, beta=7, tau=13)):
        p = sq.SsqaParams(r=1, sc=1, **kw)
        q = params(1, 1, **kw)
        for c in list(range(0, 1200, 7)) + [399, 400, 401]:
            assert sq.jperp_schedule(c, p) == orc.jperp_schedule(c, q)
    with pytest.raises(ValueError):
        sq.jperp_schedule(-1, sq.SsqaParams(r=1, sc=1))


def test_ssa_params_match_reference(orc):
    # annealer.cpp:382-408 / test_annealer.cpp:101-126, 166-185
    from oracle_py import ssa_params
    p = sq.SsaParams(sc=1)
    assert p.i0_levels() == [1, 2, 4, 8, 16] and p.cycles_per_iteration() == 50
    assert [sq.i0_schedule(c, p) for c in (0, 9, 10, 49, 50)] == [1.0, 1.0, 2.0, 16.0, 1.0]
    assert sq.SsaParams(sc=1, i0_max=10.0).i0_levels() == [1, 2, 4, 8]
    assert sq.SsaParams(sc=1, i0_min=0.5, i0_max=8.0).i0_levels() == [0.5, 1, 2, 4, 8]
    assert len(sq.SsaParams(sc=1, beta=0.3).i0_levels()) == 3
    with pytest.raises(ValueError):
        sq.i0_schedule(-1, p)
    for kw in (dict(), dict(tau=3, beta=0.7, i0_max=40.0), dict(i0_min=0.3, i0_max=0.3)):
        q = sq.SsaParams(sc=1, **kw)
        o = ssa_params(1, **kw)
        for c in range(0, 500, 3):
            assert sq.i0_schedule(c, q) == orc.i0_schedule(c, o)
    ok = sq.SsaParams(sc=10)
    ok.validate(3)
    for bad in (dict(i0_min=0.0), dict(i0_min=32.0), dict(beta=1.0), dict(beta=0.0),
                dict(tau=0), dict(sc=0), dict(alpha=0.0), dict(n_rnd=-1.0),
                dict(i0_min=1e-30, i0_max=1e30), dict(i0_min=float("nan"))):
        with pytest.raises(ValueError):
            sq.SsaParams(**{**ok.__dict__, **bad}).validate(3)


def test_compute_tts():
    # bench.cpp:144-160
    assert sq.compute_tts(1.0, 2.0).kind == "saturated"
    assert sq.compute_tts(0.0, 2.0).kind == "undefined"
    v = sq.compute_tts(0.5, 2.0)
    assert v.kind == "finite" and v.seconds == pytest.approx(2.0 * np.log(0.01) / np.log(0.5))
    with pytest.raises(ValueError):
        sq.compute_tts(0.5, 0.0)


def test_anneal_result_trace_points():
    """AnnealResult.trace: TracePoint{cycle, replica, energy, jperp} per replica
    and scanned cycle in the reference's order (annealer.cpp:343), built from the
    bulk energy trace and the jperp staircase (annealer.cpp:375-380)."""
    from paper_2302_12454_b200 import api
    p = sq.SsqaParams(r=3, sc=250)
    res = [type("R", (), dict(best_energy=1.0, best_replica=2, reached_target=0,
                              first_hit_cycle=-1, cycles_used=205, wall_seconds=0.0))()]
    tr = np.arange(1 * 251 * 3, dtype=np.float64).reshape(1, 251, 3)
    out = api._results(res, None, tr, 1, p)[0]
    tp = out.trace
    assert len(tp) == 206 * 3
    assert (tp[0].cycle, tp[0].replica, tp[0].energy, tp[0].jperp) == (0, 0, 0.0, 0.0)
    x = tp[205 * 3 + 2]
    assert (x.cycle, x.replica, x.energy) == (205, 2, float(205 * 3 + 2))
    assert x.jperp == sq.jperp_schedule(205, p) == 0.0 + 2 * (0.5 - 0.0) / 3
    assert tp[100 * 3].jperp == sq.jperp_schedule(100, p)
    # no trace recorded -> empty list; SSA traces carry jperp = 0
    assert api._results(res, None, None, 1, p)[0].trace == []
    s = api._results(res, None, tr[:, :, :1], 1, sq.SsaParams(sc=250))[0].trace
    assert len(s) == 206 and all(q.jperp == 0.0 and q.replica == 0 for q in s)


def test_column_tiling_plans():
    """make_geom through ssqa_plan_geometry (host only): the BASELINE configs'
    layouts on 148 SMs, and the searched layouts of the C3 rank blocks (512 /
    256 / 128 trials: whole tiles, then row splits that fill the SMs)."""
    import ctypes as C
    L = _lib.lib()

    def plan(n, r, t, bits, sms=148):
        o = [C.c_int() for _ in range(4)]
        _lib.check(L.ssqa_plan_geometry(n, r, t, sms, bits, *[C.byref(x) for x in o]), host=True)
        return tuple(x.value for x in o)  # tile_cols, tiles, trials per tile, row parts

    assert plan(100, 20, 100, 4) == (32, 100, 1, 1)          # C1
    assert plan(400, 20, 1024, 4) == (144, 147, 7, 1)        # C2
    assert plan(2500, 20, 1024, 4) == (144, 147, 7, 1)       # C3: whole tiles, 147 of 148 SMs
    assert plan(8192, 32, 256, 4) == (224, 37, 7, 4)         # C4: 37 x 4 = 148 CTAs (pairs)
    assert plan(32768, 16, 64, 4) == (208, 5, 13, 28)        # C5: 5 x 28 = 140 CTAs (pairs)
    cols, tiles, tpt, rs = plan(2500, 20, 512, 4)
    assert rs == 1 and tpt == 4 and tiles == 128
    for t in (256, 128, 64):
        cols, tiles, tpt, rs = plan(2500, 20, t, 4)
        assert rs > 1 and tiles * rs <= 148 and tiles * tpt >= t and cols <= 240
        assert tiles * rs >= 120                              # the split fills the SMs
    with pytest.raises(ValueError):
        plan(2500, 20, 128, 5)
