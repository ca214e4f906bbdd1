#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the reference itself (oracle/_ref).

TEST INFRASTRUCTURE.  Runs only in the build container, where /root/reference
exists and `make -C oracle` has compiled the unmodified reference sources into
oracle/_ref/.  The fixtures it writes are small and committed; the GPU box
never needs the reference.

    python scripts/make_golden.py
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle_py import Oracle, params, ssa_params  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fnv1a(data: bytes) -> int:
    h = 0xcbf29ce484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def random_model(rng, n, kind):
    """kind 'real': uniform doubles (reference test_annealer.cpp:17-25 style);
    'quarter': multiples of 1/4; 'few': the 7-value set of test_annealer.cpp:368."""
    if kind == "real":
        draw = lambda size: rng.uniform(-2.0, 2.0, size)  # noqa: E731
    elif kind == "quarter":
        draw = lambda size: rng.integers(-8, 9, size) / 4.0  # noqa: E731
    else:
        vals = np.array([-1.0, -0.5, -0.25, 0.25, 0.5, 0.75, 1.0])
        draw = lambda size: vals[rng.integers(0, 7, size)]  # noqa: E731
    h = draw(n)
    J = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    v = draw(len(iu[0]))
    if kind == "few":
        v[rng.integers(0, 4, len(v)) == 0] = 0.0
    J[iu] = v
    J = J + J.T
    off = float(draw(1)[0])
    return h, J, off


def lattice_trajectories(ref: Oracle):
    """Per-step sigma/acc of ssqa_sweep (annealer.cpp:449-463) for a spread of
    shapes: the per-step bit-exactness pins."""
    rng = np.random.default_rng(20240601)
    cases = [
        # n, r, delay, bidir, alpha, kind, cycles
        (1, 1, 0, False, 1.0, "quarter", 12),
        (2, 2, 1, False, 1.0, "quarter", 20),
        (5, 3, 2, False, 0.5, "quarter", 20),
        (6, 4, 1, True, 1.0, "quarter", 20),
        (9, 6, 1, True, 1.0, "few", 12),
        (40, 4, 2, False, 1.0, "few", 12),
        (70, 5, 1, False, 1.0, "few", 12),
        (70, 1, 0, False, 1.0, "few", 12),
        (130, 20, 1, False, 1.0, "quarter", 16),
        (6, 4, 1, True, 1.0, "real", 20),
        (5, 3, 2, False, 0.5, "real", 20),
    ]
    out = {}
    for ci, (n, r, d, bidir, alpha, kind, cycles) in enumerate(cases):
        h, J, off = random_model(rng, n, kind)
        seed = int(rng.integers(0, 2**63))
        p = params(r, 1, delay=d, alpha=alpha, bidirectional=bidir)
        sigma, acc, hist = ref.init_lattice(n, r, d, seed)
        sig_t, acc_t, jp_t, i0_t, en_t = [sigma.copy()], [acc.copy()], [], [], []
        lat_cycle = 0
        for c in range(cycles):
            jperp = 0.1 * (c % 6)
            i0 = 2.0 if c % 2 else 4.0
            p.i0 = i0
            lat_cycle = ref.ssqa_sweep(h, J, off, jperp, p, seed, c, sigma, acc, hist, lat_cycle)
            sig_t.append(sigma.copy())
            acc_t.append(acc.copy())
            jp_t.append(jperp)
            i0_t.append(i0)
            en_t.append(ref.replica_energies(h, J, off, r, sigma))
        out[f"traj{ci}"] = dict(
            n=n, r=r, delay=d, bidir=int(bidir), alpha=alpha, kind=kind, seed=np.uint64(seed),
            h=h, J=J, offset=off, jperp=np.array(jp_t), i0=np.array(i0_t),
            sigma=np.array(sig_t), acc=np.array(acc_t), energy=np.array(en_t),
            hist_final=hist.copy())
    return out


def gi_instances(ref: Oracle):
    out = {}
    for n_nodes, seed, permute, c in [(1, 3, True, 1.0), (3, 11, True, 1.0), (4, 5, False, 0.75),
                                      (10, 7, True, 1.0), (20, 7, True, 1.0), (10, 7, True, 0.75),
                                      (50, 7, True, 1.0)]:
        h, J, off = ref.gi_ising(n_nodes, 0.5, seed, permute, c, c)
        rec = dict(n_nodes=n_nodes, seed=seed, permute=int(permute), c=c, offset=off,
                   h=h, J_sha=sha(J), J_nnz=int(np.count_nonzero(J)))
        if n_nodes <= 10:
            rec["J"] = J
        out[f"gi_{n_nodes}_{seed}_{int(permute)}_{c}"] = rec
    return out


def runs(ref: Oracle):
    """ssqa_run KATs plus small random runs."""
    out = {}
    cases = [
        ("gi10", (10, 7, 1.0), dict(r=20, sc=1000), 123, 0.0, True, False),
        ("gi20", (20, 7, 1.0), dict(r=20, sc=2000), 123, 0.0, True, False),
        ("gi10_stop", (10, 7, 1.0), dict(r=20, sc=1000), 5, 0.0, True, True),
        ("gi10_bidir_d2", (10, 7, 1.0), dict(r=7, sc=700, delay=2, bidirectional=True), 9, 0.0,
         True, False),
        ("gi10_c075", (10, 7, 0.75), dict(r=16, sc=600), 77, 0.0, True, False),
        ("gi10_r1", (10, 7, 1.0), dict(r=1, sc=500, delay=0), 3, 0.0, True, False),
    ]
    for name, (nn, gseed, c), pk, seed, target, trace, stop in cases:
        h, J, off = ref.gi_ising(nn, 0.5, gseed, True, c, c)
        p = params(**pk)
        res = ref.ssqa_run(h, J, off, p, seed, target, trace, stop)
        out[name] = dict(n_nodes=nn, gi_seed=gseed, c=c, seed=np.uint64(seed), target=target,
                         stop=int(stop), **{f"p_{k}": v for k, v in pk.items()},
                         best_energy=res.best_energy, best_replica=res.best_replica,
                         reached=int(res.reached_target), first_hit=res.first_hit_cycle,
                         cycles_used=res.cycles_used, best_state=res.best_state,
                         trace=res.trace,
                         trace_fnv=np.uint64(fnv1a(res.trace.tobytes())),
                         best_state_fnv=np.uint64(fnv1a(res.best_state.tobytes())))
    # small random quarter-integer models with targets from the run itself
    rng = np.random.default_rng(7)
    for ci in range(4):
        n = int(rng.integers(3, 12))
        h, J, off = random_model(rng, n, "quarter")
        p = params(int(rng.integers(1, 6)), 80, tau=int(rng.integers(3, 20)))
        seed = int(rng.integers(0, 2**63))
        res = ref.ssqa_run(h, J, off, p, seed, None, True, False)
        out[f"rand{ci}"] = dict(h=h, J=J, offset=off, seed=np.uint64(seed), p_r=p.r, p_sc=p.sc,
                                p_tau=p.tau, best_energy=res.best_energy,
                                best_replica=res.best_replica, best_state=res.best_state,
                                trace=res.trace, cycles_used=res.cycles_used)
    return out


def ssa_runs(ref: Oracle):
    """ssa_run (annealer.cpp:489-501) on GI instances and random models, plus
    i0_schedule values (annealer.cpp:382-408)."""
    out = {}
    cases = [
        ("gi10", (10, 7, 1.0), dict(sc=2000), 1, True, False),
        ("gi10_tau25", (10, 7, 1.0), dict(sc=3000, tau=25), 1, True, False),
        ("gi10_stop", (10, 7, 1.0), dict(sc=3000, tau=25), 1, True, True),
        ("gi10_flat", (10, 7, 1.0), dict(sc=500, i0_min=2.0, i0_max=2.0), 2, True, False),
        ("gi10_coarse", (10, 7, 0.75), dict(sc=800, beta=0.3, i0_max=12.0, tau=7, n_rnd=2.0),
         4, True, False),
        ("gi20", (20, 7, 1.0), dict(sc=2000, tau=25), 5, True, False),
    ]
    for name, (nn, gseed, c), pk, seed, trace, stop in cases:
        h, J, off = ref.gi_ising(nn, 0.5, gseed, True, c, c)
        p = ssa_params(**pk)
        res = ref.ssa_run(h, J, off, p, seed, 0.0, trace, stop)
        out[name] = dict(n_nodes=nn, gi_seed=gseed, c=c, seed=np.uint64(seed), target=0.0,
                         stop=int(stop), **{f"p_{k}": v for k, v in pk.items()},
                         best_energy=res.best_energy, reached=int(res.reached_target),
                         first_hit=res.first_hit_cycle, cycles_used=res.cycles_used,
                         best_state=res.best_state, trace=res.trace)
    rng = np.random.default_rng(11)
    for ci in range(3):
        n = int(rng.integers(3, 12))
        h, J, off = random_model(rng, n, "quarter")
        p = ssa_params(120, tau=int(rng.integers(2, 9)))
        seed = int(rng.integers(0, 2**63))
        res = ref.ssa_run(h, J, off, p, seed, None, True, False)
        out[f"rand{ci}"] = dict(h=h, J=J, offset=off, seed=np.uint64(seed), p_sc=p.sc,
                                p_tau=p.tau, best_energy=res.best_energy,
                                best_state=res.best_state, trace=res.trace,
                                cycles_used=res.cycles_used)
    sched = [dict(), dict(i0_max=10.0), dict(i0_min=0.5, i0_max=8.0), dict(beta=0.3),
             dict(tau=3, beta=0.7, i0_max=40.0)]
    for si, pk in enumerate(sched):
        p = ssa_params(1, **pk)
        cyc = np.arange(0, 400, dtype=np.int64)
        out[f"sched{si}"] = dict(**{f"p_{k}": v for k, v in pk.items()}, cycles=cyc,
                                 i0=np.array([ref.i0_schedule(int(c), p) for c in cyc]))
    return out


def trials(ref: Oracle):
    """run_trials KAT (bench.cpp:359-432)."""
    outs, ps, tm, tts = ref.run_trials(params(20, 1), n_nodes=10, trials=100, ec=20000,
                                       base_seed=1000, workers=8, gi_seed=7)
    buf = b"".join(np.array([o["seed"]], np.uint64).tobytes() + bytes([o["reached_target"]]) +
                   np.array([o["first_hit_cycle"]], np.int64).tobytes() +
                   np.array([o["best_energy"]], np.float64).tobytes() for o in outs)
    return {"trials_gi10": dict(
        seed=np.array([o["seed"] for o in outs], np.uint64),
        reached=np.array([o["reached_target"] for o in outs], np.int8),
        first_hit=np.array([o["first_hit_cycle"] for o in outs], np.int64),
        best_energy=np.array([o["best_energy"] for o in outs]), p_s=ps,
        outcomes_fnv=np.uint64(fnv1a(buf)))}


def trials_fresh(ref: Oracle):
    """run_trials with a fresh GI instance per trial (the reference default,
    bench.hpp:28; instance seeds CounterRng(base_seed, 7).raw(t), bench.cpp:389)."""
    out = {}
    cases = [("fresh_gi10", dict(n_nodes=10, trials=64, ec=20000, base_seed=1000, permute=False,
                                 c1=0.75, c2=0.75), 20),
             ("fresh_gi20", dict(n_nodes=20, trials=24, ec=10000, base_seed=77, permute=True,
                                 c1=1.0, c2=1.0), 20)]
    for name, kw, r in cases:
        outs, ps, tm, tts = ref.run_trials(params(r, 1), workers=8, fresh_instance=True, **kw)
        out[name] = dict(**{f"k_{k}": v for k, v in kw.items()}, r=r,
                         seed=np.array([o["seed"] for o in outs], np.uint64),
                         reached=np.array([o["reached_target"] for o in outs], np.int8),
                         first_hit=np.array([o["first_hit_cycle"] for o in outs], np.int64),
                         best_energy=np.array([o["best_energy"] for o in outs]), p_s=ps)
    return out


def trials_large(ref: Oracle):
    """run_trials at BASELINE configs 2 and 3 at their own shapes (bench.cpp:359-432):
    C2 = GI n=20 (N=400), M=20, the full 1024-trial battery at sc=2000; C3 = GI n=50
    (N=2500), M=20, seeds 1000..1047 at the full sc=5000.  Fixed instance (gi_seed 7,
    permuted, c1=c2=1) as in BASELINE.json.  The device batch must match trial for trial."""
    out = {}
    cases = [("c2_gi20", dict(n_nodes=20, trials=1024, ec=40000, base_seed=1000)),
             ("c3_gi50", dict(n_nodes=50, trials=48, ec=100000, base_seed=1000)),
             # fresh instance per trial at the C3 size (bench.hpp:28, the reference
             # default), permuted, c1 = c2 = 1: the device-built battery's pin
             ("c3_fresh_gi50", dict(n_nodes=50, trials=16, ec=100000, base_seed=1000,
                                    fresh_instance=True))]
    only = [c for c in cases if os.environ.get("SSQA_GOLDEN_CASE", c[0]) == c[0]]
    for name, kw in only:
        outs, ps, tm, tts = ref.run_trials(params(20, 1), workers=os.cpu_count(), gi_seed=7,
                                           **kw)
        out[name] = dict(**{f"k_{k}": v for k, v in kw.items()}, r=20,
                         seed=np.array([o["seed"] for o in outs], np.uint64),
                         reached=np.array([o["reached_target"] for o in outs], np.int8),
                         first_hit=np.array([o["first_hit_cycle"] for o in outs], np.int64),
                         best_energy=np.array([o["best_energy"] for o in outs]), p_s=ps,
                         wall=np.array([o["wall_seconds"] for o in outs]))
        print(name, "p_s", ps, flush=True)
    # keep the cases already in the committed file that were not regenerated
    path = os.path.join(OUT, "trials_large.npz")
    if os.path.exists(path):
        z = np.load(path)
        for key in z.files:
            case, field = key.split("/", 1)
            if case not in out:
                out.setdefault(case + "#keep", {})[field] = z[key]
        out = {k.replace("#keep", ""): v for k, v in out.items()}
    return out


def manifests(ref: Oracle):
    """Manifests written by the reference (make_manifest, bench.cpp:519-531),
    replayed bitwise by the facade's replay_manifest in the GPU tests."""
    for name, kw in [("manifest_fresh", dict(n_nodes=10, trials=12, ec=20000, base_seed=500)),
                     ("manifest_pinned", dict(n_nodes=10, trials=20, ec=20000, base_seed=1000,
                                              permute=True, c1=1.0, c2=1.0,
                                              fresh_instance=False, gi_seed=7))]:
        js = ref.bench_manifest(params(20, 1), workers=8, **kw)
        path = os.path.join(OUT, name + ".json")
        with open(path, "w") as f:
            f.write(js)
        print(f"wrote {path}: {len(js)} bytes")
    return {}


def main():
    ref = Oracle("ref")
    os.makedirs(OUT, exist_ok=True)
    jobs = [("lattice_traj", lattice_trajectories), ("gi_instances", gi_instances),
            ("runs", runs), ("trials", trials), ("ssa_runs", ssa_runs),
            ("trials_fresh", trials_fresh), ("trials_large", trials_large)]
    only = set(sys.argv[1:])
    for fname, fn in jobs + [("manifests", manifests)]:
        if (only and fname not in only) or (not only and fname == "trials_large"):
            continue
        data = fn(ref)
        if not data:
            continue
        flat = {}
        for case, rec in data.items():
            for k, v in rec.items():
                flat[f"{case}/{k}"] = np.asarray(v)
        path = os.path.join(OUT, fname + ".npz")
        np.savez_compressed(path, **flat)
        print(f"wrote {path}: {len(data)} cases, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
