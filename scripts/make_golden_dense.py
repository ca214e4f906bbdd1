"""Full-budget golden outcomes for the dense BASELINE configs (C4, C5).

The reference's scalar ssqa_run needs hours per trial at these sizes, so the
fixture comes from oracle/lattice_np.py -- the vectorised restatement that
tests/test_oracle_golden.py pins to the C oracle and, through it, to the
reference's own fixtures.  For a few trials spread over each battery (C4:
trials 0, 100, 255; C5: 0, 63; seeds 1000 + t) it stores the outcome of the whole run
(sc = 2000 / 1000 sweeps): best energy, best replica, SHA-256 of the energy
trace [sc + 1][R] (float64 bytes) and of the best state (int8 bytes), plus
the energies of a few cycles in clear for debugging.

    python scripts/make_golden_dense.py [c4] [c5]   ->  tests/golden/dense_full.npz

C4 takes ~3 minutes on 8 cores, C5 ~20 (a 4.3 GB float32 coupling matrix).
tests/test_gpu_large.py::test_dense_full_budget_matches_golden compares the
device batch with it.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import lattice_np as lnp  # noqa: E402
import paper_2302_12454_b200 as sq  # noqa: E402
from oracle_py import params  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "dense_full.npz")
CASES = {"c4": dict(n=8192, kind=0, R=32, T=256, sc=2000, check=[0, 100, 255]),
         "c5": dict(n=32768, kind=1, R=16, T=64, sc=1000, check=[0, 63])}
PEEK = [0, 1, 2, 10, 50, 100, 500, 999, 1000, 1999, 2000]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    want = [a for a in sys.argv[1:] if a in CASES] or list(CASES)
    old = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    for name in want:
        c = CASES[name]
        t0 = time.time()
        m = sq.dense_ising(c["n"], c["kind"], 7)
        p = params(c["R"], c["sc"])
        seeds = [1000 + t for t in c["check"]]
        Jq = np.asarray(m.J, dtype=np.float32)  # integral couplings: exact in float32 products
        res = lnp.run_lattice(np.asarray(m.h), None, m.offset, c["R"], p.delay, p.n_rnd, p.alpha,
                              False, c["sc"], lnp.jperp_schedule(p), lambda cyc: p.i0, seeds,
                              J_scaled=Jq)
        for key in [k for k in old if k.startswith(name + "/")]:
            del old[key]
        old[f"{name}/k"] = np.array([c["n"], c["kind"], c["R"], c["T"], c["sc"]], np.int64)
        old[f"{name}/seed"] = np.array(seeds, np.uint64)
        old[f"{name}/trial"] = np.array(c["check"], np.int64)
        old[f"{name}/best_energy"] = np.array([o.best_energy for o in res])
        old[f"{name}/best_replica"] = np.array([o.best_replica for o in res], np.int64)
        old[f"{name}/cycles_used"] = np.array([o.cycles_used for o in res], np.int64)
        old[f"{name}/trace_sha"] = np.array([sha(o.trace.astype(np.float64)) for o in res])
        old[f"{name}/state_sha"] = np.array([sha(o.best_state.astype(np.int8)) for o in res])
        peek = [cyc for cyc in PEEK if cyc <= c["sc"]]
        old[f"{name}/peek_cycle"] = np.array(peek, np.int64)
        old[f"{name}/peek_energy"] = np.array([[o.trace[cyc] for cyc in peek] for o in res])
        print(name, "best", old[f"{name}/best_energy"], "replica", old[f"{name}/best_replica"],
              f"{time.time() - t0:.0f} s", flush=True)
        np.savez_compressed(OUT, **old)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
