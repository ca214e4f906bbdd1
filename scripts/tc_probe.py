"""Quick tcgen05 engine probe: one small batch vs the oracle (run under timeout)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import paper_2302_12454_b200 as sq
from paper_2302_12454_b200 import _lib
from oracle_py import Oracle, params
orc = Oracle("orc")
for nn, R, sc, T in [(10, 20, 50, 3), (12, 8, 30, 5), (20, 20, 20, 4)]:
    m = sq.gi_ising(nn, 0.5, 7, True, 1.0, 1.0)
    p = sq.SsqaParams(r=R, sc=sc)
    seeds = list(range(100, 100 + T))
    t0 = time.time()
    res = sq.ssqa_run_batch(m, p, seeds, 0.0, sq.RunOptions(True, False), engine=_lib.ENGINE_TCGEN05)
    print(f"n={m.n} R={R} sc={sc} T={T}: tc run {time.time()-t0:.3f}s", flush=True)
    for t in range(T):
        o = orc.ssqa_run(m.h, m.J, m.offset, params(R, sc), seeds[t], 0.0, True, False)
        r = res[t]
        ok = (r.best_energy == o.best_energy and np.array_equal(r.best_state, o.best_state)
              and np.array_equal(r.trace_energy.view(np.uint64), o.trace.view(np.uint64)))
        first_bad = None
        if not ok:
            d = np.nonzero(r.trace_energy != o.trace)[0]
            first_bad = (int(d[0]) // R, r.trace_energy[d[0]], o.trace[d[0]]) if len(d) else "state"
        print(f"  trial {t}: {'OK' if ok else 'MISMATCH'} best {r.best_energy} vs {o.best_energy} first_bad={first_bad}", flush=True)
