"""Run tcgen05 batches over shapes; print OK/MISMATCH/ERROR per shape (one process per shape)."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys; sys.path.insert(0, "{root}"); sys.path.insert(0, "{root}/oracle")
import numpy as np, paper_2302_12454_b200 as sq
from paper_2302_12454_b200 import _lib
from oracle_py import Oracle, params
nn, R, T, sc = {nn}, {R}, {T}, {sc}
m = sq.gi_ising(nn, 0.5, 7, True, 1.0, 1.0)
res = sq.ssqa_run_batch(m, sq.SsqaParams(r=R, sc=sc), list(range(T)), 0.0, sq.RunOptions(True, False), engine=_lib.ENGINE_TCGEN05)
o = Oracle("orc")
bad = 0
for t in sorted(set([0, T // 2, T - 1])):
    ob = o.ssqa_run(m.h, m.J, m.offset, params(R, sc), t, 0.0, True, False)
    bad += not np.array_equal(res[t].trace_energy.view(np.uint64), ob.trace.view(np.uint64))
print("OK" if not bad else "MISMATCH")
'''
for nn, R, T, sc in [tuple(map(int, a.split(","))) for a in sys.argv[1:]]:
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT, nn=nn, R=R, T=T, sc=sc)],
                       capture_output=True, text=True, timeout=120)
    out = (r.stdout.strip().splitlines() or [""])[-1]
    err = (r.stderr.strip().splitlines() or [""])[-1]
    print(f"n_nodes={nn} R={R} T={T} sc={sc}: {out or 'ERROR ' + err}", flush=True)
