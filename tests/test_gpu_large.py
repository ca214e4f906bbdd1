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
