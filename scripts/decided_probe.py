"""How many replica-spin updates are decided by the integer field alone?

CPU probe behind the rail-tag epilogue: for a BASELINE
config it advances a few trials with the numpy restatement's arithmetic and
counts, per sweep, the updates whose new accumulator is a clamp rail whatever
the noise draw and the delayed neighbour are, given only the integer field
and whether the old accumulator sits on a rail (and which).  Also reports
how many 32-row x 8-column epilogue chunks have no undecided element.

    python scripts/decided_probe.py [c2|c3] [trials] [sweeps]
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2302_12454_b200 as sq  # noqa: E402
import lattice_np as ln  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    sc = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
    nn, r = (50, 20) if cfg == "c3" else (20, 20)
    m = sq.gi_ising(nn, 0.5, 7, True, 1.0, 1.0)
    h, J = np.asarray(m.h), np.asarray(m.J)
    n = len(h)
    p = ln.dyadic_scale(h, J)
    Jq = (J * 2.0 ** p).astype(np.float32)
    scale = 2.0 ** -p
    print(f"n={n} p={p} max|J'|={np.abs(Jq).max()} nnz/row={np.count_nonzero(Jq) / n:.0f}")
    i0, alpha, n_rnd, delay = 2.0, 1.0, 1.0, 1
    seeds = [1000 + t for t in range(T)]
    sig = np.empty((n, T * r))
    for t, s in enumerate(seeds):
        rb = ln.raw(ln.rng_key(s, ln.STREAM_SPIN_INIT), ln.spin_counters(0, n, r))
        sig[:, t * r:(t + 1) * r] = np.where((rb >> np.uint64(63)) != 0, 1.0, -1.0)
    acc = np.zeros((n, T * r))
    hist = [sig.copy() for _ in range(delay + 1)]
    keys = [ln.rng_key(s, ln.STREAM_SWEEP_NOISE) for s in seeds]
    kup = np.array([(k + 1) % r for k in range(r)])
    hi_rail, lo_rail = i0 - alpha, -i0

    class P:
        tau, beta, jperp_min, jperp_max = 100, 3, 0.0, 0.5
    jp = ln.jperp_schedule(P)
    npad = (n + 127) // 128 * 128
    report = set(list(range(0, 20)) + [50, 100, 150, 200, 300, 400, 500, 700, 1000, 1500, 2000,
                                       3000, 4000, 4999])
    tot_und = tot = 0
    for cycle in range(sc):
        F = h[:, None] + (Jq @ sig.astype(np.float32)).astype(np.float64) * scale
        jperp = jp(cycle)
        mrg = n_rnd + abs(jperp)
        on_hi = acc == hi_rail
        on_lo = acc == lo_rail
        # new acc is a rail whatever noise / neighbour do:
        dec_hi = np.where(on_hi, F - mrg >= i0 - hi_rail,
                          np.where(on_lo, F - mrg >= i0 - lo_rail, F - mrg >= 2 * i0))
        dec_lo = np.where(on_hi, F + mrg < -i0 - hi_rail,
                          np.where(on_lo, F + mrg < -i0 - lo_rail, F + mrg < -2 * i0))
        # acc-blind rule (no tag read): decided whatever the old accumulator is
        blind = (F - mrg >= 2 * i0) | (F + mrg < -2 * i0)
        und = ~(dec_hi | dec_lo)
        tot_und += und.sum()
        tot += und.size
        if cycle in report:
            up = np.zeros((npad, T * r), dtype=bool)
            up[:n] = und
            ch = up.reshape(npad // 32, 32, (T * r) // 4, 4)  # 32 rows x 4 cols
            c8 = up.reshape(npad // 32, 32, (T * r) // 4, 4).any(axis=(1, 3))
            # transposed blocking: one row x the 20 replicas of a trial, and one
            # row x 32 consecutive columns (what a warp would hold if the lanes
            # were replicas instead of rows)
            tr20 = und.reshape(n, T, r).any(axis=2).mean()
            w32 = und[:, : (T * r) // 32 * 32].reshape(n, -1, 32).any(axis=2).mean() \
                if T * r >= 32 else float("nan")
            print(f"cycle {cycle:5d} jperp {jperp:.3f} undecided {und.mean():.4f} "
                  f"blind-undecided {(~blind).mean():.4f} on-rail {(on_hi | on_lo).mean():.4f} "
                  f"32x4 chunks with any {c8.mean():.3f}  max per 32x4 chunk "
                  f"{ch.sum(axis=(1, 3)).max()}", flush=True)
            print(f"      row x {r} replicas of a trial with any {tr20:.3f}   row x 32 columns with "
                  f"any {w32:.3f}", flush=True)
        hcur = hist[cycle % (delay + 1)]
        for t in range(T):
            cols = slice(t * r, (t + 1) * r)
            rb = ln.raw(keys[t], ln.spin_counters(cycle, n, r))
            top = rb >> np.uint64(59)
            noise = np.where(top < 14, 0.0, np.where(top < 23, -1.0, 1.0))
            inp = F[:, cols] + n_rnd * noise
            inp = inp + jperp * hcur[:, cols][:, kup]
            s = acc[:, cols] + inp
            cl = np.where(s >= i0, hi_rail, np.where(s < -i0, lo_rail, s))
            # the rule must agree with the exact update
            d_hi, d_lo = dec_hi[:, cols], dec_lo[:, cols]
            assert np.all(cl[d_hi] == hi_rail) and np.all(cl[d_lo] == lo_rail)
            acc[:, cols] = cl
        sig = np.where(acc >= 0.0, 1.0, -1.0)
        hist[cycle % (delay + 1)] = sig.copy()
    print(f"overall undecided fraction {tot_und / tot:.5f}")


if __name__ == "__main__":
    main()
