"""Vectorised numpy restatement of run_lattice -- TEST INFRASTRUCTURE ONLY.

Same algorithm as oracle/ssqa_oracle.c (each step cites the reference lines
it follows), written with numpy arrays so the full-size BASELINE configs
(N = 8192 and N = 32768 dense models) can be checked over their first steps:

* fields (annealer.cpp:216-242): h_i + sum_j J_ij sigma_j.  For the dyadic
  models the engine accepts, J * 2^p is integral and every partial sum is an
  exact integer, so a BLAS product is exact in any summation order: float32
  when max|J * 2^p| * n < 2^24, float64 otherwise;
* energies (annealer.cpp:246-256): -0.5 * sum_i sigma_i (F_i + h_i) + offset,
  exact sums of dyadic values, one final rounding as the reference;
* update_spins (annealer.cpp:258-300): the reference's per-element operation
  order (input = F; += n_rnd * noise; += jperp * sigma_up [+ sigma_dn];
  s = acc + input; clamp; sign) as elementwise IEEE double operations --
  numpy never contracts them;
* noise / init draws (rng.hpp:10-67): splitmix64 on uint64 arrays, the noise
  class from the top five bits (u < 7/16 <=> raw >> 59 < 14, u < 23/32 <=>
  raw >> 59 < 23; the identity checked in tests/test_oracle_golden.py).

Pinned against oracle/ssqa_oracle.c and the reference fixtures by
tests/test_oracle_golden.py::test_numpy_lattice_matches_oracle.  Only tests/
use it, as a checker.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
STREAM_SPIN_INIT, STREAM_SWEEP_NOISE = 1, 2  # rng.hpp:20-28


def mix64(x: np.ndarray) -> np.ndarray:
    """rng.hpp:10-15 (uint64 arithmetic wraps as in C)."""
    with np.errstate(over="ignore"):
        x = x + GOLDEN
        x = (x ^ (x >> np.uint64(30))) * M1
        x = (x ^ (x >> np.uint64(27))) * M2
        return x ^ (x >> np.uint64(31))


def rng_key(seed: int, stream: int) -> np.uint64:
    """rng.hpp:33-34: mix64(mix64(seed) ^ (2^32 + stream))."""
    s = mix64(np.array([seed], dtype=np.uint64))
    return mix64(s ^ np.uint64((1 << 32) + stream))[0]


def raw(key: np.uint64, counter: np.ndarray) -> np.ndarray:
    """rng.hpp:36-38."""
    with np.errstate(over="ignore"):
        return mix64(key + counter * GOLDEN)


def spin_counters(cycle: int, n: int, r: int) -> np.ndarray:
    """rng.hpp:65-67, laid out [i, k]."""
    i = np.arange(n, dtype=np.uint64)[:, None]
    k = np.arange(r, dtype=np.uint64)[None, :]
    return (np.uint64(cycle) << np.uint64(32)) | (k << np.uint64(20)) | i


def dyadic_scale(h: np.ndarray, J: np.ndarray) -> int:
    """Smallest p with h*2^p and J*2^p integral (the engine's quantizer)."""
    for p in range(0, 31):
        f = float(2 ** p)
        if np.all(np.floor(h * f) == h * f) and np.all(np.floor(J * f) == J * f):
            return p
    raise ValueError("model is not dyadic")


@dataclass
class TrialOut:
    best_energy: float
    best_replica: int
    reached_target: bool
    first_hit_cycle: int
    cycles_used: int
    best_state: np.ndarray
    trace: np.ndarray  # [cycles_used + 1, r]


def run_lattice(h: np.ndarray, J: np.ndarray, offset: float, r: int, delay: int,
                n_rnd: float, alpha: float, bidirectional: bool, sc: int,
                jperp_at: Callable[[int], float], i0_at: Callable[[int], float],
                seeds: Sequence[int], target: Optional[float] = None,
                stop_at_target: bool = False, max_cycles: Optional[int] = None,
                J_scaled: Optional[np.ndarray] = None) -> List[TrialOut]:
    """run_lattice (annealer.cpp:313-361) for every seed, all trials advanced
    together.  max_cycles stops after that many updates (for checking the
    first steps of a long run: results then describe cycles 0..max_cycles).
    J_scaled: optional precomputed J * 2^p (float32/float64) to avoid a copy."""
    n = len(h)
    T = len(seeds)
    p = dyadic_scale(h, J) if J_scaled is None else 0
    if J_scaled is None:
        Jq = J * float(2 ** p)
        bound = float(np.abs(Jq).max()) * n
        Jq = Jq.astype(np.float32) if bound < 2 ** 24 else Jq
    else:
        Jq = J_scaled
    scale = 2.0 ** -p
    h = np.asarray(h, dtype=np.float64)
    # init_lattice (annealer.cpp:432-447): sigma = pm1(raw(spin_counter(0,k,i)))
    sig = np.empty((n, T * r))
    for t, s in enumerate(seeds):
        rb = raw(rng_key(s, STREAM_SPIN_INIT), spin_counters(0, n, r))
        sig[:, t * r:(t + 1) * r] = np.where((rb >> np.uint64(63)) != 0, 1.0, -1.0)
    acc = np.zeros((n, T * r))
    hist = [sig.copy() for _ in range(delay + 1)]
    keys = [rng_key(s, STREAM_SWEEP_NOISE) for s in seeds]
    kup = np.array([(k + 1) % r for k in range(r)])
    kdn = np.array([(k - 1) % r for k in range(r)])
    tol = 1e-9  # annealer.hpp:113

    best_e = np.full(T, np.inf)
    best_k = np.zeros(T, dtype=int)
    best_state = np.zeros((T, n), dtype=np.int8)
    reached = np.zeros(T, dtype=bool)
    first_hit = np.full(T, -1)
    cycles_used = np.full(T, -1)
    active = np.ones(T, dtype=bool)
    traces = [[] for _ in range(T)]
    last = sc if max_cycles is None else min(sc, max_cycles)
    for cycle in range(last + 1):
        # compute_fields: exact integer product, rescaled exactly
        S = (Jq @ sig.astype(Jq.dtype)).astype(np.float64) * scale if scale != 1.0 else \
            (Jq @ sig.astype(Jq.dtype)).astype(np.float64)
        F = h[:, None] + S
        # energies_from_fields + scan_state (annealer.cpp:327-345)
        E = -0.5 * np.sum(sig * (F + h[:, None]), axis=0) + offset
        for t in range(T):
            if not active[t]:
                continue
            et = E[t * r:(t + 1) * r]
            traces[t].append(et.copy())
            for k in range(r):
                if et[k] < best_e[t]:
                    best_e[t] = et[k]
                    best_k[t] = k
                    best_state[t] = np.where(sig[:, t * r + k] > 0, 1, -1)
                    if target is not None and not reached[t] and best_e[t] <= target + tol:
                        reached[t] = True
                        first_hit[t] = cycle
        if cycle == sc:
            for t in range(T):
                if active[t]:
                    cycles_used[t] = cycle
            break
        for t in range(T):
            if active[t] and stop_at_target and reached[t]:
                active[t] = False
                cycles_used[t] = cycle
        if cycle == last or not active.any():
            for t in range(T):
                if active[t]:
                    cycles_used[t] = cycle
            break
        # update_spins (annealer.cpp:258-300)
        jperp, i0 = jperp_at(cycle), i0_at(cycle)
        hi = hist[cycle % (delay + 1)]
        new_sig = sig.copy()
        for t in range(T):
            if not active[t]:
                continue
            cols = slice(t * r, (t + 1) * r)
            rb = raw(keys[t], spin_counters(cycle, n, r))
            top = rb >> np.uint64(59)
            noise = np.where(top < 14, 0.0, np.where(top < 23, -1.0, 1.0))
            inp = F[:, cols] + n_rnd * noise
            hloc = hi[:, cols]
            inp = inp + jperp * hloc[:, kup]
            if bidirectional:
                inp = inp + jperp * hloc[:, kdn]
            s = acc[:, cols] + inp
            clamped = np.where(s >= i0, i0 - alpha, np.where(s < -i0, -i0, s))
            acc[:, cols] = clamped
            new_sig[:, cols] = np.where(clamped >= 0.0, 1.0, -1.0)
        sig = new_sig
        hist[cycle % (delay + 1)] = sig.copy()
    return [TrialOut(float(best_e[t]), int(best_k[t]), bool(reached[t]), int(first_hit[t]),
                     int(cycles_used[t]), best_state[t], np.array(traces[t]))
            for t in range(T)]


def jperp_schedule(p) -> Callable[[int], float]:
    """annealer.cpp:375-380 for an oracle_py.OrcParams."""
    def f(c: int) -> float:
        cc = c % (p.tau * (p.beta + 1))
        step = cc // p.tau
        return p.jperp_min + float(step) * (p.jperp_max - p.jperp_min) / p.beta
    return f
