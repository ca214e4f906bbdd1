"""ctypes wrappers for the CPU checkers under oracle/ -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py (its ``cpu_baseline``
leg and ``--impl reference``) import this module.  Two libraries share one
C interface (oracle/oracle_api.h):

* ``Oracle("orc")`` -- oracle/_build/libssqa_oracle.so, the scalar C
  restatement of the reference hot path (oracle/ssqa_oracle.c);
* ``Oracle("ref")`` -- oracle/_ref/libssqa_ref_{v4,v3}.so, the unmodified
  reference sources (/root/reference/proj/src) compiled by oracle/Makefile.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


class OrcParams(C.Structure):
    _fields_ = [
        ("r", C.c_int), ("jperp_min", C.c_double), ("jperp_max", C.c_double),
        ("beta", C.c_int), ("tau", C.c_int), ("delay", C.c_int), ("i0", C.c_double),
        ("n_rnd", C.c_double), ("alpha", C.c_double), ("sc", C.c_long),
        ("bidirectional", C.c_int),
    ]


class OrcSsaParams(C.Structure):
    _fields_ = [
        ("i0_min", C.c_double), ("i0_max", C.c_double), ("beta", C.c_double),
        ("tau", C.c_int), ("n_rnd", C.c_double), ("alpha", C.c_double), ("sc", C.c_long),
    ]


class OrcResult(C.Structure):
    _fields_ = [
        ("best_energy", C.c_double), ("best_replica", C.c_int), ("reached_target", C.c_int),
        ("first_hit_cycle", C.c_long), ("cycles_used", C.c_long), ("trace_len", C.c_long),
        ("wall_seconds", C.c_double),
    ]


class OrcTrial(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("reached_target", C.c_int), ("first_hit_cycle", C.c_long),
        ("best_energy", C.c_double), ("wall_seconds", C.c_double),
    ]


def _has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return "avx512f" in line.split()
    except OSError:
        pass
    return False


def lib_path(kind: str) -> str:
    if kind == "orc":
        return os.path.join(HERE, "_build", "libssqa_oracle.so")
    v = "v4" if _has_avx512() else "v3"
    return os.path.join(HERE, "_ref", f"libssqa_ref_{v}.so")


def available(kind: str) -> bool:
    return os.path.exists(lib_path(kind))


def params(r, sc, jperp_min=0.0, jperp_max=0.5, beta=3, tau=100, delay=1, i0=2.0,
           n_rnd=1.0, alpha=1.0, bidirectional=False) -> OrcParams:
    """Defaults mirror ssqa::SsqaParams (annealer.hpp:14-30)."""
    return OrcParams(r, jperp_min, jperp_max, beta, tau, delay, i0, n_rnd, alpha, sc,
                     int(bidirectional))


def ssa_params(sc, i0_min=1.0, i0_max=16.0, beta=0.5, tau=10, n_rnd=1.0,
               alpha=1.0) -> OrcSsaParams:
    """Defaults mirror ssqa::SsaParams (annealer.hpp:38-50)."""
    return OrcSsaParams(i0_min, i0_max, beta, tau, n_rnd, alpha, sc)


@dataclass
class RunOut:
    best_energy: float
    best_replica: int
    reached_target: bool
    first_hit_cycle: int
    cycles_used: int
    wall_seconds: float
    best_state: np.ndarray
    trace: np.ndarray


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Oracle:
    def __init__(self, kind: str = "orc"):
        assert kind in ("orc", "ref")
        self.kind = kind
        self.lib = C.CDLL(lib_path(kind))
        p = kind + "_"
        L = self.lib
        self._f = lambda name: getattr(L, p + name)
        self._f("last_error").restype = C.c_char_p
        for name in ("mix64",):
            self._f(name).restype = C.c_uint64
            self._f(name).argtypes = [C.c_uint64]
        self._f("rng_key").restype = C.c_uint64
        self._f("rng_key").argtypes = [C.c_uint64, C.c_uint32]
        self._f("rng_raw").restype = C.c_uint64
        self._f("rng_raw").argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
        self._f("rng_uniform01").restype = C.c_double
        self._f("rng_uniform01").argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
        self._f("spin_counter").restype = C.c_uint64
        self._f("spin_counter").argtypes = [C.c_uint64, C.c_int, C.c_int]
        if kind == "ref":
            L.ref_run_trials.argtypes = [
                C.POINTER(OrcParams), C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                C.c_int, C.c_uint64, C.c_int, C.c_long, C.c_double, C.c_uint64, C.c_int,
                C.POINTER(OrcTrial), C.POINTER(C.c_double), C.POINTER(C.c_double),
                C.POINTER(C.c_double), C.POINTER(C.c_int)]
            L.ref_gi_ising.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_double,
                                       C.c_double, C.c_void_p, C.c_void_p,
                                       C.POINTER(C.c_double)]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._f("last_error")().decode())

    # ---- rng.hpp ----
    def mix64(self, x): return self._f("mix64")(x)
    def rng_key(self, seed, stream): return self._f("rng_key")(seed, stream)
    def rng_raw(self, seed, stream, c): return self._f("rng_raw")(seed, stream, c)
    def uniform01(self, seed, stream, c): return self._f("rng_uniform01")(seed, stream, c)
    def spin_counter(self, cyc, k, i): return self._f("spin_counter")(cyc, k, i)

    def jperp_schedule(self, cycle, p: OrcParams) -> float:
        out = C.c_double()
        self._check(self._f("jperp_schedule")(C.c_long(cycle), C.byref(p), C.byref(out)))
        return out.value

    # ---- lattice API (annealer.hpp:68-93) ----
    def init_lattice(self, n, r, d, seed):
        sigma = np.zeros(n * r)
        acc = np.zeros(n * r)
        hist = np.zeros((d + 1) * n * r)
        self._check(self._f("init_lattice")(n, r, d, C.c_uint64(seed), _dp(sigma), _dp(acc),
                                            _dp(hist)))
        return sigma, acc, hist.reshape(d + 1, n * r)

    def ssqa_sweep(self, h, J, offset, jperp, p: OrcParams, seed, cycle, sigma, acc, hist,
                   lat_cycle):
        """In-place sweep of (sigma, acc, hist); returns the new lattice cycle."""
        n = len(h)
        lc = C.c_long(lat_cycle)
        hist_c = np.ascontiguousarray(hist)
        self._check(self._f("ssqa_sweep")(
            n, _dp(np.ascontiguousarray(h, dtype=np.float64)),
            _dp(np.ascontiguousarray(J, dtype=np.float64)), C.c_double(offset),
            C.c_double(jperp), C.byref(p), C.c_uint64(seed), C.c_long(cycle), _dp(sigma),
            _dp(acc), _dp(hist_c), C.byref(lc)))
        hist[...] = hist_c
        return lc.value

    def replica_energies(self, h, J, offset, r, sigma):
        out = np.zeros(r)
        self._check(self._f("replica_energies")(
            len(h), _dp(np.ascontiguousarray(h, dtype=np.float64)),
            _dp(np.ascontiguousarray(J, dtype=np.float64)), C.c_double(offset), r,
            _dp(np.ascontiguousarray(sigma)), _dp(out)))
        return out

    def ssqa_run(self, h, J, offset, p: OrcParams, seed, target=None, record_trace=False,
                 stop_at_target=True) -> RunOut:
        n = len(h)
        res = OrcResult()
        best = np.zeros(n, dtype=np.int8)
        trace = np.zeros((p.sc + 1) * p.r if record_trace else 1)
        self._check(self._f("ssqa_run")(
            n, _dp(np.ascontiguousarray(h, dtype=np.float64)),
            _dp(np.ascontiguousarray(J, dtype=np.float64)), C.c_double(offset), C.byref(p),
            C.c_uint64(seed), int(target is not None),
            C.c_double(0.0 if target is None else target), int(record_trace),
            int(stop_at_target), C.byref(res), best.ctypes.data_as(C.POINTER(C.c_int8)),
            _dp(trace)))
        return RunOut(res.best_energy, res.best_replica, bool(res.reached_target),
                      res.first_hit_cycle, res.cycles_used, res.wall_seconds, best,
                      trace[:res.trace_len] if record_trace else np.zeros(0))

    def i0_schedule(self, cycle, p: OrcSsaParams) -> float:
        out = C.c_double()
        self._check(self._f("i0_schedule")(C.c_long(cycle), C.byref(p), C.byref(out)))
        return out.value

    def ssa_run(self, h, J, offset, p: OrcSsaParams, seed, target=None, record_trace=False,
                stop_at_target=True) -> RunOut:
        n = len(h)
        res = OrcResult()
        best = np.zeros(n, dtype=np.int8)
        trace = np.zeros(p.sc + 1 if record_trace else 1)
        self._check(self._f("ssa_run")(
            n, _dp(np.ascontiguousarray(h, dtype=np.float64)),
            _dp(np.ascontiguousarray(J, dtype=np.float64)), C.c_double(offset), C.byref(p),
            C.c_uint64(seed), int(target is not None),
            C.c_double(0.0 if target is None else target), int(record_trace),
            int(stop_at_target), C.byref(res), best.ctypes.data_as(C.POINTER(C.c_int8)),
            _dp(trace)))
        return RunOut(res.best_energy, res.best_replica, bool(res.reached_target),
                      res.first_hit_cycle, res.cycles_used, res.wall_seconds, best,
                      trace[:res.trace_len] if record_trace else np.zeros(0))

    # ---- reference-only helpers ----
    def ssqa_run_many(self, h, J, offset, p: OrcParams, seeds, workers):
        """ref_ssqa_run_many: every seed on `workers` threads, one shared model."""
        assert self.kind == "ref"
        s = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        out = np.zeros(len(s))
        self._check(self.lib.ref_ssqa_run_many(
            len(h), _dp(np.ascontiguousarray(h, dtype=np.float64)),
            _dp(np.ascontiguousarray(J, dtype=np.float64)), C.c_double(offset), C.byref(p),
            s.ctypes.data_as(C.POINTER(C.c_uint64)), len(s), workers, _dp(out)))
        return out

    def bench_manifest(self, p: OrcParams, n_nodes, trials, ec, base_seed, workers,
                       edge_prob=0.5, permute=False, c1=0.75, c2=0.75, fresh_instance=True,
                       gi_seed=0, p_target=0.99) -> str:
        """The reference's make_manifest("bench", ...) of a run_trials, as JSON text."""
        assert self.kind == "ref"
        cap = 1 << 22
        buf = C.create_string_buffer(cap)
        f = self.lib.ref_bench_manifest
        f.restype = C.c_long
        f.argtypes = [C.POINTER(OrcParams), C.c_int, C.c_double, C.c_int, C.c_double,
                      C.c_double, C.c_int, C.c_uint64, C.c_int, C.c_long, C.c_double,
                      C.c_uint64, C.c_int, C.c_char_p, C.c_long]
        n = f(C.byref(p), n_nodes, edge_prob, int(permute), c1, c2, int(fresh_instance),
              gi_seed, trials, ec, p_target, base_seed, workers, buf, cap)
        if n < 0:
            raise OracleError(2, self.lib.ref_last_error().decode())
        return buf.value.decode()

    def gi_ising(self, n_nodes, edge_prob, seed, permute, c1, c2):
        assert self.kind == "ref"
        n = n_nodes * n_nodes
        h = np.zeros(n)
        J = np.zeros((n, n))
        off = C.c_double()
        self._check(self.lib.ref_gi_ising(n_nodes, edge_prob, C.c_uint64(seed), int(permute),
                                          c1, c2, h.ctypes.data, J.ctypes.data, C.byref(off)))
        return h, J, off.value

    def run_trials(self, p: OrcParams, n_nodes, trials, ec, base_seed, workers,
                   edge_prob=0.5, permute=True, c1=1.0, c2=1.0, fresh_instance=False,
                   gi_seed=7, p_target=0.99):
        assert self.kind == "ref"
        outs = (OrcTrial * trials)()
        ps, tm, tts = C.c_double(), C.c_double(), C.c_double()
        kind = C.c_int()
        self._check(self.lib.ref_run_trials(
            C.byref(p), n_nodes, edge_prob, int(permute), c1, c2, int(fresh_instance),
            C.c_uint64(gi_seed), trials, C.c_long(ec), p_target, C.c_uint64(base_seed),
            workers, outs, C.byref(ps), C.byref(tm), C.byref(tts), C.byref(kind)))
        return [dict(seed=o.seed, reached_target=bool(o.reached_target),
                     first_hit_cycle=o.first_hit_cycle, best_energy=o.best_energy,
                     wall_seconds=o.wall_seconds) for o in outs], ps.value, tm.value, \
            (tts.value, kind.value)
