"""Python mirror of the reference annealer API, served by the B200 engine.

Names, argument meaning and error behaviour follow the reference C++ API
(proj/include/ssqa/annealer.hpp, bench.hpp): ``SsqaParams``, ``SsaParams``,
``RunOptions``, ``AnnealResult``, ``ReplicaLattice``, ``init_lattice``,
``ssqa_sweep``, ``replica_energies``, ``jperp_schedule``, ``i0_schedule``,
``ssqa_run``, ``ssa_run`` and ``run_trials``.
std::invalid_argument surfaces as ``ValueError`` (``SsqaInvalidArgument``).
Everything runs through the C ABI of include/ssqa_cuda.h; there is no Python
or CPU compute path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import ENGINE_AUTO, ParamsC, ResultC, SsaParamsC, check, lib

K_TARGET_TOL = 1e-9  # annealer.hpp:113


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class SsqaParams:
    """ssqa::SsqaParams (annealer.hpp:14-30); r and sc come from the caller."""
    r: int = 0
    jperp_min: float = 0.0
    jperp_max: float = 0.5
    beta: int = 3
    tau: int = 100
    delay: int = 1
    i0: float = 2.0
    n_rnd: float = 1.0
    alpha: float = 1.0
    sc: int = 0
    bidirectional: bool = False

    def cycles_per_iteration(self) -> int:
        return self.tau * (self.beta + 1)

    def iterations(self) -> int:
        return self.sc // self.cycles_per_iteration()

    def to_c(self) -> ParamsC:
        return ParamsC(self.r, self.jperp_min, self.jperp_max, self.beta, self.tau, self.delay,
                       self.i0, self.n_rnd, self.alpha, self.sc, int(self.bidirectional))

    def validate(self, n: int) -> None:
        check(lib().ssqa_params_validate(C.byref(self.to_c()), n))


@dataclass
class SsaParams:
    """ssqa::SsaParams (annealer.hpp:38-50): one network whose accumulator
    bound climbs i0_min, i0_min/beta, ... <= i0_max every tau cycles."""
    i0_min: float = 1.0
    i0_max: float = 16.0
    beta: float = 0.5
    tau: int = 10
    n_rnd: float = 1.0
    alpha: float = 1.0
    sc: int = 0

    def to_c(self) -> SsaParamsC:
        return SsaParamsC(self.i0_min, self.i0_max, self.beta, self.tau, self.n_rnd,
                          self.alpha, self.sc)

    def i0_levels(self) -> List[float]:
        buf = (C.c_double * 65)()
        cnt = C.c_int()
        check(lib().ssqa_i0_levels(C.byref(self.to_c()), buf, C.byref(cnt)))
        return list(buf[: cnt.value])

    def cycles_per_iteration(self) -> int:
        return len(self.i0_levels()) * self.tau

    def validate(self, n: int) -> None:
        check(lib().ssqa_ssa_params_validate(C.byref(self.to_c()), n))


def i0_schedule(cycle: int, p: SsaParams) -> float:
    """annealer.cpp:403-408."""
    out = C.c_double()
    check(lib().ssqa_i0_schedule(cycle, C.byref(p.to_c()), C.byref(out)))
    return out.value


@dataclass
class RunOptions:
    record_trace: bool = False
    stop_at_target: bool = True


@dataclass
class TracePoint:
    cycle: int
    replica: int
    energy: float
    jperp: float


@dataclass
class AnnealResult:
    best_energy: float = 0.0
    best_state: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int8))
    best_replica: int = 0
    reached_target: bool = False
    first_hit_cycle: int = -1
    cycles_used: int = 0
    trace_energy: np.ndarray = field(default_factory=lambda: np.zeros(0))
    wall_seconds: float = 0.0
    # per-cycle jperp of the recorded cycles (SSA: zeros), set with trace_energy
    trace_jperp: np.ndarray = field(default_factory=lambda: np.zeros(0), repr=False)

    @property
    def trace(self) -> List[TracePoint]:
        """AnnealResult::trace (annealer.cpp:343): one TracePoint per replica and
        scanned cycle, cycle-major, replica-minor, with the cycle's jperp."""
        ncyc = len(self.trace_jperp)
        if ncyc == 0:
            return []
        r = len(self.trace_energy) // ncyc
        return [TracePoint(c, k, float(self.trace_energy[c * r + k]), float(self.trace_jperp[c]))
                for c in range(ncyc) for k in range(r)]


class IsingModel:
    """Dense mirrored Ising model, ssqa::IsingModel storage (model.hpp:45-67)."""

    def __init__(self, n: int, offset: float = 0.0):
        if n < 1:
            raise ValueError("IsingModel needs n >= 1")
        self.h = np.zeros(n)
        self.J = np.zeros((n, n))
        self.offset = float(offset)

    @property
    def n(self) -> int:
        return len(self.h)

    @classmethod
    def from_arrays(cls, h, J, offset=0.0) -> "IsingModel":
        m = cls(len(h), offset)
        m.h = np.ascontiguousarray(h, dtype=np.float64).copy()
        m.J = np.ascontiguousarray(J, dtype=np.float64).copy()
        return m

    def set_bias(self, i, v):
        self.h[i] = v

    def set_coupling(self, i, j, v):
        if i == j:
            raise ValueError("coupling needs i != j")
        self.J[i, j] = v
        self.J[j, i] = v


def gi_ising(n_nodes: int, edge_prob: float = 0.5, seed: int = 0, permute: bool = True,
             c1: float = 0.75, c2: float = 0.75) -> IsingModel:
    """qubo_to_ising(build_gi_qubo(generate_gi(...))) -- gi.cpp:102-184."""
    n = n_nodes * n_nodes
    h = np.zeros(n)
    J = np.zeros((n, n))
    off = C.c_double()
    check(lib().ssqa_gi_ising(n_nodes, edge_prob, seed, int(permute), c1, c2, _dp(h), _dp(J),
                              C.byref(off)), host=True)
    return IsingModel.from_arrays(h, J, off.value)


def gi_compact(n_nodes: int, edge_prob: float = 0.5, seed: int = 0, permute: bool = True,
               c1: float = 0.75, c2: float = 0.75):
    """Host half of the device GI generator: adjacency [2, n, n] (graph 1, graph
    2) and the closed-form biases / offset (equal to gi_ising's for dyadic c)."""
    N = n_nodes * n_nodes
    adj = np.zeros((2, n_nodes, n_nodes), dtype=np.uint8)
    h = np.zeros(N)
    off = C.c_double()
    check(lib().ssqa_gi_compact(n_nodes, edge_prob, seed, int(permute), c1, c2,
                                adj.ctypes.data_as(C.c_void_p), _dp(h), C.byref(off)), host=True)
    return adj, h, off.value


def dense_ising(n: int, kind: int, seed: int) -> IsingModel:
    """BASELINE configs C4 (kind 0, int[-8,7]) / C5 (kind 1, SK +-1)."""
    h = np.zeros(n)
    J = np.zeros((n, n))
    off = C.c_double()
    check(lib().ssqa_dense_ising(n, kind, seed, _dp(h), _dp(J), C.byref(off)), host=True)
    return IsingModel.from_arrays(h, J, off.value)


def ising_energy(m: IsingModel, spins) -> float:
    s = np.ascontiguousarray(spins, dtype=np.int8)
    out = C.c_double()
    check(lib().ssqa_ising_energy(m.n, _dp(m.h), _dp(m.J), m.offset,
                                  s.ctypes.data_as(C.POINTER(C.c_int8)), C.byref(out)), host=True)
    return out.value


def jperp_schedule(cycle: int, p: SsqaParams) -> float:
    out = C.c_double()
    check(lib().ssqa_jperp_schedule(cycle, C.byref(p.to_c()), C.byref(out)))
    return out.value


class Problem:
    """Quantized model on one device (ssqa_problem_create)."""

    def __init__(self, m: IsingModel, device: int = 0):
        self.n = m.n
        self._h = C.c_void_p()
        check(lib().ssqa_problem_create(m.n, _dp(np.ascontiguousarray(m.h)),
                                        _dp(np.ascontiguousarray(m.J)), m.offset, device,
                                        C.byref(self._h)))

    @classmethod
    def from_models(cls, models: Sequence[IsingModel], device: int = 0) -> "Problem":
        """One problem holding a fresh instance per trial
        (ssqa_problem_create_many; a batch on it runs trial t on models[t])."""
        self = cls.__new__(cls)
        n = models[0].n
        assert all(mm.n == n for mm in models), "instances must have the same size"
        self.n = n
        self._h = C.c_void_p()
        h = np.ascontiguousarray(np.concatenate([mm.h for mm in models]))
        J = np.ascontiguousarray(np.concatenate([mm.J.reshape(-1) for mm in models]))
        off = np.ascontiguousarray([mm.offset for mm in models], dtype=np.float64)
        check(lib().ssqa_problem_create_many(len(models), n, _dp(h), _dp(J), _dp(off), device,
                                             C.byref(self._h)))
        return self

    @classmethod
    def zero(cls, n: int, device: int = 0) -> "Problem":
        """All-zero n-spin problem made on the device (ssqa_problem_create_zero)."""
        self = cls.__new__(cls)
        self.n = n
        self._h = C.c_void_p()
        check(lib().ssqa_problem_create_zero(n, device, C.byref(self._h)))
        return self

    @classmethod
    def generated_dense(cls, n: int, kind: int, seed: int, device: int = 0) -> "Problem":
        """BASELINE C4 / C5 model built on the device (ssqa_problem_create_dense):
        the same quantized problem as Problem(dense_ising(n, kind, seed))."""
        self = cls.__new__(cls)
        self.n = n
        self._h = C.c_void_p()
        check(lib().ssqa_problem_create_dense(n, kind, seed, device, C.byref(self._h)))
        return self

    @classmethod
    def generated_gi(cls, n_nodes: int, seeds: Sequence[int], edge_prob: float = 0.5,
                     permute: bool = True, c1: float = 0.75, c2: float = 0.75,
                     device: int = 0) -> "Problem":
        """GI instance(s) built on the device (ssqa_problem_create_gi): one per
        seed, stacked like Problem.from_models([gi_ising(n_nodes, edge_prob, s,
        permute, c1, c2) for s in seeds]) (a single seed: a one-instance problem)."""
        self = cls.__new__(cls)
        self.n = n_nodes * n_nodes
        self._h = C.c_void_p()
        sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        check(lib().ssqa_problem_create_gi(len(sd), n_nodes, edge_prob,
                                           sd.ctypes.data_as(C.c_void_p), int(permute), c1, c2,
                                           device, C.byref(self._h)))
        return self

    def export(self):
        """(J' int8 [count*npad, npad], H' int32 [count*npad], offsets [count])."""
        inf = self.info()
        cnt = int(lib().ssqa_problem_count(self._h))
        npad = inf["n_pad"]
        J = np.zeros((cnt * npad, npad * (2 if inf["int16"] else 1)), dtype=np.int8)
        H = np.zeros(cnt * npad, dtype=np.int32)
        off = np.zeros(cnt)
        check(lib().ssqa_problem_export(self._h, J.ctypes.data_as(C.c_void_p),
                                        H.ctypes.data_as(C.c_void_p), _dp(off)))
        return J, H, off

    def info(self) -> dict:
        v = [C.c_int() for _ in range(5)]
        check(lib().ssqa_problem_info(self._h, *[C.byref(x) for x in v]))
        d = dict(zip(("n", "n_pad", "shift_p", "max_abs_j", "max_abs_h"), [x.value for x in v]))
        # FP4 (e2m1) image uploaded when every coupling is 0, +-1, +-2, +-3, +-4 or +-6
        d["fp4"] = int(lib().ssqa_problem_fp4(self._h))
        # int16 couplings held as two int8 planes (J' = 256 Ahi + Alo)
        d["int16"] = int(lib().ssqa_problem_int16(self._h))
        return d

    def close(self):
        if self._h:
            lib().ssqa_problem_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Batch:
    """Device-resident state for `trials` x r replica columns (ssqa_batch_*).
    An ``SsaParams`` batch is the SSA engine (r = 1, delay = 0)."""

    def __init__(self, prob: Problem, p, trials: int, record_trace: bool = False,
                 engine: int = ENGINE_AUTO):
        self.prob, self.p, self.trials, self.record_trace = prob, p, trials, record_trace
        self._b = C.c_void_p()
        if isinstance(p, SsaParams):
            self.r, self.delay = 1, 0
            check(lib().ssqa_batch_create_ssa(prob._h, C.byref(p.to_c()), trials,
                                              int(record_trace), engine, C.byref(self._b)))
        else:
            self.r, self.delay = p.r, p.delay
            check(lib().ssqa_batch_create(prob._h, C.byref(p.to_c()), trials,
                                          int(record_trace), engine, C.byref(self._b)))

    @property
    def engine(self) -> int:
        return lib().ssqa_batch_engine(self._b)

    @property
    def operand_bits(self) -> int:
        """4 (FP4 e2m1 operands) or 8 (int8) for the contraction."""
        return lib().ssqa_batch_operand_bits(self._b)

    @property
    def stream(self) -> int:
        return lib().ssqa_batch_stream(self._b) or 0

    def set_seeds(self, seeds: Sequence[int]):
        s = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        assert len(s) == self.trials
        check(lib().ssqa_batch_set_seeds(self._b, s.ctypes.data_as(C.POINTER(C.c_uint64))))

    def launch(self, target: Optional[float] = None, stop_at_target: bool = True):
        check(lib().ssqa_batch_launch(self._b, int(target is not None),
                                      0.0 if target is None else float(target),
                                      int(stop_at_target)))

    def launch_count(self) -> int:
        return lib().ssqa_batch_launch_count(self._b)

    def elapsed_ms(self) -> float:
        out = C.c_double()
        check(lib().ssqa_batch_elapsed_ms(self._b, C.byref(out)))
        return out.value

    def synchronize(self) -> None:
        """Wait for everything queued on the batch stream."""
        check(lib().ssqa_batch_synchronize(self._b))

    def profile_field(self, iters: int = 20) -> float:
        out = C.c_double()
        check(lib().ssqa_batch_profile_field(self._b, iters, C.byref(out)))
        return out.value

    def fetch(self, best_states: bool = True, trace: bool = False):
        T, n = self.trials, self.prob.n
        res = (ResultC * T)()
        best = np.zeros((T, n), np.int8) if best_states else None
        tr = np.zeros((T, self.p.sc + 1, self.r)) if trace else None
        check(lib().ssqa_batch_fetch(
            self._b, res, best.ctypes.data_as(C.POINTER(C.c_int8)) if best is not None else None,
            _dp(tr) if tr is not None else None))
        return res, best, tr

    # GPU row shards (ssqa_batch_set_shard ... in include/ssqa_cuda.h)
    def set_shard(self, shard: int, nshards: int):
        check(lib().ssqa_batch_set_shard(self._b, shard, nshards))

    def shard_bytes(self) -> int:
        return int(lib().ssqa_batch_shard_bytes(self._b))

    def shard_begin(self, target: Optional[float] = None, stop_at_target: bool = True):
        check(lib().ssqa_batch_shard_begin(self._b, int(target is not None),
                                           0.0 if target is None else float(target),
                                           int(stop_at_target)))

    def shard_pass(self, chunk_ptr: int):
        check(lib().ssqa_batch_shard_pass(self._b, C.c_void_p(chunk_ptr)))

    def shard_merge(self, chunks_ptr: int):
        check(lib().ssqa_batch_shard_merge(self._b, C.c_void_p(chunks_ptr)))

    def shard_pass_to(self, dests: Sequence[int], flags: Sequence[int], epoch: int):
        """Peer push: pack this shard's chunk straight into every dests[d] and
        raise *flags[d] = epoch (ssqa_batch_shard_pass_to)."""
        n = len(dests)
        d = (C.c_void_p * n)(*[C.c_void_p(x) for x in dests])
        f = (C.c_void_p * n)(*[C.c_void_p(x) for x in flags])
        check(lib().ssqa_batch_shard_pass_to(self._b, d, f, n, C.c_uint(epoch & 0xFFFFFFFF)))

    def shard_direct_ok(self) -> bool:
        return bool(lib().ssqa_batch_shard_direct_ok(self._b))

    def sig4_ptr(self) -> int:
        out = C.c_void_p()
        check(lib().ssqa_batch_sig4(self._b, C.byref(out)))
        return int(out.value)

    def shard_pass_direct(self, peer_sig4: Sequence[int], peer_parts: Sequence[int],
                          flags: Sequence[int], epoch: int):
        """Shard pass with the exchange fused in (ssqa_batch_shard_pass_direct)."""
        n = len(peer_sig4)
        arr = lambda xs: (C.c_void_p * n)(*[C.c_void_p(x) for x in xs])
        check(lib().ssqa_batch_shard_pass_direct(self._b, arr(peer_sig4), arr(peer_parts),
                                                 arr(flags), n, C.c_uint(epoch & 0xFFFFFFFF)))

    def shard_merge_direct(self, parts_ptr: int, part_stride: int, flags_ptr: int, nflags: int,
                           epoch: int):
        check(lib().ssqa_batch_shard_merge_direct(self._b, C.c_void_p(parts_ptr), part_stride,
                                                  C.c_void_p(flags_ptr), nflags,
                                                  C.c_uint(epoch & 0xFFFFFFFF)))

    def shard_merge_from(self, chunks_ptr: int, flags_ptr: int, nflags: int, epoch: int):
        """Wait for every shard's flag to reach epoch, then merge."""
        check(lib().ssqa_batch_shard_merge_from(self._b, C.c_void_p(chunks_ptr),
                                                C.c_void_p(flags_ptr), nflags,
                                                C.c_uint(epoch & 0xFFFFFFFF)))

    def shard_end(self):
        check(lib().ssqa_batch_shard_end(self._b))

    # per-step API
    def init(self):
        check(lib().ssqa_batch_init(self._b))

    def sweep(self, count: int = 1):
        check(lib().ssqa_batch_sweep(self._b, count))

    def sweep_with(self, jperp: float, i0: float):
        check(lib().ssqa_batch_sweep_with(self._b, jperp, i0))

    def energies(self) -> np.ndarray:
        out = np.zeros((self.trials, self.r))
        check(lib().ssqa_batch_energies(self._b, _dp(out)))
        return out

    def read_lattice(self, trial: int):
        n, r, d = self.prob.n, self.r, self.delay
        sigma, acc, hist = np.zeros(n * r), np.zeros(n * r), np.zeros((d + 1) * n * r)
        cyc = C.c_long()
        check(lib().ssqa_batch_read_lattice(self._b, trial, _dp(sigma), _dp(acc), _dp(hist),
                                            C.byref(cyc)))
        return sigma, acc, hist.reshape(d + 1, n * r), cyc.value

    def write_lattice(self, trial: int, sigma, acc, hist, cycle: int):
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        a = np.ascontiguousarray(acc, dtype=np.float64)
        h = np.ascontiguousarray(hist, dtype=np.float64)
        check(lib().ssqa_batch_write_lattice(self._b, trial, _dp(s), _dp(a), _dp(h), cycle))

    def close(self):
        if self._b:
            lib().ssqa_batch_destroy(self._b)
            self._b = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _results(res, best, tr, trials, p=None) -> List[AnnealResult]:
    """p: the run's parameters; SsqaParams give the trace its jperp column
    (jperp_schedule of each recorded cycle), SSA traces carry jperp = 0."""
    out = []
    jp = None
    if tr is not None:
        ncyc = tr.shape[1]
        jp = (np.array([jperp_schedule(c, p) for c in range(ncyc)])
              if isinstance(p, SsqaParams) else np.zeros(ncyc))
    for t in range(trials):
        r = res[t]
        te = tj = np.zeros(0)
        if tr is not None:
            te = tr[t, : r.cycles_used + 1].reshape(-1).copy()
            tj = jp[: r.cycles_used + 1].copy()
        out.append(AnnealResult(r.best_energy, best[t].copy() if best is not None else None,
                                r.best_replica, bool(r.reached_target), r.first_hit_cycle,
                                r.cycles_used, te, r.wall_seconds, tj))
    return out


def ssqa_run_batch(m: IsingModel, p: SsqaParams, seeds: Sequence[int],
                   target_energy: Optional[float] = None, opts: RunOptions = RunOptions(),
                   engine: int = ENGINE_AUTO, device: int = 0,
                   problem: Optional[Problem] = None) -> List[AnnealResult]:
    """ssqa_run for every seed, as one device batch."""
    p.validate(m.n)
    prob = problem or Problem(m, device)
    b = Batch(prob, p, len(seeds), opts.record_trace, engine)
    try:
        b.set_seeds(seeds)
        b.launch(target_energy, opts.stop_at_target)
        res, best, tr = b.fetch(True, opts.record_trace)
        return _results(res, best, tr, len(seeds), p)
    finally:
        b.close()


def ssqa_run(m: IsingModel, p: SsqaParams, seed: int, target_energy: Optional[float] = None,
             opts: RunOptions = RunOptions(), engine: int = ENGINE_AUTO) -> AnnealResult:
    """annealer.cpp:474-487."""
    return ssqa_run_batch(m, p, [seed], target_energy, opts, engine)[0]


def ssa_run_batch(m: IsingModel, p: SsaParams, seeds: Sequence[int],
                  target_energy: Optional[float] = None, opts: RunOptions = RunOptions(),
                  engine: int = ENGINE_AUTO, device: int = 0,
                  problem: Optional[Problem] = None) -> List[AnnealResult]:
    """ssa_run for every seed, as one device batch."""
    p.validate(m.n)
    prob = problem or Problem(m, device)
    b = Batch(prob, p, len(seeds), opts.record_trace, engine)
    try:
        b.set_seeds(seeds)
        b.launch(target_energy, opts.stop_at_target)
        res, best, tr = b.fetch(True, opts.record_trace)
        return _results(res, best, tr, len(seeds), p)
    finally:
        b.close()


def ssa_run(m: IsingModel, p: SsaParams, seed: int, target_energy: Optional[float] = None,
            opts: RunOptions = RunOptions(), engine: int = ENGINE_AUTO) -> AnnealResult:
    """annealer.cpp:489-501."""
    return ssa_run_batch(m, p, [seed], target_energy, opts, engine)[0]


@dataclass
class ReplicaLattice:
    """ssqa::ReplicaLattice (annealer.hpp:68-81), layout [i*replicas + k]."""
    n: int
    replicas: int
    delay: int
    cycle: int
    sigma: np.ndarray
    is_acc: np.ndarray
    history: np.ndarray  # (delay+1, n*replicas)

    def spin(self, i, k):
        return self.sigma[i * self.replicas + k]

    def acc(self, i, k):
        return self.is_acc[i * self.replicas + k]

    def delayed_sigma(self):
        return self.history[self.cycle % (self.delay + 1)]


def init_lattice(n: int, replicas: int, delay: int, seed: int,
                 engine: int = ENGINE_AUTO) -> ReplicaLattice:
    """annealer.cpp:432-447, evaluated by the device init kernel."""
    prob = Problem.zero(n)
    p = SsqaParams(r=replicas, delay=delay, sc=1)
    b = Batch(prob, p, 1, engine=engine)
    b.set_seeds([seed])
    b.init()
    s, a, h, c = b.read_lattice(0)
    return ReplicaLattice(n, replicas, delay, c, s, a, h)


def ssqa_sweep(lat: ReplicaLattice, m: IsingModel, jperp: float, p: SsqaParams, seed: int,
               cycle: int, engine: int = ENGINE_AUTO) -> None:
    """annealer.cpp:449-463 (in place)."""
    if lat.n != m.n or lat.replicas != p.r:
        raise _lib.SsqaInvalidArgument(1, "lattice dimensions do not match model/params")
    if cycle != lat.cycle:
        raise _lib.SsqaInvalidArgument(1, "sweep cycle does not match lattice history")
    q = SsqaParams(**{**p.__dict__, "sc": max(1, p.sc)})
    b = Batch(Problem(m), q, 1, engine=engine)
    b.set_seeds([seed])
    b.write_lattice(0, lat.sigma, lat.is_acc, lat.history, lat.cycle)
    b.sweep_with(jperp, p.i0)
    s, a, h, c = b.read_lattice(0)
    lat.sigma[:], lat.is_acc[:], lat.history[...], lat.cycle = s, a, h, c


def replica_energies(lat: ReplicaLattice, m: IsingModel, engine: int = ENGINE_AUTO) -> np.ndarray:
    """annealer.cpp:465-472."""
    if lat.n != m.n:
        raise _lib.SsqaInvalidArgument(1, "lattice does not match model")
    p = SsqaParams(r=lat.replicas, delay=0, sc=1)
    b = Batch(Problem(m), p, 1, engine=engine)
    b.set_seeds([0])
    b.write_lattice(0, lat.sigma, np.zeros_like(lat.sigma), lat.sigma[None, :], 0)
    return b.energies()[0]


# ---- bench.hpp: trial batteries and time-to-solution -------------------------

@dataclass
class TtsValue:
    kind: str  # "finite" | "saturated" | "undefined"
    seconds: float = 0.0


def pool_stats(device: int = 0) -> dict:
    """Bytes the engine's device pool caches / hands out (csrc/devpool.h)."""
    c, u = C.c_longlong(0), C.c_longlong(0)
    lib().ssqa_pool_stats(device, C.byref(c), C.byref(u))
    return {"cached": int(c.value), "in_use": int(u.value)}


def pool_trim(device: int = -1) -> int:
    """Release the pool's cached device blocks; returns the bytes released."""
    return int(lib().ssqa_pool_trim(device))


def compute_tts(p_s: float, t_seconds: float, p_target: float = 0.99) -> TtsValue:
    """bench.cpp:144-160."""
    if not (0.0 < p_target < 1.0):
        raise ValueError("p_target must lie in (0, 1)")
    if not (0.0 <= p_s <= 1.0):
        raise ValueError("p_s outside [0, 1]")
    if t_seconds <= 0.0:
        raise ValueError("t must be > 0")
    if p_s == 0.0:
        return TtsValue("undefined")
    if p_s == 1.0:
        return TtsValue("saturated", 0.0)
    return TtsValue("finite", t_seconds * math.log(1.0 - p_target) / math.log(1.0 - p_s))


@dataclass
class TrialOutcome:
    seed: int
    reached_target: bool
    first_hit_cycle: int
    best_energy: float
    wall_seconds: float


def _mix64(x: int) -> int:
    """rng.hpp:10-15 on Python ints."""
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def trial_instance_seeds(base_seed: int, trials: int) -> List[int]:
    """CounterRng(base_seed, kStreamTrialInstance).raw(t) (rng.hpp:30-38),
    the GI instance seed of trial t in run_trials (bench.cpp:373, 389)."""
    key = _mix64(_mix64(base_seed) ^ ((1 << 32) + 7))
    return [_mix64((key + t * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)) for t in range(trials)]


@dataclass
class _Shape:
    n: int


def run_trials_fresh(n_nodes: int, p, trials: int, ec: int, base_seed: int,
                     edge_prob: float = 0.5, permute: bool = False, c1: float = 0.75,
                     c2: float = 0.75, p_target: float = 0.99, device: int = 0):
    """run_trials (bench.cpp:359-432) with a fresh GI instance per trial (the
    reference default, bench.hpp:28): instance t from seed
    CounterRng(base_seed, kStreamTrialInstance).raw(t), target 0, the whole
    battery as one multi-instance device batch."""
    seeds = [base_seed + t for t in range(trials)]
    # every trial's instance built on the device (no host model per trial)
    prob = Problem.generated_gi(n_nodes, trial_instance_seeds(base_seed, trials), edge_prob,
                                permute, c1, c2, device)
    shape = _Shape(n_nodes * n_nodes)  # the size is all the batch call needs
    try:
        if isinstance(p, SsaParams):
            q = SsaParams(**{**p.__dict__, "sc": ec})
            res = ssa_run_batch(shape, q, seeds, 0.0, RunOptions(False, False), problem=prob)
        else:
            q = SsqaParams(**{**p.__dict__, "sc": ec // p.r})
            res = ssqa_run_batch(shape, q, seeds, 0.0, RunOptions(False, False), problem=prob)
    finally:
        prob.close()
    outs = [TrialOutcome(s, r.reached_target, r.first_hit_cycle, r.best_energy, r.wall_seconds)
            for s, r in zip(seeds, res)]
    p_s = sum(o.reached_target for o in outs) / trials
    t_mean = sum(o.wall_seconds for o in outs) / trials
    return outs, p_s, t_mean, compute_tts(p_s, max(t_mean, 1e-12), p_target)


def run_trials(m: IsingModel, p, trials: int, ec: int, base_seed: int,
               target: float = 0.0, p_target: float = 0.99, engine: int = ENGINE_AUTO,
               device: int = 0):
    """run_trials (bench.cpp:359-432) on a pinned instance: fixed budget
    sc = ec / r (r = 1 for SsaParams, bench.cpp:362-363), seeds base_seed + t,
    stop_at_target = false."""
    seeds = [base_seed + t for t in range(trials)]
    if isinstance(p, SsaParams):
        q = SsaParams(**{**p.__dict__, "sc": ec})
        res = ssa_run_batch(m, q, seeds, target, RunOptions(False, False), engine, device)
    else:
        q = SsqaParams(**{**p.__dict__, "sc": ec // p.r})
        res = ssqa_run_batch(m, q, seeds, target, RunOptions(False, False), engine, device)
    outs = [TrialOutcome(s, r.reached_target, r.first_hit_cycle, r.best_energy, r.wall_seconds)
            for s, r in zip(seeds, res)]
    p_s = sum(o.reached_target for o in outs) / trials
    t_mean = sum(o.wall_seconds for o in outs) / trials
    return outs, p_s, t_mean, compute_tts(p_s, max(t_mean, 1e-12), p_target)


def tune(**overrides) -> None:
    """Engine overrides for parity tests and tuning (include/ssqa_tune.h):
    tune(tab=1), tune(fp4=0, rs=2), ...; tune() with no arguments resets all."""
    L = lib()
    if not overrides:
        L.ssqa_tune_reset()
        return
    for k, v in overrides.items():
        if k == "trace":
            L.ssqa_tune_trace(v.encode() if v else None)
        elif L.ssqa_tune_set(k.encode(), int(v)) != 0:
            raise ValueError(f"unknown tune key {k!r}")
