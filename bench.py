#!/usr/bin/env python3
"""SSQA replica-lattice benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
                    [--impl ours|reference] [--engine auto|simt|tcgen05]

A *step* is one full batched annealing run of the configured workload --
init_lattice + run_lattice for every trial, sc sweeps each -- i.e. one pass of
the hot path (annealer.cpp:313-361) over one batch, with the reference's
fixed-budget bench semantics (stop_at_target = false, bench.cpp:336).
Default workload is BASELINE config 3 (the metric's config): GI n=50 ->
N=2500 spins, M=20 replicas, 1024 trials, 5000 sweeps, 99 % TTS.

value : replica-spin updates/s = N*M*T*sc / step time, device-timed with CUDA
        events on the engine's stream, inputs resident in HBM, max over ranks.
e2e   : same metric through the public C-ABI call ssqa_run_batch with HOST
        buffers (quantize + upload of the model, seeds and schedule, the run,
        download of per-trial results and best states) inside the timed region.
roofline.traffic : DRAM bytes (read + write) of one launch of this workload,
        measured in the run by one ncu metric pass over a child process
        (scripts/prof_run.py), outside every timed region; null without ncu.
--impl reference : the reference's own C++ run_trials (oracle/_ref, built from
        /root/reference by oracle/Makefile) on the host cores, rank 0 only.

Multi-GPU (torchrun): trials are split into contiguous blocks, one per rank,
no data-path collective; total work fixed ("strong").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "replica-spin updates/sec at N=2500, M=20, batched trials; 99% time-to-solution"
UNIT = "replica-spin updates/s"

# BASELINE.json configs; sc in sweeps.
CONFIGS = {
    "c1": dict(kind="gi", n_nodes=10, R=20, T=100, sc=1000,
               desc="C1: GI n=10 -> N=100, M=20, 100 trials, 1000 sweeps"),
    "c2": dict(kind="gi", n_nodes=20, R=20, T=1024, sc=2000,
               desc="C2: GI n=20 -> N=400, M=20, 1024 trials, 2000 sweeps"),
    "c3": dict(kind="gi", n_nodes=50, R=20, T=1024, sc=5000,
               desc="C3: GI n=50 -> N=2500, M=20, 1024 trials, 5000 sweeps, TTS99"),
    "c4": dict(kind="dense", n=8192, dense_kind=0, R=32, T=256, sc=2000,
               desc="C4: dense int[-8,7] N=8192, M=32, 256 trials, 2000 sweeps"),
    "c5": dict(kind="dense", n=32768, dense_kind=1, R=16, T=64, sc=1000,
               desc="C5: SK +-1 N=32768, M=16, 64 trials, 1000 sweeps"),
}
GI_SEED, EDGE_P, C12, BASE_SEED = 7, 0.5, 1.0, 1000


def build_model(cfg):
    import paper_2302_12454_b200 as sq
    if cfg["kind"] == "gi":
        return sq.gi_ising(cfg["n_nodes"], EDGE_P, GI_SEED, True, C12, C12)
    return sq.dense_ising(cfg["n"], cfg["dense_kind"], GI_SEED)


def pin_model(m):
    """The e2e leg copies the model from PINNED host memory (the contract's
    host->device input copy): move h and J into page-locked buffers once,
    outside the timed region, so the per-call upload runs at DMA speed."""
    import torch
    m.pinned = False
    try:
        for name in ("h", "J"):
            a = np.ascontiguousarray(getattr(m, name), dtype=np.float64)
            t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
            t.numpy()[...] = a
            setattr(m, name, t.numpy())
            setattr(m, "_pinned_" + name, t)  # keeps the page-locked storage alive
        m.pinned = True
    except RuntimeError:  # no driver: pageable arrays stay
        pass
    return m


def n_spins(cfg):
    return cfg["n_nodes"] ** 2 if cfg["kind"] == "gi" else cfg["n"]


def config_of(cfg):
    """The `config` object of both arms (identical keys and values)."""
    N, R, T = n_spins(cfg), cfg["R"], cfg["T"]
    return {"workload": cfg["desc"], "n": N, "replicas": R, "trials": T, "sweeps": cfg["sc"],
            "l2": "no flush needed: per-step state (acc f64 "
                  f"{8 * N * R * T / 2**20:.0f} MiB + spins) exceeds L2"
                  if 8 * N * R * T > 126 * 2**20 else "state fits L2 (small config)"}


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs ~0.1-0.5 s to start: wait for its first sample so a
            # short timed region (C1: ~20 ms) still sits between samples
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.01)
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return None

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0])]
        smax = max([num(r[1]) for r in rows if num(r[1])] or [0])
        load = [s for s in sm if s >= 0.5 * smax] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max([num(r[2]) for r in rows if num(r[2])] or [0])}


def peaks():
    """(HBM GB/s, bf16 TF/s for the tensor roofline, label, bf16 burst TF/s).
    The fused sweep kernel is ONE launch of the whole job (0.5-1.2 s at the
    BASELINE configs): the measured SUSTAINED bf16 figure applies to a kernel
    timed inside a long step (MEASURED_PEAKS.json; the burst one is kept
    beside it).  HBM has a single measured copy bandwidth."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        burst = d.get("bf16_tflops", 1590.0)
        return (d.get("hbm_gbs", 6650.0), d.get("bf16_tflops_sustained", burst),
                "measured sustained", burst)
    return 6650.0, 1590.0, "fallback", 1590.0


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
def reference_sample(cfg, workers, target_s):
    """Time the reference's run_trials (oracle/_ref) on a bounded sample of
    the workload: `workers` trials (one per thread) x S sweeps, S calibrated
    so the sample takes about target_s seconds.  Per-sweep cost is
    data-independent, so updates/s extrapolates linearly."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py
    if not oracle_py.available("ref"):
        o = oracle_py.Oracle("orc")
        kind = "port"
    else:
        o = oracle_py.Oracle("ref")
        kind = "reference"
    R = cfg["R"]
    N = n_spins(cfg)
    if kind == "reference" and cfg["kind"] == "gi":
        h, J, off = o.gi_ising(cfg["n_nodes"], EDGE_P, GI_SEED, True, C12, C12)

        class _M:  # the reference's own instance
            pass
        m = _M()
        m.h, m.J, m.offset = h, J, off
    else:
        m = build_model(cfg)
    # calibrate single-thread cost per sweep
    p_cal = oracle_py.params(R, 4)
    t0 = time.perf_counter()
    o.ssqa_run(m.h, m.J, m.offset, p_cal, 1, None, False, False)
    per_sweep = max((time.perf_counter() - t0) / 5.0, 1e-6)
    S = int(max(4, min(cfg["sc"], target_s / per_sweep)))
    T = workers
    if kind == "reference" and cfg["kind"] == "gi":
        t_inst0 = time.perf_counter()
        o.gi_ising(cfg["n_nodes"], EDGE_P, GI_SEED, True, C12, C12)
        t_inst = time.perf_counter() - t_inst0
        t0 = time.perf_counter()
        o.run_trials(oracle_py.params(R, 1), n_nodes=cfg["n_nodes"], trials=T, ec=R * S,
                     base_seed=BASE_SEED, workers=workers, gi_seed=GI_SEED)
        wall = time.perf_counter() - t0 - t_inst
        sample = (f"reference run_trials: {T} trials x {S} sweeps on {workers} threads "
                  f"(of the {cfg['sc']}-sweep, {cfg['T']}-trial workload)")
    else:
        # dense configs (or no reference build): one ssqa_run per thread
        import concurrent.futures as cf
        p = oracle_py.params(R, S)
        t0 = time.perf_counter()
        if kind == "reference":
            # one shared reference model for all threads (a dense N=32768
            # IsingModel is 8.6 GB: one per call would not fit)
            t_m0 = time.perf_counter()
            o.ssqa_run_many(m.h, m.J, m.offset, oracle_py.params(R, 1), [BASE_SEED], 1)
            t_model = time.perf_counter() - t_m0  # model build + a 1-sweep run
            t0 = time.perf_counter()
            o.ssqa_run_many(m.h, m.J, m.offset, p, [BASE_SEED + s for s in range(T)], workers)
            wall = time.perf_counter() - t0 - t_model
        else:
            with cf.ThreadPoolExecutor(workers) as ex:
                list(ex.map(lambda s: o.ssqa_run(m.h, m.J, m.offset, p, BASE_SEED + s, None,
                                                 False, False), range(T)))
            wall = time.perf_counter() - t0
        sample = (f"{kind} ssqa_run: {T} trials x {S} sweeps on {workers} threads")
    upd = float(N) * R * T * S
    return dict(value=upd / wall, unit=UNIT, cores=workers, kind=kind, sample=sample,
                cpu=cpu_model(), seconds=wall)


def reference_full_sc(cfg, workers, trials=16):
    """the reference's run_trials on `trials` trials at the
    config's FULL sweep count (p_s and TTS99 with the reference's own
    formula, bench.cpp:414-430), one trial per host thread."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py
    kind = "reference" if oracle_py.available("ref") else "port"
    if kind != "reference" or cfg["kind"] != "gi":
        return None
    o = oracle_py.Oracle("ref")
    R, sc, N = cfg["R"], cfg["sc"], n_spins(cfg)
    w = max(1, min(workers, trials))
    t0 = time.perf_counter()
    outs, ps, t_mean, (tts_s, tts_kind) = o.run_trials(
        oracle_py.params(R, 1), n_nodes=cfg["n_nodes"], trials=trials, ec=R * sc,
        base_seed=BASE_SEED, workers=w, gi_seed=GI_SEED)
    wall = time.perf_counter() - t0
    hits = sum(1 for x in outs if x["reached_target"])
    import math
    amort = (wall / trials) * math.log(0.01) / math.log(1.0 - ps) if 0.0 < ps < 1.0 else None
    return {"trials": trials, "sweeps": sc, "threads": w, "seconds": wall,
            "value": float(N) * R * trials * sc / wall, "unit": UNIT, "p_s": ps, "hits": hits,
            "t_mean_trial_s": t_mean,
            "tts99_ref_formula_s": tts_s if tts_kind == 0 else None,
            "tts99_amortised_s": amort,
            "sample": f"reference run_trials: {trials} trials x {sc} sweeps (full budget) on "
                      f"{w} threads, seeds {BASE_SEED}+t"}


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    workers = os.cpu_count() or 1
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    for i in range(args.warmup + args.steps):
        s = reference_sample(cfg, workers, per_step)
        if i >= args.warmup:
            vals.append(s)
    v = statistics.median(x["value"] for x in vals)
    last = vals[-1]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    full = None
    if world == 1 and not args.no_full_sc:
        try:
            full = reference_full_sc(cfg, workers)
        except Exception as e:  # reported, never fatal
            full = {"error": str(e)}
    N = n_spins(cfg)
    ms = 1e3 * float(N) * cfg["R"] * cfg["T"] * cfg["sc"] / v
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference GI generator, instance seed 7)",
        "config": config_of(cfg),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"] + "; ms_per_step extrapolated to the full "
                         "workload", "cpu": last["cpu"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "full_sc_sample": full,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_rows(args, cfg):
    """--shard rows: J' row-sharded across the GPUs (the
    C4/C5 layout): every rank runs all trials on its spin rows, one in-place
    NCCL all-gather of bit-packed spin rows + energy partials per cycle."""
    import torch

    import paper_2302_12454_b200 as sq
    from paper_2302_12454_b200 import _lib, shard
    from paper_2302_12454_b200.rowshard import (ExchangeRegion, P2PLayout, _ipc_handle,
                                                _map_peers, run_row_sharded, shard_cycles,
                                                shard_cycles_direct, shard_cycles_p2p)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    R, T, sc = cfg["R"], cfg["T"], cfg["sc"]
    N = n_spins(cfg)
    seeds = [BASE_SEED + t for t in range(T)]
    m = pin_model(build_model(cfg))
    p = sq.SsqaParams(r=R, sc=sc)
    target = 0.0 if cfg["kind"] == "gi" else None
    prob = sq.Problem(m, local)
    b = sq.Batch(prob, p, T, False, _lib.ENGINE_TCGEN05)
    b.set_shard(rank, world)
    b.set_seeds(seeds)
    buf = torch.empty(world * b.shard_bytes(), dtype=torch.uint8, device=f"cuda:{local}")
    stream = torch.cuda.ExternalStream(b.stream, device=f"cuda:{local}")
    p2p = args.exchange in ("p2p", "direct")
    direct = args.exchange == "direct"
    if p2p:  # exchange regions mapped across the ranks (CUDA IPC), peer push
        layout = P2PLayout(world, b.shard_bytes())
        region = ExchangeRegion(layout.total, local)
        opened = []
        bases = _map_peers(region.base, region.handle(), local, None, world, rank, opened)
        if direct:
            sig4 = _map_peers(b.sig4_ptr(), _ipc_handle(b.sig4_ptr()), local, None, world, rank,
                              opened)
        if dist:
            dist.barrier()
        epoch = [0]

    def all_gather(out, mine):
        with torch.cuda.stream(stream):
            dist.all_gather_into_tensor(out, mine)

    graph = None

    def step():
        if graph is not None:
            graph.replay_on_engine()
            return b.elapsed_ms()
        b.shard_begin(target, False)
        if p2p:
            # every rank's previous step (its last merge reads the slots peers
            # push into) and this step's repack are done before any pass 0
            b.synchronize()
            if dist:
                dist.barrier()
        if direct:
            epoch[0] = shard_cycles_direct(b, layout, rank, bases, sig4, sc + 1, epoch[0])
        elif p2p:
            epoch[0] = shard_cycles_p2p(b, layout, rank, bases, sc + 1, epoch[0])
        else:
            shard_cycles(b, buf, rank, world, sc + 1, all_gather)
        b.shard_end()
        return b.elapsed_ms()

    for _ in range(args.warmup):
        step()
    if args.graph and not p2p:
        # the whole run (begin, sc+1 x (pass, all-gather, merge), end) as one
        # CUDA graph: one host launch per step (rowshard.capture_run)
        from paper_2302_12454_b200.rowshard import capture_run
        graph = capture_run(b, buf, rank, world, sc + 1, all_gather, stream, target, False)
        step()
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    times, launches = [], 0
    for _ in range(args.steps):
        barrier()
        times.append(step())
        launches += b.launch_count()
    barrier()
    clk = clocks.stop()
    step_ms = shard.max_over_ranks(statistics.mean(times), dist, "cuda")
    value = float(N) * R * T * sc / (step_ms * 1e-3)
    hbm_peak, bf16_peak, peak_kind, bf16_burst = peaks()
    tc_peak = 2.0 * bf16_peak
    ops_rank = 2.0 * N * (N / world) * R * T * (sc + 1)
    tensor_tops = ops_rank / (statistics.mean(times) * 1e-3) / 1e12
    # e2e: the public driver from host arrays (problem upload included)
    e2e_times = []
    for i in range(max(1, args.steps)):
        barrier()
        t0 = time.perf_counter()
        run_row_sharded(m, p, seeds, target, sq.RunOptions(False, False), local,
                        exchange=args.exchange)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = shard.max_over_ranks(statistics.mean(e2e_times), dist, "cuda")
    # the model's double couplings (quantized on the device) + H' + seeds + schedule
    h2d = 8 * N * N + 4 * prob.info()["n_pad"] + 8 * T + 8 * (sc + 1)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": ("fp4" if b.operand_bits == 4 else "int8") + " contraction + f64 update",
            "data": "synthetic (seeded dense instance generator, seed 7)",
            "config": {"workload": cfg["desc"], "n": N, "replicas": R, "trials": T,
                       "sweeps": sc, "engine": "tcgen05 row shards",
                       "parallelism": f"J rows x{world} (" + {
                           "nccl": "NCCL all-gather", "p2p": "pack kernel pushes to peers",
                           "direct": "exchange fused into the sweep kernel's stores"}[
                           args.exchange] + " per cycle"
                           + (", whole run as one CUDA graph" if graph is not None else "") + ")",
                       "l2": "no flush needed: per-step state exceeds L2"},
            "roofline": {"bound": "tensor", "achieved": tensor_tops, "peak": tc_peak,
                         "unit": "TOPS", "frac": tensor_tops / tc_peak, "traffic": None,
                         "kernel": "k_sweep_tc (one pass per cycle, own rows)",
                         "operands": "int8-equivalent ops (the passes stream the problem's "
                                     f"{b.operand_bits}-bit operand image)",
                         "peak_note": f"int8 dense = 2 x {peak_kind} bf16 ({bf16_peak} TF/s)"},
            "e2e": {"value": float(N) * R * T * sc / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(T * (N + 40)),
                    "seconds_per_step": e2e_s},
            "gpu_launches": launches // max(1, args.steps),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()  # no peer still pushes into this rank's region
    if p2p:
        for ptr in opened:
            _lib.lib().ssqa_ipc_close(ptr)
        region.close()
    b.close()
    prob.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def time_dense_config(name, steps=2, warmup=1):
    """Device-timed run of a dense BASELINE config (C4 / C5) for the extra keys
    of the headline line: the problem is built on the device
    (ssqa_problem_create_dense), all trials x all sweeps per step."""
    import torch

    import paper_2302_12454_b200 as sq
    from paper_2302_12454_b200 import _lib
    cfg = CONFIGS[name]
    N, R, T, sc = cfg["n"], cfg["R"], cfg["T"], cfg["sc"]
    prob = sq.Problem.generated_dense(N, cfg["dense_kind"], GI_SEED)
    info = prob.info()
    b = sq.Batch(prob, sq.SsqaParams(r=R, sc=sc), T, False, _lib.ENGINE_TCGEN05)
    b.set_seeds([BASE_SEED + t for t in range(T)])
    for _ in range(warmup):
        b.launch(None, False)
        b.elapsed_ms()
    clocks = ClockSampler(0)
    torch.cuda.synchronize()
    clocks.start()
    times = []
    for _ in range(steps):
        b.launch(None, False)
        times.append(b.elapsed_ms())
    clk = clocks.stop()
    ms = statistics.mean(times)
    _, bf16_peak, peak_kind, bf16_burst = peaks()
    op_bits = b.operand_bits
    planes = 2 if (op_bits == 4 and info.get("fp4") == 2) else 1
    tc_mult = 4.0 if op_bits == 4 else 2.0
    ops = 2.0 * N * N * R * T * (sc + 1) * planes
    i8 = 2.0 * N * N * R * T * (sc + 1)
    out = {"workload": cfg["desc"], "ms_per_step": ms, "steps": steps, "warmup": warmup,
           "value": float(N) * R * T * sc / (ms * 1e-3), "unit": UNIT,
           "tensor": {"achieved_tops": ops / (ms * 1e-3) / 1e12,
                      "peak_tops": tc_mult * bf16_peak,
                      "frac": ops / (ms * 1e-3) / 1e12 / (tc_mult * bf16_peak),
                      "operands": ("fp4 pair" if planes == 2 else "fp4") if op_bits == 4 else "int8"},
           "int8_equiv": {"achieved_tops": i8 / (ms * 1e-3) / 1e12, "peak_tops": 2.0 * bf16_peak,
                          "frac": i8 / (ms * 1e-3) / 1e12 / (2.0 * bf16_peak)},
           "tensor_frac_vs_burst_peak": ops / (ms * 1e-3) / 1e12 / (tc_mult * bf16_burst),
           "peak_note": f"{peak_kind} bf16 x {tc_mult:g} (operand format) / x 2 (int8)",
           "clocks": clk, "gpu_launches": b.launch_count()}
    b.close()
    prob.close()
    return out


def run_ours(args, cfg):
    import numpy as np
    import torch

    import paper_2302_12454_b200 as sq
    from paper_2302_12454_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    from paper_2302_12454_b200 import shard

    def max_over_ranks(x: float) -> float:
        return shard.max_over_ranks(x, dist, "cuda")

    R, T, sc = cfg["R"], cfg["T"], cfg["sc"]
    N = n_spins(cfg)
    # contiguous trial blocks per rank, seeds base + global trial index
    seeds = shard.shard_seeds(BASE_SEED, T, world, rank)
    engine = {"auto": _lib.ENGINE_AUTO, "simt": _lib.ENGINE_SIMT,
              "tcgen05": _lib.ENGINE_TCGEN05}[args.engine]
    m = pin_model(build_model(cfg))
    p = sq.SsqaParams(r=R, sc=sc)
    prob = sq.Problem(m, local)
    info = prob.info()
    b = sq.Batch(prob, p, len(seeds), False, engine)
    b.set_seeds(seeds)
    eng_name = _lib.ENGINE_NAMES.get(b.engine, str(b.engine))

    # ---- device-resident timing (value) ----
    for _ in range(args.warmup):
        b.launch(0.0 if cfg["kind"] == "gi" else None, False)
        b.elapsed_ms()
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    times, launches = [], 0
    for _ in range(args.steps):
        barrier()
        b.launch(0.0 if cfg["kind"] == "gi" else None, False)
        times.append(b.elapsed_ms())
        launches += b.launch_count()
    barrier()
    clk = clocks.stop()
    res, best, _ = b.fetch(True, False)
    reached = [bool(res[t].reached_target) for t in range(len(seeds))]
    step_ms = max_over_ranks(statistics.mean(times))
    upd_per_step = float(N) * R * T * sc
    value = upd_per_step / (step_ms * 1e-3)

    # ---- dominant kernel, live CUDA-event timing on the engine's stream ----
    # Roofline: per replica-spin update the path needs 2N
    # int8 ops (tensor bound) and 16 B of accumulator state (f64 read+write)
    # + 0.25 B of packed spins + N/(M*T) B of J streamed once per sweep
    # (HBM bound); the binding one is reported, the other kept beside it.
    hbm_peak, bf16_peak, peak_kind, bf16_burst = peaks()
    # dense tensor peak of the operand format the kernel streams: int8 = 2x
    # bf16, FP4 (kind::mxf4) = 4x bf16 on B200
    op_bits = b.operand_bits
    # FP4 pair operands (J' = A1 + A2, problem info fp4 == 2): two kind::mxf4
    # MMAs per coupling block, i.e. twice the FP4 ops of a single image
    planes = 2 if (op_bits == 4 and info.get("fp4") == 2) else 1
    tc_mult = 4.0 if op_bits == 4 else 2.0
    tc_peak = tc_mult * bf16_peak
    tc_name = ("fp4 pair (e2m1, J'=A1+A2)" if planes == 2 else "fp4 (e2m1)") if op_bits == 4 \
        else "int8"
    cols = R * len(seeds)
    # algorithmic bytes (format independent): f64 acc
    # read+write, bit-packed spins, int8 J streamed once per sweep
    alg_bytes_per_update = 16.0 + 0.25 + float(N) / float(R * T)
    updates_per_sweep = float(N) * cols
    if b.engine == _lib.ENGINE_SIMT:
        kname = "k_field_simt"
        k_ms = b.profile_field(10)
        ops = 2.0 * N * N * cols
        launch_bytes = None
        sweeps_per_launch = 1
    else:
        kname = "k_sweep_tc (fused, persistent: whole run in one launch)"
        k_ms = statistics.mean(times)
        ops = 2.0 * N * N * cols * (sc + 1) * planes
        sweeps_per_launch = sc
        launch_bytes = alg_bytes_per_update * updates_per_sweep * sc
    tensor_tops = ops / (k_ms * 1e-3) / 1e12
    # DRAM bytes of one launch: measured in this run, outside every timed
    # region, by one ncu metric pass over a separate process that runs this
    # workload's launch (scripts/prof_run.py); null where ncu is unavailable
    traffic = None
    traffic_note = "not measured (--no-traffic, N > 1, SIMT engine or no ncu)"
    if (rank == 0 and world == 1 and b.engine != _lib.ENGINE_SIMT and not args.no_traffic):
        traffic, traffic_note = measure_traffic(args.config, sc)
    tensor = {"achieved": tensor_tops, "peak": tc_peak, "unit": "TOPS",
              "frac": tensor_tops / tc_peak, "operands": tc_name,
              "frac_vs_burst_peak": tensor_tops / (tc_mult * bf16_burst)}
    # BASELINE.json's target is phrased against the int8 tensor roofline: the
    # algorithmic 2N ops per update (one coupling plane) at the int8 dense peak
    # (2 x bf16), whatever operand format the kernel streams
    i8_tops = 2.0 * N * N * cols * (sc + 1) / (k_ms * 1e-3) / 1e12 if b.engine != _lib.ENGINE_SIMT \
        else tensor_tops
    tensor["int8_equiv"] = {"achieved": i8_tops, "peak": 2.0 * bf16_peak, "unit": "TOPS",
                            "frac": i8_tops / (2.0 * bf16_peak)}
    peak_note = (f"{peak_kind} HBM copy bandwidth (MEASURED_PEAKS.json); {tc_name} dense = "
                 f"{tc_mult:g} x {peak_kind} bf16 ({bf16_peak} TF/s)")
    if launch_bytes is not None:
        achieved = launch_bytes / (k_ms * 1e-3) / 1e9
        hbm = {"achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak}
        # report the binding roofline (the larger fraction), the other beside it
        if hbm["frac"] >= tensor["frac"]:
            roofline = {"bound": "hbm", **hbm, "traffic": traffic, "traffic_note": traffic_note,
                        "kernel": kname, "kernel_ms": k_ms,
                        "alg_bytes_per_update": alg_bytes_per_update,
                        "tensor": tensor, "peak_note": peak_note}
        else:
            roofline = {"bound": "tensor", **{k: tensor[k] for k in ("achieved", "peak", "unit",
                                                                      "frac")},
                        "traffic": traffic, "traffic_note": traffic_note, "kernel": kname,
                        "kernel_ms": k_ms,
                        "operands": tc_name, "alg_bytes_per_update": alg_bytes_per_update,
                        "int8_equiv": tensor["int8_equiv"], "hbm": hbm, "peak_note": peak_note}
    else:
        roofline = {"bound": "tensor", **{k: tensor[k] for k in ("achieved", "peak", "unit",
                                                                  "frac")},
                    "traffic": traffic, "traffic_note": traffic_note, "kernel": kname,
                    "kernel_ms": k_ms,
                    "operands": tc_name, "peak_note": peak_note, "int8_equiv": tensor["int8_equiv"]}

    # ---- e2e through the public C-ABI call with host buffers ----
    e2e_times = []
    for i in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        out = sq.ssqa_run_batch(m, p, seeds, 0.0 if cfg["kind"] == "gi" else None,
                                sq.RunOptions(False, False), engine, local)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_times.append(dt)
        if i == 0:
            assert [o.best_energy for o in out] == [res[t].best_energy for t in range(len(seeds))]
    e2e_s = max_over_ranks(statistics.mean(e2e_times))
    npad = info["n_pad"]
    # the model's double couplings (quantized on the device) + int32 H' + seeds +
    # the jperp schedule table
    h2d = 8 * N * N + 4 * npad + 8 * len(seeds) + 8 * (sc + 1)
    d2h = len(seeds) * (8 + 4 + 4 + 8 + 8 + 8) + len(seeds) * N

    # ---- TTS99 (amortised and reference-formula) ----
    hits = shard.sum_over_ranks(sum(reached), dist, "cuda")
    p_s = hits / T
    t_trial = step_ms * 1e-3 / T * world  # device time per trial on one GPU
    tts = sq.compute_tts(p_s, t_trial) if cfg["kind"] == "gi" else None
    # the reference's formula (bench.cpp:424-430) with t = a trial's own wall
    # time: every trial of the batch runs for the whole batch
    tts_ref = sq.compute_tts(p_s, step_ms * 1e-3) if cfg["kind"] == "gi" else None

    others = None
    if world == 1 and args.config == "c3" and not args.no_other_configs:
        others = {}
        for name in ("c4", "c5"):
            try:
                others[name] = time_dense_config(name)
            except Exception as e:  # reported, never fatal to the headline number
                others[name] = {"error": str(e)}
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = reference_sample(cfg, os.cpu_count() or 1, args.cpu_seconds)
            except Exception as e:  # reported, never fatal to the GPU number
                cpu = {"error": str(e)}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": (f"{tc_name} contraction (exact f32 acc)" if op_bits == 4 else
                      "int8 contraction (int32 acc)") + " + f64 update",
            "data": "synthetic (reference GI generator, instance seed 7; seeds 1000+t)"
                    if cfg["kind"] == "gi" else "synthetic (CounterRng stream 8/9, seed 7)",
            "config": config_of(cfg),
            "engine_config": {"n_pad": npad, "engine": eng_name,
                              "parallelism": f"trial-sharded x{world}",
                              "operands": tc_name},
            "roofline": roofline,
            "e2e": {"value": upd_per_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "seconds_per_step": e2e_s,
                    "h2d_source": "pinned" if m.pinned else "pageable"},
            "gpu_launches": launches,
            "clocks": clk,
            "tts": {"p_s": p_s, "hits": hits, "trials": T, "t_trial_s": t_trial,
                    "tts99_s": None if tts is None else
                    (tts.seconds if tts.kind == "finite" else tts.kind),
                    "definition": "amortised: batch device time / trials per GPU",
                    "tts99_ref_formula_s": None if tts_ref is None else
                    (tts_ref.seconds if tts_ref.kind == "finite" else tts_ref.kind),
                    "ref_formula": "bench.cpp:424-430 with t = per-trial wall = the batch's "
                                   "device time (all trials run concurrently)"},
            "cpu_baseline": cpu,
            "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    b.close()
    prob.close()
    if dist:
        dist.destroy_process_group()
    return 0


def cfg_name(args):
    return args.config


def measure_traffic(config: str, sc: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of ONE launch of the fused
    kernel on this config's workload: `ncu --metrics ... --clock-control none`
    over a child process (scripts/prof_run.py: two launches, the second one
    captured).  Nothing here is timed or reported as throughput.  Returns
    (bytes or None, note)."""
    import csv as _csv
    import shutil
    import subprocess
    import tempfile
    # never nest profilers: when this process already runs under one (the
    # launch-list pass runs bench.py under ncu), injection variables are set
    if any(k in os.environ for k in ("CUDA_INJECTION64_PATH", "CUDA_INJECTION32_PATH",
                                     "NV_COMPUTE_PROFILER_PERFWORKS_DIR", "NVTX_INJECTION64_PATH")):
        return None, "not measured: this run is itself under a profiler"
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu"
                                  if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    script = os.path.join(ROOT, "scripts", "prof_run.py")
    if not ncu or not os.path.exists(script):
        return None, "not measured: ncu or scripts/prof_run.py not found"
    try:
        with tempfile.TemporaryDirectory() as td:
            log = os.path.join(td, "t.csv")
            cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum",
                   "--clock-control", "none", "-k", "regex:k_sweep", "-s", "1", "-c", "1", "--csv",
                   "--log-file", log, sys.executable, script, config, "tcgen05", str(sc)]
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
            if r.returncode != 0 or not os.path.exists(log):
                return None, f"not measured: ncu exited {r.returncode}"
            tot = 0.0
            seen = 0
            for row in _csv.reader(open(log)):
                if len(row) > 3 and row[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v = float(row[-1].replace(",", ""))
                    unit = row[-2].lower()
                    scale = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}
                    tot += v * scale.get(unit, 1.0)
                    seen += 1
            if seen != 2:
                return None, "not measured: ncu log without the DRAM metrics"
            return tot, ("dram__bytes_read.sum + dram__bytes_write.sum of one launch (this "
                         "workload, separate process under ncu --clock-control none, in this run, "
                         "outside the timed regions)")
    except Exception as e:  # noqa: BLE001 -- the bench line must not depend on the profiler
        return None, f"not measured: {type(e).__name__}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--engine", default="auto", choices=["auto", "simt", "tcgen05"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-sc", action="store_true",
                    help="reference arm: skip the 16-trial full-budget run (p_s, TTS99)")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the ncu metric pass that measures roofline.traffic")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the device-timed C4/C5 lines added to the C3 line")
    ap.add_argument("--shard", default="trials", choices=["trials", "rows"],
                    help="multi-GPU layout: trial blocks per GPU (default) or J' rows per GPU")
    ap.add_argument("--graph", action="store_true",
                    help="--shard rows, nccl: capture each run as one CUDA graph")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p", "direct"],
                    help="--shard rows: NCCL all-gather, pack-kernel peer push, or the push "
                         "fused into the sweep kernel (CUDA IPC peer memory over NVLink)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    if args.shard == "rows":
        return run_rows(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
