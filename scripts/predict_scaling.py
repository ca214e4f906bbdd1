"""Predicted multi-GPU scaling from per-rank shapes timed on ONE GPU.

The pool this repo is developed on has one B200, so the 2/4/8-GPU runs of
bench.py cannot be measured here.  What each rank would run can: this script
times, on one GPU,

* trial sharding (C1-C3, bench.py default under torchrun): the contiguous block
  of T/G trials rank 0 anneals (full sweep budget, no data-path collective) --
  the step time of G GPUs is the max over ranks, i.e. this block's time;
* J' row sharding (C4 / C5, bench.py --shard rows): one cycle of rank 0 of G
  shards -- a pass over npad/G rows (all trials) plus the merge of G chunks --
  times the cycle count, plus a model of the per-cycle all-gather of the
  bit-packed spin rows and energy partials over NVLink (bytes x (G-1)/G at
  PEER_BW, plus COLL_US of launch/latency per collective);
* and, for C4, trial sharding as the comparison SURVEY.md 8.1(e) names.

    python scripts/predict_scaling.py [--out profiles/r02/scaling_prediction.json]

Writes the JSON and prints a markdown table.  Predictions, not measurements.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2302_12454_b200 as sq  # noqa: E402
from paper_2302_12454_b200 import _lib, shard  # noqa: E402

PEER_BW = 700e9   # B/s per direction, NVLink 5 peer (B300 microarch notes: 723-775)
COLL_US = 12.0    # per all-gather: launch + NVSwitch latency (NCCL small messages)


def problem(cfg):
    if cfg["kind"] == "gi":
        return sq.Problem.generated_gi(cfg["n_nodes"], [bench.GI_SEED], bench.EDGE_P, True,
                                       bench.C12, bench.C12)
    return sq.Problem.generated_dense(cfg["n"], cfg["dense_kind"], bench.GI_SEED)


def time_trials(prob, cfg, trials, sc, reps=2):
    seeds = [bench.BASE_SEED + t for t in range(trials)]
    b = sq.Batch(prob, sq.SsqaParams(r=cfg["R"], sc=sc), trials, False, _lib.ENGINE_TCGEN05)
    b.set_seeds(seeds)
    b.launch(None, False)
    b.elapsed_ms()
    ms = []
    for _ in range(reps):
        b.launch(None, False)
        ms.append(b.elapsed_ms())
    b.close()
    return min(ms) * 1e-3


def time_row_shard(prob, cfg, G, cycles):
    """Rank 0 of G shards on this GPU: per-cycle pass (npad/G rows) + merge."""
    import torch
    T = cfg["T"]
    b = sq.Batch(prob, sq.SsqaParams(r=cfg["R"], sc=cycles), T, False, _lib.ENGINE_TCGEN05)
    b.set_shard(0, G)
    b.set_seeds([bench.BASE_SEED + t for t in range(T)])
    nb = b.shard_bytes()
    buf = torch.zeros(G * nb, dtype=torch.uint8, device="cuda:0")
    b.shard_begin(None, False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    from paper_2302_12454_b200.rowshard import shard_cycles
    shard_cycles(b, buf, 0, 1, cycles, None)  # no all-gather (one process)
    b.synchronize()
    dt = (time.perf_counter() - t0) / cycles
    b.shard_end()
    b.close()
    return dt, nb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02",
                                                  "scaling_prediction.json"))
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    args = ap.parse_args()
    rows = []
    for name in args.configs.split(","):
        cfg = bench.CONFIGS[name]
        N = bench.n_spins(cfg)
        R, T, sc = cfg["R"], cfg["T"], cfg["sc"]
        upd = float(N) * R * T * sc
        prob = problem(cfg)
        t1 = None
        for G in (1, 2, 4, 8):
            lo, hi = shard.shard_trials(T, G, 0)
            ts = time_trials(prob, cfg, hi - lo, sc)
            t1 = ts if G == 1 else t1
            rows.append({"config": name, "layout": "trials", "gpus": G, "step_s": ts,
                         "value": upd / ts, "efficiency": (t1 / ts) / G})
        if cfg["kind"] == "dense":
            cyc = 6
            for G in (1, 2, 4, 8):
                dt, nb = time_row_shard(prob, cfg, G, cyc)
                coll = 0.0 if G == 1 else (nb * G * (G - 1) / G) / PEER_BW + COLL_US * 1e-6
                step = (sc + 1) * (dt + coll)
                rows.append({"config": name, "layout": "rows (model: all-gather)", "gpus": G,
                             "step_s": step, "value": upd / step,
                             "cycle_compute_us": dt * 1e6, "cycle_allgather_us": coll * 1e6,
                             "chunk_bytes": nb})
            base = [r for r in rows if r["config"] == name and r["layout"].startswith("rows")]
            for r in base:
                r["efficiency"] = (base[0]["step_s"] / r["step_s"]) / r["gpus"]
        prob.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"note": __doc__.split("\n\n")[0], "peer_bw": PEER_BW, "coll_us": COLL_US,
                   "rows": rows}, f, indent=1)
    print("| config | layout | GPUs | step (s) | upd/s (whole job) | efficiency |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['config']} | {r['layout']} | {r['gpus']} | {r['step_s']:.4f} | "
              f"{r['value']:.3e} | {r['efficiency']:.2f} |")


if __name__ == "__main__":
    main()
