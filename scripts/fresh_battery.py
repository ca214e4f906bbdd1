"""Time a fresh-instance GI battery (the reference's default run_trials:
one new instance per trial, bench.hpp:28) built on the device:
    python scripts/fresh_battery.py [n_nodes] [trials] [sweeps]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2302_12454_b200 as sq

nn = int(sys.argv[1]) if len(sys.argv) > 1 else 50
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
sc = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
for rep in range(2):
    t0 = time.perf_counter()
    outs, p_s, t_mean, tts = sq.run_trials_fresh(nn, sq.SsqaParams(r=20), T, 20 * sc, 1000,
                                                 permute=True, c1=1.0, c2=1.0)
    dt = time.perf_counter() - t0
    upd = nn * nn * 20 * T * sc
    print(f"n={nn} T={T} sc={sc}: {dt:.3f} s end to end, {upd / dt:.3e} upd/s, device "
          f"{t_mean * T:.3f} s ({upd / (t_mean * T):.3e} upd/s), p_s {p_s:.3f}", flush=True)
