"""Time the C3 per-rank trial blocks (G = 2/4/8 -> 512/256/128 trials) under
forced column-tile widths and row splits (tune keys "wide", "rs"):
    python scripts/geom_sweep.py [sweeps]
Prints ms per run; used to calibrate make_geom's choice for small batteries."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2302_12454_b200 as sq
from paper_2302_12454_b200 import _lib

sc = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
cfg = bench.CONFIGS["c3"]
prob = sq.Problem.generated_gi(cfg["n_nodes"], [bench.GI_SEED], bench.EDGE_P, True, bench.C12, bench.C12)
CASES = {128: [(0, 0), (12, 12), (12, 13), (11, 12), (10, 10), (10, 11), (8, 9), (7, 7), (6, 6), (5, 5), (4, 4)],
         256: [(0, 0), (12, 6), (11, 6), (10, 5), (9, 5), (8, 4), (7, 4), (6, 3), (5, 2), (2, 1)],
         512: [(0, 0), (12, 3), (10, 2), (8, 2), (7, 2), (4, 1)]}
CTA2 = int(os.environ.get("GEOM_CTA2", "-1"))
if os.environ.get("GEOM_DEFAULT_ONLY"):
    CASES = {T: [(0, 0)] for T in (64, 128, 256, 384, 512, 768, 1024)}
for T, combos in CASES.items():
    for wide, rs in combos:
        sq.tune()
        if wide:
            sq.tune(wide=wide, rs=rs)
            if CTA2 >= 0:
                sq.tune(cta2=CTA2)
        try:
            b = sq.Batch(prob, sq.SsqaParams(r=cfg["R"], sc=sc), T, False, _lib.ENGINE_TCGEN05)
            b.set_seeds([1000 + t for t in range(T)])
            ms = []
            for _ in range(3):
                b.launch(None, False)
                ms.append(b.elapsed_ms())
            b.close()
            print(f"T={T:4d} wide={wide:2d} rs={rs:2d}: {min(ms[1:]):8.2f} ms  ({min(ms[1:]) / (sc + 1) * 1e3:6.1f} us/sweep)", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"T={T:4d} wide={wide:2d} rs={rs:2d}: failed {str(e)[:80]}", flush=True)
sq.tune()
