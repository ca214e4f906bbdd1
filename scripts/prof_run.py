"""One short batched run for profiling: python scripts/prof_run.py c3 tcgen05 20"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2302_12454_b200 as sq
from paper_2302_12454_b200 import _lib
# dev tooling: SSQA_TC_<KEY>=v environment variables map onto engine overrides
for k, v in os.environ.items():
    if k.startswith("SSQA_TC_"):
        key = k[len("SSQA_TC_"):].lower()
        sq.tune(**{key: v if key == "trace" else int(v)})
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
eng = {"simt": _lib.ENGINE_SIMT, "tcgen05": _lib.ENGINE_TCGEN05}[sys.argv[2] if len(sys.argv) > 2 else "tcgen05"]
sc = int(sys.argv[3]) if len(sys.argv) > 3 else 20
m = bench.build_model(cfg)
p = sq.SsqaParams(r=cfg["R"], sc=sc)
prob = sq.Problem(m)
b = sq.Batch(prob, p, cfg["T"], False, eng)
b.set_seeds([1000 + t for t in range(cfg["T"])])
for _ in range(2):
    b.launch(0.0, False)
    ms = b.elapsed_ms()
print(f"{sys.argv[1:]} run {ms:.3f} ms, {ms / (sc + 1) * 1e3:.1f} us/sweep")
