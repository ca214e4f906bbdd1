"""Where the e2e time of one C3 ssqa_run_batch call goes (problem upload,
batch allocation, run, fetch, teardown)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2302_12454_b200 as sq
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
m = bench.build_model(cfg)
p = sq.SsqaParams(r=cfg["R"], sc=cfg["sc"])
seeds = [1000 + t for t in range(cfg["T"])]
for it in range(3):
    t0 = time.perf_counter(); prob = sq.Problem(m); t1 = time.perf_counter()
    b = sq.Batch(prob, p, len(seeds)); t2 = time.perf_counter()
    b.set_seeds(seeds); b.launch(0.0, False); ms = b.elapsed_ms(); t3 = time.perf_counter()
    b.fetch(True, False); t4 = time.perf_counter()
    b.close(); prob.close(); t5 = time.perf_counter()
    print(f"problem {1e3*(t1-t0):.1f} ms  batch {1e3*(t2-t1):.1f} ms  run(wall) {1e3*(t3-t2):.1f} ms "
          f"(device {ms:.1f})  fetch {1e3*(t4-t3):.1f} ms  teardown {1e3*(t5-t4):.1f} ms")
