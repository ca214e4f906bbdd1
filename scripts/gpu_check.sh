#!/bin/bash
# GPU suite + smoke + C3/C5 bench lines (e2e through the pool, pinned model).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-check}
timeout 1200 python -m pytest tests -m gpu -q -x -rs > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
for c in c3 c5; do
  timeout 900 python bench.py --config $c --cpu-seconds 10 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "bench $c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$c.json')); print('$c', 'value %.4g e2e %.4g (%.3f s, %s) ms/step %.1f frac %.3f clk %s' % (d['value'], d['e2e']['value'], d['e2e']['seconds_per_step'], d['e2e'].get('h2d_source'), d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz']))"
done
