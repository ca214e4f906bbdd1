#!/bin/bash
# GPU suite + smoke + a short C3 bench line (no CPU baseline, no other configs).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-quick}
timeout 1800 python -m pytest tests -m gpu -q -x -rs > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_c3.json')); r=d['roofline']
print('C3 value %.4g ms %.1f e2e %.4g frac %.3f clk %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], r['frac'], d['clocks']))"
