#!/bin/bash
# GPU suite (incl. SSA) + first C4/C5 measurements
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-ssa}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log; tail -3 gpurun_out/pytest_$TAG.log
for c in c4 c5; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "bench $c rc=$?"
  tail -c 600 gpurun_out/bench_${TAG}_$c.json; tail -3 gpurun_out/bench_${TAG}_$c.err
done
