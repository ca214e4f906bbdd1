#!/bin/bash
# iteration pass: full GPU suite, then per-config sweep timings (prof_run)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-iter}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for c in c3 c4 c5; do
  echo "$c: $(timeout 300 python scripts/prof_run.py $c tcgen05 40 2>&1 | tail -1)"
done
