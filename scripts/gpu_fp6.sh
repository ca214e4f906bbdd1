#!/bin/bash
# FP6 operand probe: parity tests under a short timeout, then C4 timing A/B.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-fp6}
timeout 300 python -m pytest tests -m gpu -q -x -k "fp6" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest fp6 rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
for r in 1 2; do
  for v in 0 1; do echo -n "fp6=$v "; SSQA_TC_FP6=$v timeout 120 python scripts/prof_run.py c4 tcgen05 100 2>&1 | tail -1; done
done
