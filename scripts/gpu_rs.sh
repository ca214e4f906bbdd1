#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-rs}
timeout 600 python -m pytest tests -m gpu -q -x -k "row_split or wide_row" > gpurun_out/pytest_${TAG}_rs.log 2>&1; echo "pytest rs rc=$?"; tail -4 gpurun_out/pytest_${TAG}_rs.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest all rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1
timeout 300 python scripts/prof_run.py c4 tcgen05 20 2>&1 | tail -1
timeout 600 python scripts/prof_run.py c5 tcgen05 10 2>&1 | tail -1
