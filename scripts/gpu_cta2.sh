#!/bin/bash
# CTA pairs: row-split parity (pairs / single), full-size C4/C5, timings
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-cta2}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "row_split or pair or wide or multi_instance" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 900 python -m pytest tests/test_gpu_large.py -q -x > gpurun_out/pytest_large_$TAG.log 2>&1; echo "pytest large rc=$?"; tail -2 gpurun_out/pytest_large_$TAG.log
for c in c4 c5; do
  for v in 1 0; do
    echo "$c CTA2=$v: $(SSQA_TC_CTA2=$v timeout 300 python scripts/prof_run.py $c tcgen05 40 2>&1 | tail -1)"
  done
done
