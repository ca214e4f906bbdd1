#!/bin/bash
# A/B of the resident accumulator tags (SSQA_TC_RES=0/1/2) on full-length runs.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-res}
if [ "${2:-tests}" = tests ]; then
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
fi
for r in 1 2; do
  for cfg in "c3 5000" "c3 1000" "c2 2000"; do
    set -- $cfg
    for res in 0 1 2; do echo -n "res=$res "; SSQA_TC_RES=$res timeout 300 python scripts/prof_run.py $1 tcgen05 $2 2>&1 | tail -1; done
  done
done
