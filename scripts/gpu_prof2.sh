#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
TAG=${1:-x}
timeout 120 python scripts/prof_run.py c3 tcgen05 20 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/prof_run.py c3 tcgen05 20 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
