#!/bin/bash
# round deliverable 2: ncu --set full of the fused sweep kernel at C3 (20 sweeps)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-final}
timeout 120 python scripts/prof_run.py c3 tcgen05 20 > gpurun_out/plain2_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/prof_run.py c3 tcgen05 20 > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
