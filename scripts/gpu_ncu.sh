#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
TAG=$1; CFG=${2:-c3}; SC=${3:-20}
timeout 120 python scripts/prof_run.py $CFG tcgen05 $SC > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/prof_run.py $CFG tcgen05 $SC > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
