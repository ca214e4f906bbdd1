#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-p4}
SSQA_TC_TRACE=gpurun_out/tl_$TAG.bin timeout 120 python scripts/prof_run.py c3 tcgen05 4 > /dev/null
python scripts/tc_timeline.py gpurun_out/tl_$TAG.bin | sed -n '18,30p;$p'
timeout 120 python scripts/prof_run.py c3 tcgen05 20 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/prof_run.py c3 tcgen05 20 > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
