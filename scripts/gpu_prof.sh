#!/bin/bash
# usage: gpu_prof.sh <tag> [config] [engine] [sc]
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-x}; CFG=${2:-c3}; ENG=${3:-tcgen05}; SC=${4:-50}
timeout 180 python scripts/tc_probe.py > gpurun_out/tc_probe_$TAG.log 2>&1; echo "probe rc=$?" >> gpurun_out/tc_probe_$TAG.log
if grep -q "MISMATCH\|Error\|error" gpurun_out/tc_probe_$TAG.log; then echo "probe failed"; cat gpurun_out/tc_probe_$TAG.log; exit 0; fi
timeout 300 python scripts/prof_run.py $CFG $ENG $SC > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/prof_run.py $CFG $ENG $SC > gpurun_out/ncu_$TAG.log 2>&1
cat gpurun_out/prof_plain_$TAG.log
