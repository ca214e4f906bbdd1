#!/bin/bash
# Rail-tag epilogue vs FP64 epilogue: C3 run time against the sweep budget
# (the undecided fraction falls with the cycle, scripts/decided_probe.py).
# usage: gpu_rt_phase.sh [cfg] ["ENV=.. ENV=.." variants separated by ';']
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
CFG=${1:-c3}
VARS=${2:-"SSQA_TC_RT=0;SSQA_TC_RT=1"}
IFS=';' read -ra VV <<< "$VARS"
for sc in 100 400 1000 2000 5000; do
  for v in "${VV[@]}"; do
    echo -n "sc=$sc $v: "
    env $v timeout 300 python scripts/prof_run.py $CFG tcgen05 $sc 2>&1 | tail -1
  done
done
