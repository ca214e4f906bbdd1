#!/bin/bash
# Block-0 timeline (MMA / loader / epilogue per row tile) of a C3 run, from
# row tile SKIP on: gpu_timeline.sh [sweeps] [skip] ["ENV=.."]
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
SC=${1:-4}; SKIP=${2:-0}; EXTRA=${3:-}
env $EXTRA SSQA_TC_TSKIP=$SKIP SSQA_TC_TRACE=gpurun_out/tl_c3.bin timeout 300 python scripts/prof_run.py c3 tcgen05 $SC | tail -1
python scripts/tc_timeline.py gpurun_out/tl_c3.bin
