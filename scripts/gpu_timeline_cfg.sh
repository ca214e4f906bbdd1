#!/bin/bash
# per-row-tile timeline (block 0) for a config: scripts/gpu_timeline_cfg.sh TAG CFG [ENV=V ...]
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=$1; CFG=$2; shift 2
env "$@" SSQA_TC_TRACE=gpurun_out/tl_${TAG}_$CFG.bin timeout 120 python scripts/prof_run.py $CFG tcgen05 3 > /dev/null
python scripts/tc_timeline.py gpurun_out/tl_${TAG}_$CFG.bin
