#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
SSQA_TC_TRACE=gpurun_out/tl2_c3.bin timeout 120 python scripts/prof_run.py c3 tcgen05 4 > /dev/null
python scripts/tc_timeline.py gpurun_out/tl2_c3.bin
