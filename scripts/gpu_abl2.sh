#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for X in 0 4 8 12 1; do
  echo "EXP=$X: $(SSQA_TC_EPI=16 SSQA_TC_EXP=$X SSQA_TC_TRACE=gpurun_out/tl.bin timeout 120 python scripts/prof_run.py c3 tcgen05 20 2>&1 | tail -1) | $(python scripts/tc_timeline.py gpurun_out/tl.bin | tail -1)"
done
