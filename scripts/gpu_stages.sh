#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for cfg in "2 1" "2 2" "3 1" "3 2" "4 1"; do
  set -- $cfg
  echo "stages=$1 nps=$2: $(SSQA_TC_STAGES=$1 SSQA_TC_NPS=$2 SSQA_TC_TRACE=gpurun_out/tl.bin timeout 120 python scripts/prof_run.py c3 tcgen05 3 2>&1 | tail -1) | $(python scripts/tc_timeline.py gpurun_out/tl.bin | tail -1)"
done
