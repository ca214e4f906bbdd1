#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
echo "BASE: $(SSQA_TC_EPI=16 SSQA_TC_TRACE=gpurun_out/tl.bin timeout 120 python scripts/prof_run.py c3 tcgen05 20 2>&1 | tail -1) | $(python scripts/tc_timeline.py gpurun_out/tl.bin | tail -1)"
for A in 16 32 64 112; do
  echo "ABL=$A: $(SSQA_LIB_PATH=$PWD/ablbuild/libssqa_abl$A.so SSQA_TC_EPI=16 SSQA_TC_TRACE=gpurun_out/tl.bin timeout 120 python scripts/prof_run.py c3 tcgen05 20 2>&1 | tail -1) | $(python scripts/tc_timeline.py gpurun_out/tl.bin | tail -1)"
done
