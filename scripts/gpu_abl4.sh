#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 300 python scripts/tc_bisect.py 10,20,100,30 20,20,40,20 50,20,7,5 12,7,37,25 2>&1 | tr '\n' ' '; echo
for E in 12 16; do
echo "SHFL EPI=$E: $(SSQA_TC_EPI=$E SSQA_TC_TRACE=gpurun_out/tl.bin timeout 120 python scripts/prof_run.py c3 tcgen05 20 2>&1 | tail -1) | $(python scripts/tc_timeline.py gpurun_out/tl.bin | tail -1)"
echo "REDUX EPI=$E: $(SSQA_LIB_PATH=$PWD/ablbuild/libssqa_abl0_r0.so SSQA_TC_EPI=$E SSQA_TC_TRACE=gpurun_out/tl.bin timeout 120 python scripts/prof_run.py c3 tcgen05 20 2>&1 | tail -1) | $(python scripts/tc_timeline.py gpurun_out/tl.bin | tail -1)"
done
