#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 300 python scripts/tc_bisect.py 10,20,100,30 20,20,40,20 50,20,7,5 20,20,1024,12 12,7,37,25 2>&1 | tr '\n' ' '; echo
timeout 900 python -m pytest tests -m gpu -q -x -k tcgen05 2>&1 | tail -2
for c in c1 c2 c3; do timeout 120 python scripts/prof_run.py $c tcgen05 50 2>&1 | grep -v "^ " | tail -1; done
SSQA_TC_TRACE=gpurun_out/tl_c3.bin timeout 120 python scripts/prof_run.py c3 tcgen05 3 > /dev/null
python scripts/tc_timeline.py gpurun_out/tl_c3.bin | tail -1
