#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 300 python scripts/tc_bisect.py 10,20,100,30 20,20,40,20 50,20,7,5 12,7,37,25 2>&1 | tr '\n' ' '; echo
for F in 1 0; do
  for c in c2 c3; do echo "FP4=$F $(SSQA_TC_FP4=$F timeout 120 python scripts/prof_run.py $c tcgen05 50 2>&1 | grep -v '^ ' | tail -1)"; done
done
SSQA_TC_TRACE=gpurun_out/tl_f4.bin timeout 120 python scripts/prof_run.py c3 tcgen05 20 > /dev/null 2>&1
python scripts/tc_timeline.py gpurun_out/tl_f4.bin | tail -1
timeout 900 python -m pytest tests -m gpu -q -x -k tcgen05 2>&1 | tail -2
