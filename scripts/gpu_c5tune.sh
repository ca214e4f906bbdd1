#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for w in 15 12 11 8; do echo -n "wide=$w "; SSQA_TC_WIDE=$w timeout 300 python scripts/prof_run.py c5 tcgen05 30 2>&1 | tail -1; done
for st in 2 3 4; do for np in 1 2; do echo -n "wide=11 stages=$st nps=$np "; SSQA_TC_WIDE=11 SSQA_TC_STAGES=$st SSQA_TC_NPS=$np timeout 300 python scripts/prof_run.py c5 tcgen05 30 2>&1 | tail -1; done; done
for w in 8 6 4; do echo -n "c4 wide=$w "; SSQA_TC_WIDE=$w timeout 300 python scripts/prof_run.py c4 tcgen05 30 2>&1 | tail -1; done
