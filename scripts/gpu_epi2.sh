#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for E in 12 16 8; do
  echo "== EPI=$E"
  SSQA_TC_EPI=$E timeout 600 python scripts/tc_bisect.py 10,20,100,30 12,8,5,30 20,20,40,20 50,20,7,5 10,7,300,9 20,20,1024,12 2>&1 | tr '\n' ' '; echo
  for c in c1 c2 c3; do SSQA_TC_EPI=$E timeout 120 python scripts/prof_run.py $c tcgen05 50 2>&1 | grep -v "^ " | tail -1; done
done
