#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 1200 python scripts/tc_bisect.py 50,20,148,3 50,20,300,3 50,20,1024,3 50,20,1024,20
timeout 120 python scripts/prof_run.py c3 tcgen05 5
timeout 120 python scripts/prof_run.py c2 tcgen05 50
timeout 120 python scripts/prof_run.py c3 tcgen05 50
