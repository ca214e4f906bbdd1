#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 300 python scripts/tc_bisect.py 10,20,100,30 20,20,40,20 50,20,7,5 12,7,37,25 3,2,5,20 2>&1 | tr '\n' ' '; echo
timeout 900 python -m pytest tests -m gpu -q -x -k tcgen05 2>&1 | tail -2
bash scripts/gpu_ncu.sh f4a c3 20
