#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
export SSQA_TC_EPI=12
timeout 120 python scripts/prof_run.py c2 tcgen05 50 > gpurun_out/dbg_c2.log 2>&1
grep watchdog gpurun_out/dbg_c2.log | awk '{print $3, $5, $6, $12}' | sort | uniq -c | sort -k3,3n -k5 | head -60
