#!/bin/bash
# correctness probe + timing of C1..C3 (+ optional ncu of C3)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 600 python scripts/tc_bisect.py 10,20,100,30 12,8,5,30 20,20,40,20 50,20,7,5 10,20,1024,5 || exit 1
for c in c1 c2 c3; do timeout 120 python scripts/prof_run.py $c tcgen05 50; done
if [ "$1" == "ncu" ]; then
timeout 120 python scripts/prof_run.py c3 tcgen05 20 > /dev/null && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_$2 python scripts/prof_run.py c3 tcgen05 20 > gpurun_out/ncu_$2.log 2>&1
tail -1 gpurun_out/ncu_$2.log
fi
