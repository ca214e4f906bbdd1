#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for E in 8 12 16; do
  SSQA_TC_EPI=$E timeout 180 python scripts/tc_probe.py > gpurun_out/tc_probe_e$E.log 2>&1
  echo "epi=$E probe: $(grep -c OK gpurun_out/tc_probe_e$E.log) ok, $(grep -c MISMATCH gpurun_out/tc_probe_e$E.log) bad"
  SSQA_TC_EPI=$E timeout 300 python scripts/prof_run.py c3 tcgen05 50
done
SSQA_TC_EPI=16 timeout 300 python scripts/prof_run.py c3 tcgen05 50 > /dev/null 2>&1 && \
SSQA_TC_EPI=16 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_e16 python scripts/prof_run.py c3 tcgen05 50 > gpurun_out/ncu_e16.log 2>&1
echo done
