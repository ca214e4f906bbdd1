#!/bin/bash
# ncu --set full of the sweep kernel for configs: scripts/gpu_ncu_cfg.sh TAG SWEEPS CFG...
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=$1; SW=$2; shift 2
for c in "$@"; do
  timeout 300 python scripts/prof_run.py $c tcgen05 $SW > gpurun_out/pre_${TAG}_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_${TAG}_$c python scripts/prof_run.py $c tcgen05 $SW > gpurun_out/ncu_${TAG}_$c.log 2>&1; tail -1 gpurun_out/ncu_${TAG}_$c.log
done
