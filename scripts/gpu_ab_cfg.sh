#!/bin/bash
# Quick timing of the fused kernel per config (second launch of prof_run): gpu_ab_cfg.sh ["ENV=.." variants separated by ';']
cd "$GRAFT_REPO_ROOT" || cd /root/repo
VARS=${1:-"SSQA_TC_EXP=0"}
IFS=';' read -ra VV <<< "$VARS"
for v in "${VV[@]}"; do
  for c in "c3 100" "c3 5000" "c2 2000" "c1 1000"; do
    set -- $c; echo -n "$v $1 $2: "; env $v timeout 300 python scripts/prof_run.py $1 tcgen05 $2 2>&1 | tail -1
  done
done
