#!/bin/bash
# Quick timing of the fused kernel per config: gpu_ab_exp.sh ["ENV=.." variants separated by ';']
cd "$GRAFT_REPO_ROOT" || cd /root/repo
VARS=${1:-"SSQA_TC_EXP=0"}
IFS=';' read -ra VV <<< "$VARS"
for v in "${VV[@]}"; do
  for c in "c3 5000" "c2 2000" "c1 1000" "c4 400" "c5 200"; do
    set -- $c; echo -n "$v $1: "; env $v timeout 300 python scripts/prof_run.py $1 tcgen05 $2 | tail -1
  done
done
