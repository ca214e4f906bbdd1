#!/bin/bash
# Timing ablations of the fused kernel at C3 (results are wrong by design;
# tune key "exp": 2 no MMA, 16 no spin operand loads, 8 no J' loads, 32 stale
# neighbour-sign tiles (no copier work), 64 no accumulator stores, 1 no epilogue math)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for e in 0 2 8 16 32 64 96 1; do
  echo -n "exp=$e: "; SSQA_TC_EXP=$e timeout 300 python scripts/prof_run.py c3 tcgen05 ${1:-2000} 2>&1 | tail -1
done
