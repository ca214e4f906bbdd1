#!/bin/bash
# C3 operand stages x accumulator-ring slots per epilogue subgroup
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for v in "3 2" "2 3" "2 4" "3 1" "4 1"; do set -- $v
  echo "stages=$1 nps=$2: $(SSQA_TC_STAGES=$1 SSQA_TC_NPS=$2 timeout 300 python scripts/prof_run.py c3 tcgen05 100 2>&1 | tail -1)"
done
