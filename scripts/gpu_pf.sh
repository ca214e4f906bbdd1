#!/bin/bash
# J' L2 prefetch distance x CTA pairs for the row-split configs
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for c in c5 c4; do for cta in 1 0; do for pf in 0 8 16 32; do
  echo "$c CTA2=$cta PF=$pf: $(SSQA_TC_CTA2=$cta SSQA_TC_PF=$pf timeout 300 python scripts/prof_run.py $c tcgen05 40 2>&1 | tail -1)"
done; done; done
