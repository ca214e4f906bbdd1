cd "$GRAFT_REPO_ROOT"
for v in "SSQA_TC_RT=1" "SSQA_TC_RT=1 SSQA_TC_EXP=256" "SSQA_TC_RT=1 SSQA_TC_EXP=768" "SSQA_TC_RT=1 SSQA_TC_EXP=1792"; do
  for sc in 2000 4000; do echo -n "$v sc=$sc: "; env $v timeout 300 python scripts/prof_run.py c3 tcgen05 $sc | tail -1; done
done
