#!/bin/bash
# timeline (MMA / epilogue per row tile) of ablation builds: scripts/gpu_abl_tl.sh CFG ABL...
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CFG=$1; shift
echo "base: $(bash scripts/gpu_timeline_cfg.sh base $CFG | tail -1)"
echo "exp1: $(bash scripts/gpu_timeline_cfg.sh e1 $CFG SSQA_TC_EXP=1 | tail -1)"
for a in "$@"; do
  echo "abl$a: $(bash scripts/gpu_timeline_cfg.sh a$a $CFG SSQA_LIB_PATH=ablbuild/libssqa_abl$a.so | tail -1)"
done
