#!/bin/bash
# A/B: the build before the fused shard exchange (ablbuild/pre, its own package) vs HEAD.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for r in 1 2 3; do
  for cfg in "c4 200" "c5 100" "c3 1000"; do
    set -- $cfg
    echo -n "pre  $1 "; (cd ablbuild/pre && timeout 200 python scripts/prof_run.py $1 tcgen05 $2 2>&1 | tail -1)
    echo -n "head $1 "; timeout 200 python scripts/prof_run.py $1 tcgen05 $2 2>&1 | tail -1
  done
done
