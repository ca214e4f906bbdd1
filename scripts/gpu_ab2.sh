#!/bin/bash
# A/B of engine builds on full-length runs: ablbuild/ab/lib_<NAME>.so, configs c3 c4 c5.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for r in 1 2; do
  for cfg in "c3 2000" "c4 200" "c5 100"; do
    set -- $cfg
    for v in "${@:3}" $LIBS; do echo -n "$v $1 "; SSQA_LIB_PATH=ablbuild/ab/lib_$v.so timeout 200 python scripts/prof_run.py $1 tcgen05 $2 2>&1 | tail -1; done
  done
done
