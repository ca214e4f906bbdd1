#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for r in 1 2 3; do for v in $LIBS; do echo -n "$v "; SSQA_LIB_PATH=ablbuild/ab/lib_$v.so timeout 200 python scripts/prof_run.py c3 tcgen05 2000 2>&1 | tail -1; done; done
