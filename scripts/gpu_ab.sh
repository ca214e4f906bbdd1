#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for r in 1 2; do for v in A C E F; do echo -n "$v "; SSQA_LIB_PATH=ablbuild/ab/lib_$v.so timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1; done; done
