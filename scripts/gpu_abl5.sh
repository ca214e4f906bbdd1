#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1
SSQA_LIB_PATH=ablbuild/libssqa_abl128.so timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1
timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1
