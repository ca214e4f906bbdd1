#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for r in 1 2 3; do for v in OLD NEW; do echo -n "$v "; SSQA_LIB_PATH=ablbuild/ab/lib_$v.so timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1; done; done
SSQA_LIB_PATH=ablbuild/ab/lib_NEW.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05 and (runs or trials or many)" 2>&1 | tail -2
