#!/bin/bash
# A/B timing of engine builds: ablbuild/ab/lib_<NAME>.so for each NAME given
# (build them with nvcc as in scripts/build_ablations.sh), C3, 300 sweeps, 3 rounds.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for r in 1 2 3; do for v in "$@"; do echo -n "$v "; SSQA_LIB_PATH=ablbuild/ab/lib_$v.so timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1; done; done
