#!/bin/bash
# A/B of engine builds on the bench workload (power-capped, long runs):
#   scripts/gpu_ab_bench.sh CFG NAME... (ablbuild/ab/lib_NAME.so), 2 rounds
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CFG=$1; shift
for r in 1 2; do for v in "$@"; do
  SSQA_LIB_PATH=ablbuild/ab/lib_$v.so timeout 600 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['ms_per_step'],1), 'ms/step', d['clocks']['sm_mhz'], 'MHz', d['clocks']['power_w_max'], 'W')"
done; done
