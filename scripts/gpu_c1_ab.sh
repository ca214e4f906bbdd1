#!/bin/bash
# C1 (N=100, latency-bound) A/B: engines and epilogue variants, same box.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
run() { local tag=$1; shift; env "$@" timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 5 --warmup 3 ${ENGARG} > gpurun_out/c1ab_$tag.json 2> gpurun_out/c1ab_$tag.err; python -c "import json; d=json.load(open('gpurun_out/c1ab_$tag.json')); print('$tag', '%.3f ms/step' % d['ms_per_step'], '%.4g' % d['value'], d['config'].get('engine'))" 2>/dev/null || echo "$tag failed"; }
for rep in 1 2; do
ENGARG="" run base$rep SSQA_X=0
ENGARG="" run tab1_$rep SSQA_TC_TAB=1
ENGARG="" run epi12_$rep SSQA_TC_EPI=12
ENGARG="--engine simt" run simt$rep SSQA_X=0
done
