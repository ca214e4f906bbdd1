#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-pf}
timeout 300 python scripts/prof_run.py c1 tcgen05 50 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1
SSQA_TC_STAGES=2 SSQA_TC_NPW=3 timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1
SSQA_TC_STAGES=2 SSQA_TC_NPW=4 timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1
SSQA_TC_EPI=12 timeout 120 python scripts/prof_run.py c3 tcgen05 300 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])"
