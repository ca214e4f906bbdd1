#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-rows}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for c in c4 c5; do
timeout 900 python bench.py --config $c --shard rows --steps 1 --warmup 3 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "rows $c rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$c.json')); print('$c rows value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'tensor', d['roofline']['frac'], 'launches', d['gpu_launches'])"
tail -2 gpurun_out/bench_${TAG}_$c.err
done
