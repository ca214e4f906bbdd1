#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-large}
free -g | head -2; nproc
timeout 900 python -m pytest tests/test_gpu_large.py -q -x -s > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest large rc=$?"; tail -4 gpurun_out/pytest_$TAG.log
for c in c4 c5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "bench $c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$c.json')); print('$c value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'tensor', d['roofline'].get('tensor',{}).get('frac'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
done
