#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-c5}
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "bench c5 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_c5.json')); print('c5 value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'tensor', d['roofline'].get('tensor',{}).get('frac'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
tail -3 gpurun_out/bench_${TAG}_c5.err
