#!/bin/bash
# FP4 pair operands: parity tests, full-size C4 check, C4 bench (pair vs int8)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-pair}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair or dense or row_split or quantizer" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python -m pytest tests/test_gpu_large.py -q -x -k c4 > gpurun_out/pytest_large_$TAG.log 2>&1; echo "pytest large rc=$?"; tail -2 gpurun_out/pytest_large_$TAG.log
for v in pair int8; do
  if [ $v = int8 ]; then export SSQA_TC_FP4=0; fi
  timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c4_$v.json 2> gpurun_out/bench_${TAG}_c4_$v.err; echo "bench $v rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_c4_$v.json')); print('$v value', d['value'], 'ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'tensor', d['roofline'].get('tensor',{}).get('frac'))"
done
