#!/bin/bash
# End-of-session check on one box: full GPU suite, smoke, C3 headline bench,
# C4/C5 bench lines, the reference arm, row-shard exchanges at G=1.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-final}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err; echo "bench c3 rc=$?"
for c in c4 c5; do
  timeout 900 python bench.py --config $c --cpu-seconds 10 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; echo "bench ref rc=$?"
for c in c3 c4 c5; do
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$c.json')); r=d['roofline']; i8=r.get('int8_equiv') or r.get('tensor',{}).get('int8_equiv'); print('$c value %.4g ms/step %.1f e2e %.4g frac %.3f (%s) int8eq %.3f clk %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], r['frac'], r['bound'], i8['frac'], d['clocks']['sm_mhz']))"
done
