#!/bin/bash
# Round deliverables on one box: GPU suite, smoke, C3 headline bench (+CPU
# baseline), C4/C5 bench lines, the reference arm, ncu launch list of the C3
# bench, ncu --set full captures of the sweep kernel for C3/C4/C5.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-deliver}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err; echo "bench c3 rc=$?"
for c in c4 c5 c2 c1; do
  timeout 900 python bench.py --config $c --cpu-seconds 10 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; echo "bench ref rc=$?"
for c in c3 c4 c5 c2 c1; do
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$c.json')); r=d['roofline']; print('$c value %.4g ms/step %.1f e2e %.4g frac %.3f (%s) tensor %s cpu %s clk %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], r['frac'], r['bound'], (r.get('tensor') or {}).get('frac', r['frac'] if r['bound']=='tensor' else None), (d.get('cpu_baseline') or {}).get('value'), d['clocks']['sm_mhz']))"
done
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
bash scripts/gpu_ncu_cfg.sh $TAG 20 c3
bash scripts/gpu_ncu_cfg.sh $TAG 6 c4 c5
