#!/bin/bash
# Round-2 deliverables on one box: GPU suite + smoke, the C3 bench line (with
# CPU baseline and the C4/C5 device lines), the reference arm, the ncu launch
# list of a short bench, and ncu --set full captures of the sweep kernel at
# C3 / C4 / C5.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r2}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_c3.json')); r=d['roofline']
print('C3 value %.4g ms %.1f e2e %.4g frac %.3f clk %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], r['frac'], d['clocks']))
for k,v in (d.get('other_configs') or {}).items(): print(k, 'ms %.1f value %.4g tensor %.3f int8eq %.3f clk %s' % (v['ms_per_step'], v['value'], v['tensor']['frac'], v['int8_equiv']['frac'], v['clocks']))
print('cpu', d['cpu_baseline'])"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
for c in c3 c4 c5; do
  sw=20; [ $c != c3 ] && sw=6
  timeout 300 python scripts/prof_run.py $c tcgen05 $sw > gpurun_out/pre_${TAG}_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_${TAG}_$c python scripts/prof_run.py $c tcgen05 $sw > gpurun_out/ncu_${TAG}_$c.log 2>&1; echo "ncu $c rc=$?"
  # the text summary travels back; the report itself (~20 MB) does not fit gpurun_out's 64 MiB
  python scripts/ncu_summary.py gpurun_out/prof_${TAG}_$c.ncu-rep gpurun_out/ncu_k_sweep_tc_${c}_$TAG.txt > /dev/null 2>&1
  rm -f gpurun_out/prof_${TAG}_$c.ncu-rep
done
