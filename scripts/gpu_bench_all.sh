#!/bin/bash
# Large-shape GPU tests + one bench line with the C4/C5 device lines (no CPU baseline).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_large.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_all_c3.json 2> gpurun_out/bench_all_c3.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_all_c3.json')); r=d['roofline']
print('C3 value %.4g ms %.1f e2e %.4g frac %.3f clk %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], r['frac'], d['clocks']))
for k,v in (d.get('other_configs') or {}).items(): print(k, 'ms %.1f value %.4g tensor %.3f int8eq %.3f clk %s' % (v['ms_per_step'], v['value'], v['tensor']['frac'], v['int8_equiv']['frac'], v['clocks']))"
