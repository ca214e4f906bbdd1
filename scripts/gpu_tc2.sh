#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 180 python scripts/tc_probe.py > gpurun_out/tc_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/tc_probe.log
if grep -q "MISMATCH\|Error\|error" gpurun_out/tc_probe.log; then echo "probe failed"; exit 0; fi
timeout 900 python -m pytest tests -m gpu -q -k tcgen05 > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
timeout 300 python scripts/prof_run.py c3 tcgen05 50 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_tc -s 1 -c 1 -o gpurun_out/prof_tc_c3 python scripts/prof_run.py c3 tcgen05 50 > gpurun_out/ncu_tc.log 2>&1
timeout 600 python bench.py --config c3 --engine tcgen05 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_tc.log 2>&1
echo done
