#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 180 python scripts/tc_probe.py > gpurun_out/tc_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/tc_probe.log
if grep -q "MISMATCH\|Error\|error" gpurun_out/tc_probe.log; then echo "probe failed"; exit 0; fi
timeout 900 python -m pytest tests -m gpu -q -k tcgen05 > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
timeout 600 python bench.py --config c3 --engine tcgen05 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c3_tc.log 2>&1
echo done
