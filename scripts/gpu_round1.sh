#!/bin/bash
# First GPU pass: parity tests, smoke, short benches.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python bench.py --config c1 --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_c1.log 2>&1
timeout 900 python bench.py --config c3 --steps 2 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c3.log 2>&1
echo done
