#!/bin/bash
# C4 (FP4 pair) geometry / pipeline-depth sweep with prof_run, then one ncu capture
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-tune}
CFG=${2:-c4}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair or quantizer or multi_instance" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
run() { echo "$*: $(env "$@" timeout 300 python scripts/prof_run.py $CFG tcgen05 40 2>&1 | tail -1)"; }
run X=0
run SSQA_TC_STAGES=5 SSQA_TC_NPS=1
run SSQA_TC_EPI=12
run SSQA_TC_EPI=12 SSQA_TC_STAGES=5 SSQA_TC_NPS=1
run SSQA_TC_WIDE=6
run SSQA_TC_WIDE=6 SSQA_TC_STAGES=5 SSQA_TC_NPS=1
run SSQA_TC_FP4=0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_${TAG}_$CFG python scripts/prof_run.py $CFG tcgen05 6 > gpurun_out/ncu_${TAG}_$CFG.log 2>&1; tail -1 gpurun_out/ncu_${TAG}_$CFG.log
