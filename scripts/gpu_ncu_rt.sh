#!/bin/bash
# ncu source-level capture (stall samples per SASS line) of the fused sweep
# kernel over a run long enough to reach the decided phase.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-rt}; SC=${2:-3000}; CFG=${3:-c3}
timeout 300 python scripts/prof_run.py $CFG tcgen05 $SC > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1500 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/prof_run.py $CFG tcgen05 $SC > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log; cat gpurun_out/plain_$TAG.log | tail -1
