#!/bin/bash
# Row-shard exchanges on one GPU: peer-push tests, then --shard rows C4 with the
# NCCL all-gather and with the peer push (G = 1: own region, no IPC).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-p2p}
timeout 900 python -m pytest tests -m gpu -q -x -k "row_shard or peer_push or pool or fused_run or row_split" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for ex in nccl p2p direct; do
  timeout 900 python bench.py --config c4 --shard rows --exchange $ex > gpurun_out/bench_${TAG}_c4_$ex.json 2> gpurun_out/bench_${TAG}_c4_$ex.err; echo "rows $ex rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_c4_$ex.json')); print('$ex', 'value %.4g e2e %.4g ms/step %.1f frac %.3f clk %s launches %s' % (d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['gpu_launches']))"
done
