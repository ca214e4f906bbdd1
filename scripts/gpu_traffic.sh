#!/bin/bash
# DRAM traffic of the fused kernel over the whole bench workload of each
# config (one metric pass, no source counters): gpu_traffic.sh TAG
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r2}
for c in "c3 5000" "c4 2000" "c5 1000" "c2 2000"; do
  set -- $c
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum \
    --clock-control none -k regex:k_sweep -s 1 -c 1 --csv --log-file gpurun_out/traffic_${TAG}_$1.csv \
    python scripts/prof_run.py $1 tcgen05 $2 > gpurun_out/traffic_${TAG}_$1.log 2>&1
  echo "$1 rc=$?"; grep -E "dram__|gpu__time|lts__|xbar" gpurun_out/traffic_${TAG}_$1.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
