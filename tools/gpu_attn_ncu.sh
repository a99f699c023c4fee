#!/bin/bash
# ncu --set full (with source) of one prefill attention launch, variant $2
TAG=${1:-attnncu}; V=${2:-3}; H=${3:-32}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
LP_ATTN_TC=$V ATTN_ITERS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention_ -s 5 -c 1 \
  -o gpurun_out/${TAG} python tools/attn_perf.py pone $H 8 1 2048 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/${TAG}_ncu.log
