#!/bin/bash
# decode-step timing (8B, B=16) and the per-kernel launch list of one captured step under ncu
TAG=${1:-dec}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python tools/decode_perf.py llama3-8b 16 > gpurun_out/${TAG}_perf.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/decode_profile.py 16 > gpurun_out/${TAG}_ncu.log 2>&1
