#!/bin/bash
# N=1 bench (ours + reference arm) -> gpurun_out/TAG_bench*.json
TAG=${1:-b}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
echo "ref exit $?" >> gpurun_out/${TAG}_bench_ref.log
free -g > gpurun_out/${TAG}_mem.txt; nproc >> gpurun_out/${TAG}_mem.txt
