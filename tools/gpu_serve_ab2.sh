#!/bin/bash
# execute-while-load with the default (FLOP-budget) pipeline prefill: 8B GPU-
# and host-sourced, 70B (in-kernel multicast, as bench.py runs it) at
# pipeline batch 16 (bench default) and 1 (the reference's capacity)
TAG=${1:-sab2}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for args in "" "--host-source" "--model llama3-70b --executor kernel --pull-ctas 64" \
            "--model llama3-70b --executor kernel --pull-ctas 64 --pipeline-batch 1"; do
  echo "== $args" >> gpurun_out/${TAG}_serve.log
  timeout 400 python tools/serve_bench.py --gpus $N $args >> gpurun_out/${TAG}_serve.log 2>&1
done
