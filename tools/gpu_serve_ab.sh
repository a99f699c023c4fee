#!/bin/bash
# execute-while-load A/B over the pipeline's batch and prefill budget
# (serve_bench, GPU-sourced and host-sourced plans) + the host-fed GPU tests
TAG=${1:-sab}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_serving_host_gpu.py tests/test_serving_gpu.py -m gpu -q -rs -p no:cacheprovider \
  > gpurun_out/${TAG}_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_tests.log
for src in "" "--host-source"; do
  for cfg in "1 256" "16 256" "16 128" "4 256" "16 512"; do
    set -- $cfg
    echo "== src=${src:-gpu} pipeline_batch=$1 prefill_tokens=$2" >> gpurun_out/${TAG}_serve.log
    timeout 300 python tools/serve_bench.py --gpus $N $src --pipeline-batch $1 --pipeline-prefill-tokens $2 \
      >> gpurun_out/${TAG}_serve.log 2>&1
  done
done
