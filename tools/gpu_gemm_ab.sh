#!/bin/bash
# GEMM A/B: parity tests, then tools/gemm_perf.py with the pair kernel's
# stream-K on (default) and off (LP_GEMM_PAIR_STREAMK=0), 8B and 70B shapes
TAG=${1:-gemmab}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_llama_slices_gpu.py -q -x -p no:cacheprovider \
  > gpurun_out/${TAG}_tests.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_tests.log
for m in llama3-8b llama3-70b; do
  for sk in 1 0; do
    echo "== $m LP_GEMM_PAIR_STREAMK=$sk" >> gpurun_out/${TAG}_perf.txt
    LP_GEMM_PAIR_STREAMK=$sk timeout 600 python tools/gemm_perf.py 128,256,1024,2048,4096 $m >> gpurun_out/${TAG}_perf.txt 2>&1
  done
done
