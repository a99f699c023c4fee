#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${1:-attn}
timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_llama_slices_gpu.py -q -x -s -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_tests.log
timeout 300 python tools/attn_perf.py prefill > gpurun_out/${TAG}_perf_tc.txt 2>&1
LP_ATTN_TC=1 timeout 300 python tools/attn_perf.py prefill > gpurun_out/${TAG}_perf_tc1.txt 2>&1
