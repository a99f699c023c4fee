#!/bin/bash
# prefill attention variant A/B: parity tests under each LP_ATTN_TC variant
# given, then the prefill timing table for the default (1) and each variant,
# plus a chunk trace of the last one
TAG=${1:-attnab}; shift; VS=${@:-3}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for V in $VS; do
  echo "== LP_ATTN_TC=$V" >> gpurun_out/${TAG}_tests.log
  LP_ATTN_TC=$V timeout 600 python -m pytest tests/test_decoder_gpu.py tests/test_llama_slices_gpu.py -q -x \
    -k "attention or tiny or generate or slice" -p no:cacheprovider >> gpurun_out/${TAG}_tests.log 2>&1
  echo "exit $?" >> gpurun_out/${TAG}_tests.log
done
for v in 1 $VS; do
  echo "== LP_ATTN_TC=$v" >> gpurun_out/${TAG}_perf.txt
  LP_ATTN_TC=$v timeout 300 python tools/attn_perf.py prefill >> gpurun_out/${TAG}_perf.txt 2>&1
done
LP_ATTN_TC=$V LP_ATTN_TRACE=1 ATTN_ITERS=1 timeout 120 python tools/attn_perf.py pone 32 8 1 2048 > gpurun_out/${TAG}_trace.txt 2>&1
