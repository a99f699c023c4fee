#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python tools/verify_debug.py > gpurun_out/dbg_verify.log 2>&1
echo "exit $?" >> gpurun_out/dbg_verify.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/verify_debug.py > gpurun_out/dbg_verify_blocking.log 2>&1
timeout 300 python tools/parity_probe.py tiny 24 > gpurun_out/dbg_probe_tiny.log 2>&1
timeout 300 python tools/parity_probe.py llama3-8b 160 > gpurun_out/dbg_probe_8b.log 2>&1
