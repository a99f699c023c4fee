#!/bin/bash
# One GPU-box pass: GPU tests, smoke, smoke under ncu (launch list).
#   gpurun -- bash tools/gpu_check.sh TAG      (outputs under gpurun_out/TAG_*)
TAG=${1:-check}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
nproc >> gpurun_out/${TAG}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rs -s -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/${TAG}_gputests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" \
  > gpurun_out/${TAG}_smoke_ncu.log 2>&1
echo "ncu smoke exit $?" >> gpurun_out/${TAG}_smoke_ncu.log
