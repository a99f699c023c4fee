#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over smoke() (tiny config)
TAG=${1:-san}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_${tool}.log 2>&1
  echo "$tool exit $?" >> gpurun_out/${TAG}_${tool}.log
done
