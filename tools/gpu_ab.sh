#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${1:-ab}
for v in "" "--no-verify" "--no-poison" "--executor kernel"; do
  echo "== $v" >> gpurun_out/${TAG}.log
  timeout 600 python bench.py --steps 5 --warmup 2 $v 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['config']['host_executors'])" >> gpurun_out/${TAG}.log 2>&1
done
