#!/bin/bash
# split executor (every other block's GPU->GPU transfers on the copy engines
# in 64 MiB tiles, the rest in-kernel) vs the in-kernel executor: byte-exact
# tests, then Llama-3-8B GPU0 -> N-1 peers at b = 16
TAG=${1:-split}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_scaleout_gpu.py tests/test_multicast_gpu.py -q -x -p no:cacheprovider \
  > gpurun_out/${TAG}_tests.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for v in "kernel --pull 64 --tile 2097152" "split --pull 64 --tile 2097152" "split --pull 48 --tile 2097152" \
         "split --pull 64 --tile 4194304"; do
  set -- $v; ex=$1; shift
  echo "== $ex $*" >> gpurun_out/${TAG}_mc.log
  timeout 600 $TR --master-port 29600 tools/mc_perf.py --dist --config llama3-8b --nodes $N --blocks 16 \
    --executor $ex --direction 1 --push 0 --pull-mode 0 --iters 5 "$@" >> gpurun_out/${TAG}_mc.log 2>&1
done
