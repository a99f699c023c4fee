#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${1:-nvl}
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
nvidia-smi nvlink -gt d > gpurun_out/${TAG}_smi_gt.txt 2>&1
nvidia-smi nvlink -s > gpurun_out/${TAG}_smi_s.txt 2>&1
for v in "kernel 1 --push 0 --pull 64 --tile 2097152 --pull-mode 0" "ce 1 --push 0 --pull 1 --tile 268435456"; do
  set -- $v; ex=$1; dir=$2; shift 2
  timeout 600 python tools/nvlink_counters.py -- $TR --master-port 29600 tools/mc_perf.py --dist --config llama3-8b \
    --nodes $N --blocks 16 --executor $ex --direction $dir --iters 5 "$@" >> gpurun_out/${TAG}_mc.log 2>&1
done
