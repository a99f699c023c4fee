#!/bin/bash
# GPU-sourced multicast on a multi-GPU box: kernel pull / kernel push (TMA) /
# copy engines, Llama-3-8B GPU0 -> N-1 peers, with NVLink byte counters
TAG=${1:-mc}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for b in 16 32; do
  for v in "kernel 1 --push 0 --pull 64 --tile 2097152 --pull-mode 0" \
           "kernel 0 --push 32,64 --pull 0 --tile 2097152 --push-mode 1" \
           "kernel 0 --push 64 --pull 0 --tile 2097152 --push-mode 0" \
           "ce 1 --push 0 --pull 1 --tile 268435456"; do
    set -- $v; ex=$1; dir=$2; shift 2
    timeout 600 python tools/nvlink_counters.py -- $TR --master-port 29600 tools/mc_perf.py --dist --config llama3-8b \
      --nodes $N --blocks $b --executor $ex --direction $dir --iters 5 "$@" >> gpurun_out/${TAG}_mc.log 2>&1
    echo "== b=$b $ex dir=$dir $*" >> gpurun_out/${TAG}_mc.log
  done
done
