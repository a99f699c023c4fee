#!/bin/bash
# GPU-sourced multicast block-count sweep (in-kernel pull and copy engines):
# Llama-3-8B GPU0 -> N-1 peers; the reference planner's elbow is b = 10 at
# N = 4 and 14 at N = 8 (select_block_count, 900 GB/s, 10 us per step)
TAG=${1:-mcb}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for b in 10 12 16 24 32; do
  for v in "kernel 1 --push 0 --pull 64 --tile 2097152 --pull-mode 0" "ce 1 --push 0 --pull 1 --tile 268435456"; do
    set -- $v; ex=$1; dir=$2; shift 2
    echo "== b=$b $ex" >> gpurun_out/${TAG}_mc.log
    timeout 600 $TR --master-port 29600 tools/mc_perf.py --dist --config llama3-8b \
      --nodes $N --blocks $b --executor $ex --direction $dir --iters 5 "$@" >> gpurun_out/${TAG}_mc.log 2>&1
  done
done
