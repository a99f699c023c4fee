#!/bin/bash
# multi-GPU pass: GPU tests (incl. -m multigpu), bench at N GPUs (torchrun), reference arm
TAG=${1:-multi}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/${TAG}_topo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/${TAG}_gputests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_gputests.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus $N --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
echo "ref exit $?" >> gpurun_out/${TAG}_bench_ref.log
