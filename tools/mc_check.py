"""Distributed multicast parity check (one process per GPU, torchrun).

For each executor (in-kernel pull, in-kernel push, copy engines) and source
tier (GPU, pinned host) it runs the reference schedule across the ranks and
checks every rank's per-block checksums against the source's.  Prints one
JSON line on rank 0; exit code 1 on any mismatch.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2502_09922_b200 import image as I  # noqa: E402
from paper_2502_09922_b200 import scaleout as SO  # noqa: E402


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    cfg = I.LlamaConfig("mc-check", 8, 1024, 8, 2, 3072, 16384)
    results, ok = [], True
    cases = [("kernel-pull", dict(executor="kernel", direction=1, copy_mode=0, tile_bytes=1 << 20), False),
             ("kernel-push-tma", dict(executor="kernel", direction=0, copy_mode=1, tile_bytes=1 << 20,
                                      push_ctas=16, pull_ctas=16), False),
             ("copy-engine", dict(executor="ce", direction=1, tile_bytes=8 << 20), False),
             ("kernel-pull", dict(executor="kernel", direction=1, copy_mode=0, tile_bytes=1 << 20), True),
             ("copy-engine", dict(executor="ce", direction=1, tile_bytes=8 << 20), True)]
    for name, kw, host in cases:
        n = world + (1 if host else 0)
        plan = SO.plan_scale_out(cfg, n, 1, 8, host_source=host)
        kw = dict(kw)
        kw.setdefault("pull_ctas", 32)
        kw.setdefault("push_ctas", 0 if kw.get("direction", 1) == 1 else 32)
        so = SO.ScaleOut(plan, distributed=True, seed=3, device=torch.cuda.current_device(), **kw)
        so.load_sources()
        for _ in range(2):
            dist.barrier()
            so.run()
        mine = {nd: so.checksums(nd) for nd in so.cluster.exec_nodes}
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        src = [so.checksums(0) if rank == 0 else None]
        dist.broadcast_object_list(src, src=0)
        good = all(v == src[0] for d in allv for v in d.values())
        ok &= good
        results.append({"case": name, "host_source": host, "nodes": n, "byte_exact": good})
        dist.barrier()
        so.close()
    if rank == 0:
        print(json.dumps({"world": world, "results": results, "ok": ok}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
