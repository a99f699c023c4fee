"""Debug timings of the sharded host load on N ranks (dev tool)."""
import dataclasses, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2502_09922_b200 import scaleout as SO, multicast as M

dist.init_process_group("nccl")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(r)
plan = SO.plan_scale_out("llama2-13b", w + 1, 1, 40, host_source=True, strategy="sharded_host")
scatter = M.MulticastSchedule(plan.schedule.groups, [[t for t in row if t.sender == 0] for row in plan.schedule.steps],
                              max_send_degree=w, enforce_step_bound=False, label="scatter")


def run(name, p, ex, verify, tile=SO.HYBRID_TILE, pull=64, own=False):
    so = SO.ScaleOut(p, distributed=True, executor=ex, tile_bytes=tile, pull_ctas=pull, push_ctas=0,
                     direction=1, copy_mode=0, verify=verify, device=r)
    so.load_sources()
    ts = []
    st = torch.cuda.Stream() if own else None
    for i in range(4):
        dist.barrier()
        torch.cuda.synchronize()
        res = so.run(st)
        t = torch.tensor([res.kernel_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ts.append(round(t.item(), 1))
    if r == 0:
        print(name, ex, "verify" if verify else "", "tile", tile >> 20, "pull", pull, "own stream" if own else "", ts, flush=True)
    dist.barrier()
    so.close()


run("sharded", plan, "hybrid", True)
run("sharded", plan, "hybrid", True, own=True)
run("sharded", plan, "hybrid", False, own=True)
dist.destroy_process_group()
