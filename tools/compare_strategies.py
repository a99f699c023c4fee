"""Scale-out strategies side by side on real GPUs (one process per GPU).

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/compare_strategies.py \
      --config llama3-8b --blocks 16 --out gpurun_out/compare.json

Every arm moves the same packed image from rank 0 to all other ranks:

* ``lambdapipe/<executor>`` — the λPipe binomial pipeline (compose_schedule)
  executed by the multicast engine;
* ``binary_tree/<executor>`` and ``broadcast_groups/kernel`` — the reference's
  comparator schedules (simengine.py:106-151, our cluster.baseline_schedule)
  executed by the same engine, so only the schedule differs;
* ``nccl_broadcast/blocks`` and ``nccl_broadcast/whole`` — the image sent with
  ``torch.distributed.broadcast`` (NCCL over NVLink) per block / in one call,
  on a freshly created communicator whose creation time is reported
  separately (the reference models it as ``baseline_group_init_s``).

Times are device time, max over ranks, median of ``--iters``; every arm is
verified by per-block checksums against the source.
"""
import argparse
import dataclasses
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2502_09922_b200 import engine as E  # noqa: E402
from paper_2502_09922_b200 import scaleout as SO  # noqa: E402
from paper_2502_09922_b200.cluster import b200_box, baseline_schedule  # noqa: E402


def _max(x: float) -> float:
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def run_engine(plan, executor, iters, tile):
    # the bench's in-kernel configuration: receivers pull with LDG vectors
    # (copy_mode 0), 64 CTAs per receiver
    so = SO.ScaleOut(plan, distributed=True, executor=executor, tile_bytes=tile, copy_mode=0, pull_ctas=64,
                     device=torch.cuda.current_device())
    so.load_sources()
    times = []
    for it in range(iters + 2):
        dist.barrier()
        torch.cuda.synchronize()
        r = so.run()
        ms = _max(r.kernel_ms)
        if it >= 2:
            times.append(ms)
    ref = [None]
    if dist.get_rank() == 0:
        ref = [so.checksums(0)]
    dist.broadcast_object_list(ref, src=0)
    ok = so.checksums(dist.get_rank()) == ref[0]
    ok = _max(0.0 if ok else 1.0) == 0.0
    dist.barrier()
    so.close()
    return sorted(times)[len(times) // 2], min(times), ok


def run_nccl(plan, iters, seed=0):
    lay = plan.layout
    dev = torch.cuda.current_device()
    rank = dist.get_rank()
    buf = torch.empty(lay.weights_bytes, dtype=torch.uint8, device="cuda")
    if rank == 0:
        E.fill_image(buf.data_ptr(), lay, seed)
    else:
        buf.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    # fresh communicator: NCCL creates it lazily on the first collective
    t0 = time.perf_counter()
    grp = dist.new_group(list(range(dist.get_world_size())), backend="nccl")
    one = torch.zeros(1, device="cuda")
    dist.broadcast(one, 0, group=grp)
    torch.cuda.synchronize()
    init_ms = _max((time.perf_counter() - t0) * 1e3)
    views = [buf[o:o + n] for o, n in zip(lay.block_offsets, lay.block_lengths)]
    out = {}
    for mode in ("blocks", "whole"):
        times = []
        for it in range(iters + 2):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if mode == "blocks":
                for v in views:
                    dist.broadcast(v, 0, group=grp)
            else:
                dist.broadcast(buf, 0, group=grp)
            e1.record()
            torch.cuda.synchronize()
            ms = _max(e0.elapsed_time(e1))
            if it >= 2:
                times.append(ms)
        out[mode] = (sorted(times)[len(times) // 2], min(times))
    cs = E.block_checksums(buf.data_ptr(), lay.block_offsets, lay.block_lengths)
    ref = [cs]
    dist.broadcast_object_list(ref, src=0)
    ok = _max(0.0 if cs == ref[0] else 1.0) == 0.0
    dist.destroy_process_group(grp)
    del buf
    torch.cuda.empty_cache()
    return init_ms, out, ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3-8b")
    ap.add_argument("--blocks", type=int, default=16)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    plan = SO.plan_scale_out(a.config, world, 1, a.blocks)
    cluster = b200_box(node_count=world)
    M = plan.layout.weights_bytes
    rows = []

    def emit(name, med, best, ok, steps, extra=None):
        rec = {"arm": name, "ms_med": round(med, 3), "ms_best": round(best, 3), "byte_exact": ok,
               "steps": steps, "agg_GBps": round((world - 1) * M / (med * 1e-3) / 1e9, 1)}
        rec.update(extra or {})
        rows.append(rec)
        if rank == 0:
            print(json.dumps(rec), flush=True)

    arms = [("lambdapipe", plan.schedule)]
    for strat in ("binary_tree", "broadcast_groups"):
        arms.append((strat, baseline_schedule(strat, plan.nodes, plan.layout.plan, cluster)))
    for name, sched in arms:
        p = dataclasses.replace(plan, schedule=sched)
        execs = [("kernel", 2 << 20), ("ce", SO.CE_TILE)] if name != "broadcast_groups" \
            else [("kernel", 2 << 20)]
        for ex, tile in execs:
            med, best, ok = run_engine(p, ex, a.iters, tile)
            emit(f"{name}/{ex}", med, best, ok, sched.step_count)
    init_ms, out, ok = run_nccl(plan, a.iters)
    for mode, (med, best) in out.items():
        emit(f"nccl_broadcast/{mode}", med, best, ok, None, {"comm_init_ms": round(init_ms, 1)})
    if rank == 0:
        summary = {"config": a.config, "n_gpus": world, "blocks": a.blocks, "image_bytes": M,
                   "source": "gpu rank 0", "arms": rows}
        print(json.dumps(summary), flush=True)
        if a.out:
            os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
            json.dump(summary, open(a.out, "w"), indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
