"""Multicast engine perf sweep (dev tool).  Single GPU (local emulation) or
one process per GPU under torchrun (real NVLink / IPC).

  python tools/mc_perf.py --config llama2-13b --n 2 --host --b 40
  torchrun --nproc-per-node 4 tools/mc_perf.py --dist --config llama3-8b --n 4 --b 16
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2502_09922_b200 import scaleout as SO  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3-8b")
    ap.add_argument("--nodes", type=int, default=4)
    ap.add_argument("--sources", type=int, default=1)
    ap.add_argument("--blocks", type=int, default=16)
    ap.add_argument("--host", action="store_true")
    ap.add_argument("--dist", action="store_true")
    ap.add_argument("--push", default="16,32,64")
    ap.add_argument("--pull", default="16")
    ap.add_argument("--tile", default="524288")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--verify", action="store_true")
    ap.add_argument("--direction", type=int, default=1)
    ap.add_argument("--push-mode", type=int, default=1)
    ap.add_argument("--pull-mode", type=int, default=1)
    ap.add_argument("--chunk", default="16384")
    ap.add_argument("--timeline", default="")
    ap.add_argument("--window", default="3")
    ap.add_argument("--executor", default="kernel")
    ap.add_argument("--ce-streams", type=int, default=2)
    ap.add_argument("--wide", default="0")
    a = ap.parse_args()
    rank = 0
    if a.dist:
        dist.init_process_group("nccl")
        rank = dist.get_rank()
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    else:
        torch.cuda.set_device(0)
    plan = SO.plan_scale_out(a.config, a.nodes, a.sources, a.blocks, host_source=a.host)
    M = plan.layout.weights_bytes
    R = len(plan.receivers)
    results = []
    for tile in [int(x) for x in a.tile.split(",")]:
        so = SO.ScaleOut(plan, distributed=a.dist, tile_bytes=tile, device=torch.cuda.current_device(),
                         executor=a.executor, ce_streams=a.ce_streams, direction=a.direction)
        so.load_sources()
        for chunk, window, wide in [(int(c), int(w), int(x)) for c in a.chunk.split(",") for w in a.window.split(",")
                                    for x in a.wide.split(",")]:
          so.cluster.engine.configure(a.direction, a.push_mode, a.pull_mode, chunk, window)
          so.cluster.engine.set_option("wide_loads", wide)
          for push in [int(x) for x in a.push.split(",")]:
            for pull in [int(x) for x in a.pull.split(",")]:
                so.push_ctas, so.pull_ctas = push, pull
                times = []
                for it in range(a.iters + 2):
                    if a.dist:
                        dist.barrier()
                    torch.cuda.synchronize()
                    r = so.run()
                    t = torch.tensor([r.kernel_ms], device="cuda")
                    if a.dist:
                        dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    if it >= 2:
                        times.append(t.item())
                best = min(times)
                med = sorted(times)[len(times) // 2]
                rec = {"tile": tile, "chunk": chunk, "window": window, "wide": wide, "push": push, "pull": pull, "ms_best": round(best, 3),
                       "ms_med": round(med, 3), "agg_GBps": round(R * M / (med * 1e-3) / 1e9, 1),
                       "nvlink_frac": round(M / (900e9 * med * 1e-3), 4),
                       "pcie64_frac": round(M / (64e9 * med * 1e-3), 4)}
                results.append(rec)
                if rank == 0:
                    print(json.dumps(rec), flush=True)
        if a.timeline:
            rows = {node: so.arrivals(node) for node in so.cluster.exec_nodes}
            allr = [None] * (dist.get_world_size() if a.dist else 1)
            if a.dist:
                dist.all_gather_object(allr, rows)
            else:
                allr = [rows]
            if rank == 0:
                merged = {}
                for r in allr:
                    merged.update({str(k): v for k, v in r.items()})
                json.dump({"arrivals_ns": merged, "lines": plan.lines(),
                           "block_bytes": plan.layout.block_lengths}, open(a.timeline, "w"))
        if a.verify:
            ref = so.checksums(plan.sources[-1]) if not a.host else None
            for node in so.cluster.exec_nodes:
                cs = so.checksums(node)
                if ref is not None and cs != ref:
                    print("CHECKSUM MISMATCH at node", node, flush=True)
            if rank == 0:
                print("verify done", flush=True)
        if a.dist:
            dist.barrier()
        so.close()
    if rank == 0:
        print(json.dumps({"config": a.config, "n": a.nodes, "k": a.sources, "b": a.blocks, "host": a.host, "M": M,
                          "receivers": R, "steps": plan.schedule.step_count}))
    if a.dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
