"""N > 1 host logic on CPU with a world_size-2 gloo group (no GPU):
every rank derives the identical plan, and the per-rank op lists (the
host-side mirror of the engine's op assignment, push and pull directions)
partition the schedule's transfer set exactly once."""
import os
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, tmp, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_09922_b200 import scaleout as SO
        for direction in (0, 1):
            for n_gpu, k, b, host in [(2, 1, 4, False), (2, 1, 4, True), (2, 2, 4, True)]:
                if k >= n_gpu + int(host):
                    continue
                plan = SO.plan_scale_out("tiny", n_gpu + int(host), k=k, block_count=b, host_source=host)
                mine = plan.lines()
                everyone = [None] * world
                dist.all_gather_object(everyone, mine)
                assert all(x == mine for x in everyone)          # identical plans on every rank
                node = rank + (1 if host else 0)
                ops = SO.node_ops(plan, node, direction)
                allops = [None] * world
                dist.all_gather_object(allops, ops)
                if rank == 0:
                    union = sorted(o[:4] for lst in allops for o in lst)
                    # every transfer has exactly one GPU executor (host-sourced ones are pulled)
                    want = sorted(tuple(int(v) for v in ln.split(",")) for ln in mine)
                    assert union == want
                    results.append((direction, n_gpu, k, b, host, len(union)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_plan_partition():
    port = 29000 + os.getpid() % 1000
    with tempfile.TemporaryDirectory() as tmp:
        mgr = mp.get_context("spawn").Manager()
        results = mgr.list()
        mp.spawn(_worker, args=(2, port, tmp, results), nprocs=2, join=True)
        assert len(results) == 6


def test_node_ops_cover_schedule_single_process():
    from paper_2502_09922_b200 import scaleout as SO
    for n, k, b, host in [(8, 1, 16, False), (9, 1, 16, True), (8, 2, 16, False), (5, 2, 8, True)]:
        plan = SO.plan_scale_out("tiny", n, k=k, block_count=min(b, 4), host_source=host)
        want = sorted(tuple(int(v) for v in ln.split(",")) for ln in plan.lines())
        for direction in (0, 1):
            got = sorted(o[:4] for node in range(n) for o in SO.node_ops(plan, node, direction))
            assert got == want
            for node in range(n):
                steps = [o[0] for o in SO.node_ops(plan, node, direction)]
                assert steps == sorted(steps)
