"""GPU parity of the λPipe multicast engine against the oracle.

Every receiver's per-block checksum after the CUDA dataflow run must equal the
oracle's checksum of the CPU-generated source image, for schedules taken from
the drop-in planner (itself pinned to the reference).  Runs all nodes on one
GPU (Cluster.local) so it needs a single B200.
"""
import numpy as np
import pytest

from paper_2502_09922_b200 import image as I
from paper_2502_09922_b200 import multicast as M
from paper_2502_09922_b200 import engine as E

pytestmark = pytest.mark.gpu

CFG = I.LlamaConfig("mc-test", 8, 512, 8, 2, 1536, 8192)
SEED = 1234


@pytest.fixture(scope="module")
def oracle_sums():
    from oracle import dataplane as D
    cache = {}

    def get(b):
        if b not in cache:
            lay = I.build_layout(CFG, b)
            img = D.fill_image(lay, SEED)
            cache[b] = D.block_checksums(img, lay.block_offsets, lay.block_lengths)
        return cache[b]
    return get


def run_case(n, k, b, host, tile, push, pull, oracle_sums, epochs=2, push_mode=1, pull_mode=0, chunk=16384,
             direction=0, executor="kernel"):
    lay = I.build_layout(CFG, b)
    n_gpu = n - (1 if host else 0)
    cl = E.Cluster.local(n_gpu, lay.block_offsets, lay.block_lengths, lay.weights_bytes,
                         host_node=host, tile_bytes=tile)
    try:
        nodes = list(range(n))
        sources = nodes[:k]
        plan = M.partition_blocks(I.model_spec(CFG), b)
        groups = M.attach_orders(M.partition_subgroups(nodes, sources), M.k_way_orders(b, k))
        sched = M.compose_schedule(groups, plan)
        for s in sources:
            E.load_source_image(cl, s, lay, SEED)
        cl.set_schedule(sched, sources)
        cl.engine.configure(direction, push_mode, pull_mode, chunk)
        want = oracle_sums(b)
        for ep in range(epochs):
            for i in nodes[k:]:
                E.N.call("lp_memset", E.C.c_void_p(cl.node(i).image), 0, lay.weights_bytes, None)
            if executor == "ce":
                import torch
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream())   # CE streams must see the memsets above
                cl.launch_ce(1, after=ev)
                cl.join_ce(torch.cuda.current_stream())
                torch.cuda.synchronize()
            elif executor == "hybrid":
                import torch
                cl.engine.set_option("host_dma", 1)
                cl.launch_hybrid(torch.cuda.current_stream(), push_ctas=push, pull_ctas=pull)
                cl.wait(torch.cuda.current_stream().cuda_stream)
            else:
                cl.launch(push_ctas=push, pull_ctas=pull)
                cl.wait()
            for i in nodes:
                if cl.node(i).kind != E.LP_NODE_GPU:
                    continue
                got = E.block_checksums(cl.node(i).image, lay.block_offsets, lay.block_lengths)
                assert got == want, (n, k, b, host, ep, i)
            for i in nodes[k:]:
                assert all(cl.engine.complete(i, cl.epoch))
                if executor == "kernel":      # copy-engine ops record no arrival timestamps
                    arr = cl.engine.arrivals_ns(i)
                    assert all(a > 0 for a in arr)
    finally:
        cl.close()


@pytest.mark.parametrize("n,k,b,host,tile,push,pull", [
    (4, 1, 4, False, 512 * 1024, 8, 0),
    (8, 1, 8, False, 256 * 1024, 8, 0),
    (8, 2, 8, False, 512 * 1024, 8, 0),
    (8, 4, 8, False, 64 * 1024, 4, 0),
    (5, 1, 1, False, 512 * 1024, 8, 0),
    (2, 1, 8, True, 512 * 1024, 4, 8),
    (5, 1, 8, True, 256 * 1024, 4, 4),
    (9, 1, 8, True, 512 * 1024, 4, 4),
    (9, 2, 8, True, 512 * 1024, 4, 4),   # host + GPU source mix (k=2)
    (3, 1, 3, False, 4096, 2, 0),
])
@pytest.mark.parametrize("direction,push_mode,pull_mode", [(0, 0, 0), (0, 1, 0), (0, 1, 1), (1, 0, 0), (1, 0, 1)])
def test_multicast_delivers_source_bytes(n, k, b, host, tile, push, pull, direction, push_mode, pull_mode,
                                         oracle_sums):
    if direction == 0 and pull_mode == 1 and not host:
        pytest.skip("pull mode only matters with a host source")
    chunk = min(16384, tile)
    if direction == 1:
        pull = max(pull, push)
    run_case(n, k, b, host, tile, push, pull, oracle_sums, push_mode=push_mode, pull_mode=pull_mode,
             chunk=chunk, direction=direction)


@pytest.mark.parametrize("n,k,b,host,tile", [(4, 1, 4, False, 1 << 20), (8, 2, 8, False, 1 << 20),
                                             (9, 1, 8, True, 2 << 20), (9, 2, 8, True, 1 << 20),
                                             (5, 1, 1, False, 4096)])
@pytest.mark.parametrize("direction", [0, 1])
def test_copy_engine_executor_delivers_source_bytes(n, k, b, host, tile, direction, oracle_sums):
    run_case(n, k, b, host, tile, 0, 1, oracle_sums, direction=direction, executor="ce", chunk=min(16384, tile))


@pytest.mark.parametrize("n,k,b,tile", [(2, 1, 8, 1 << 20), (3, 1, 8, 512 * 1024), (5, 1, 8, 1 << 20),
                                         (9, 1, 8, 2 << 20), (9, 2, 8, 1 << 20), (5, 1, 1, 4096)])
@pytest.mark.parametrize("direction", [0, 1])
def test_hybrid_executor_delivers_source_bytes(n, k, b, tile, direction, oracle_sums):
    """Host hop on the copy engines, NVLink relays in the kernel (host_dma)."""
    push, pull = (4, 0) if direction == 0 else (0, 8)
    run_case(n, k, b, True, tile, push, pull, oracle_sums, direction=direction, executor="hybrid",
             chunk=min(16384, tile))


def test_engine_rejects_bad_schedules():
    lay = I.build_layout(CFG, 4)
    cl = E.Cluster.local(3, lay.block_offsets, lay.block_lengths, lay.weights_bytes)
    try:
        with pytest.raises(E.NativeError):
            cl.set_schedule(["0,1,2,0"], [0])     # fine to set; rejected at compile
            cl.launch(push_ctas=2)
        cl.set_schedule(["0,0,1,0", "1,0,1,0"], [0])   # double delivery
        with pytest.raises(E.NativeError):
            cl.launch(push_ctas=2)
    finally:
        cl.close()
