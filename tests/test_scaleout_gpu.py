"""GPU parity of the ``scale_out`` drop-in (plan + execute) for every executor,
with verify-as-it-lands: the per-block checksums the receivers compute WHILE
the blocks stream in (lp_mc_verify) must equal the oracle's checksums of the
CPU-generated source image, every epoch.  One GPU (nodes emulated on it)."""
import pytest

from paper_2502_09922_b200 import engine as E
from paper_2502_09922_b200 import scaleout as SO

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def want():
    from oracle import dataplane as D
    cache = {}

    def get(plan):
        lay = plan.layout
        key = (lay.weights_bytes, tuple(lay.block_lengths))
        if key not in cache:
            img = D.fill_image(lay, 0)
            cache[key] = D.block_checksums(img, lay.block_offsets, lay.block_lengths)
        return cache[key]
    return get


@pytest.mark.parametrize("n,k,b,host,executor,tile", [
    (2, 1, 4, True, "hybrid", 1 << 20),
    (3, 1, 4, True, "hybrid", 512 * 1024),
    (5, 1, 4, True, "hybrid", 1 << 20),
    (5, 2, 4, True, "hybrid", 1 << 20),
    (4, 1, 4, False, "kernel", 1 << 20),
    (4, 1, 4, False, "ce", 2 << 20),
    (3, 1, 4, True, "kernel", 1 << 20),
    (3, 1, 4, True, "ce", 1 << 20),
    (4, 2, 3, False, "kernel", 4096 * 16),
    (4, 1, 4, False, "split", 1 << 20),
    (5, 2, 4, False, "split", 64 * 1024),
    (5, 1, 4, True, "split", 1 << 20),
])
def test_scale_out_verifies_while_landing(n, k, b, host, executor, tile, want):
    plan = SO.plan_scale_out("tiny", n, k=k, block_count=b, host_source=host)
    so = SO.ScaleOut(plan, executor=executor, tile_bytes=tile, pull_ctas=8, push_ctas=0,
                     direction=1, copy_mode=0, verify=True, verify_ctas=8)
    try:
        so.load_sources()
        ref = want(plan)
        for _ in range(3):
            for node in plan.receivers:   # wipe receivers so stale bytes cannot pass
                E.N.call("lp_memset", E.C.c_void_p(so.cluster.node(node).image), 0,
                         plan.layout.weights_bytes, None)
            r = so.run()
            gpu_receivers = [x for x in plan.receivers if so.cluster.node(x).kind == E.LP_NODE_GPU]
            assert sorted(r.checksums) == gpu_receivers
            for node in gpu_receivers:
                assert r.checksums[node] == ref, (node, r.epoch)
                assert so.checksums(node) == ref
            # one checksum launch per received block, plus the executor's kernels
            assert r.launches == sum(len(so.cluster.engine.received_blocks(x)) for x in gpu_receivers) + \
                (0 if executor == "ce" else so.kernel_launches)
    finally:
        so.close()


def test_hybrid_is_the_host_policy():
    plan = SO.plan_scale_out("tiny", 3, k=1, block_count=4, host_source=True)
    assert SO.choose_executor(plan)[0] == "hybrid"
    plan = SO.plan_scale_out("tiny", 4, k=1, block_count=4)
    assert SO.choose_executor(plan)[0] == "ce"


@pytest.mark.parametrize("n,executor", [(3, "hybrid"), (5, "hybrid"), (5, "kernel"), (4, "ce"), (2, "hybrid")])
def test_sharded_host_load_verifies(n, executor, want):
    plan = SO.plan_scale_out("tiny", n, k=1, block_count=4, host_source=True, strategy="sharded_host")
    so = SO.ScaleOut(plan, executor=executor, tile_bytes=1 << 20, pull_ctas=8, push_ctas=0,
                     direction=1, copy_mode=0, verify=True, verify_ctas=8)
    try:
        so.load_sources()
        ref = want(plan)
        for _ in range(2):
            for node in plan.receivers:
                E.N.call("lp_memset", E.C.c_void_p(so.cluster.node(node).image), 0,
                         plan.layout.weights_bytes, None)
            r = so.run()
            assert sorted(r.checksums) == plan.receivers
            for node in plan.receivers:
                assert r.checksums[node] == ref
    finally:
        so.close()


@pytest.mark.parametrize("strategy", ["binary_tree", "broadcast_groups"])
@pytest.mark.parametrize("executor", ["kernel", "ce"])
def test_comparator_strategies_byte_exact(strategy, executor, want):
    """The reference's comparator schedules (simengine.py:106-151, golden in
    tests/test_hostpath_golden.py) executed by the same engine as λPipe —
    only the schedule differs — deliver the source's bytes to every node
    (5 emulated nodes on cuda:0, verify-as-it-lands sums == oracle)."""
    import dataclasses
    from paper_2502_09922_b200.cluster import b200_box, baseline_schedule
    plan = SO.plan_scale_out("tiny", 5, k=1, block_count=4)
    sched = baseline_schedule(strategy, plan.nodes, plan.layout.plan, b200_box(node_count=5))
    plan = dataclasses.replace(plan, schedule=sched, strategy=strategy, pipelines=[])
    so = SO.ScaleOut(plan, executor=executor, tile_bytes=1 << 20, pull_ctas=8, push_ctas=0,
                     direction=1, copy_mode=0, verify=True, verify_ctas=8)
    try:
        so.load_sources()
        ref = want(plan)
        for _ in range(2):
            for node in plan.receivers:
                E.N.call("lp_memset", E.C.c_void_p(so.cluster.node(node).image), 0,
                         plan.layout.weights_bytes, None)
            r = so.run()
            assert sorted(r.checksums) == plan.receivers
            for node in plan.receivers:
                assert r.checksums[node] == ref, (strategy, executor, node)
    finally:
        so.close()
