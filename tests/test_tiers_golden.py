"""Tier-driven scale-out planning vs the reference simulator itself
(tests/golden/tiers.json, dumped by make_tiers_golden.py from
``simengine.run``): for the same initial residency and demand nodes,
``scaleout.plan_from_tiers`` yields the reference's hot/warm/cold classes,
startup sources and — relabelled to reference node ids — exactly the
schedule lines the simulator composed (simengine.py:442-467, :564-590)."""
import pytest

from paper_2502_09922_b200 import scaleout as SO
from paper_2502_09922_b200.image import LlamaConfig
from paper_2502_09922_b200.modelmgr import TierMap

from conftest import load_golden

CASES = load_golden("tiers")["cases"]
MODEL = LlamaConfig("m0", 32, 4096, 32, 8, 14336, 128256)   # 32 layers, as the golden's ModelSpec


@pytest.mark.parametrize("case", CASES, ids=[c["label"] for c in CASES])
def test_plan_from_tiers_matches_reference_simulator(case):
    b = case["b"]
    tm = TierMap()
    for n in range(case["node_count"]):
        tm.ensure(n, "m0").ssd = True                       # initial_ssd="all"
    for n in case["initial_memory"]:
        tm.ensure(n, "m0").mem_blocks = set(range(b))
    for n in case["initial_gpu"]:
        tm.ensure(n, "m0").gpu_blocks = set(range(b))
    so = case["scale_outs"][0]
    tp = SO.plan_from_tiers(MODEL, so["nodes"], tm, k=case["k"], block_count=b)
    assert {str(n): c for n, c in tp.startup.classes.items()} == so["classes"]
    assert tp.startup.sources == so["sources"]
    ref = case["compose"][0]
    assert [g["source"] for g in ref["groups"]] == tp.sources
    assert tp.ref_lines() == ref["lines"]
    assert tp.ref_nodes == [n for g in ref["groups"] for n in g["members"][:1]] + \
        [n for g in ref["groups"] for n in g["members"][1:]]
    # memory-only sources become HOST positions (the box's pinned host copy)
    for i, n in enumerate(tp.sources):
        st = tm.get(n, "m0")
        assert (i in tp.plan.host_nodes) == (len(st.gpu_blocks) < b and len(st.mem_blocks) >= b)


def test_box_tiers_host_copy_after_gpu_copies():
    tm = SO.box_tiers("tiny", 4, gpu_resident=(0,), host_copy=True, host_id=4)
    tp = SO.plan_from_tiers("tiny", [1, 2, 3], tm, k=2, block_count=4, host_id=4)
    assert tp.sources == [0, 4] and tp.cold == [1, 2, 3] and tp.plan.host_nodes == (1,)
    assert tp.plan.pipelines, "host-fed pipelines exist before any receiver holds the model"
    tm = SO.box_tiers("tiny", 4, gpu_resident=(), host_copy=True, host_id=4)
    tp = SO.plan_from_tiers("tiny", [0, 1, 2, 3], tm, k=2, block_count=4, host_id=4)
    assert tp.sources == [4] and tp.plan.host_nodes == (0,)


def test_warm_pipeline_plan_shapes():
    """Warm-node pipelines: warm node i loads chunk i of
    the k-way orders first; the warm pipeline's stage i holds chunk i and
    activates once every stage's chunk has landed; the combined execution
    schedule (λPipe rows + warm loads) passes the reference's validator."""
    from paper_2502_09922_b200.multicast import k_way_orders, validate_schedule
    tm = SO.box_tiers("tiny", 4, gpu_resident=(0,), host_copy=True, host_id=6, warm=(3, 4))
    tp = SO.warm_pipeline_plan(SO.plan_from_tiers("tiny", [1, 2, 3, 4, 5], tm, k=2, block_count=4, host_id=6),
                               "tiny", 4)
    p = tp.exec_plan
    assert tp.cold == [1, 2, 5] and tp.warm == [3, 4] and tp.sources == [0, 3]
    assert validate_schedule(p.schedule) == []
    warm_pos = [i for i, n in enumerate(tp.exec_ref_nodes) if n in tp.warm and i not in p.sources]
    orders = k_way_orders(4, 2)
    for w, order in zip(warm_pos, orders):
        got = [t.block_id for row in p.schedule.steps for t in row if t.receiver == w]
        assert got == list(order)
    ep = p.pipelines[-1]
    assert [st.node for st in ep.stages] == warm_pos
    assert [(st.block_lo, st.block_hi) for st in ep.stages] == [(0, 1), (2, 3)] and ep.activation_step == 1
    # the λPipe part is untouched
    assert p.pipelines[:len(tp.plan.pipelines)] == tp.plan.pipelines
