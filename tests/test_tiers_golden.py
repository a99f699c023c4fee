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
