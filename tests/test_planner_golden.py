"""Planner parity: every output of the drop-in planner equals the reference's.

Fixtures were dumped from the reference itself (tests/golden/make_golden.py);
SURVEY.md Appendix B hashes are re-checked here too.
"""
import hashlib

import pytest

from paper_2502_09922_b200 import multicast as M
from paper_2502_09922_b200 import pipeline as P

GB = 10 ** 9


def sha16(lines):
    return hashlib.sha256("\n".join(lines).encode()).hexdigest()[:16]


def plan_case(n, k, b, layers=None, size=26 * GB):
    layers = layers or max(b, 80)
    plan = M.partition_blocks(M.ModelSpec("m", size, layers), b)
    nodes = list(range(n))
    groups = M.attach_orders(M.partition_subgroups(nodes, nodes[:k]), M.k_way_orders(b, k))
    sched = M.compose_schedule(groups, plan)
    ordered = P.completion_ordered_groups(groups, sched)
    pipes = P.generate_pipelines(ordered) if any(g.receivers for g in ordered) else []
    orders = [g.transfer_order for g in ordered]
    eps = [P.assign_blocks_to_stages(pn, orders, b, sched, i) for i, pn in enumerate(pipes)]
    return plan, groups, sched, ordered, pipes, eps


def test_full_schedules_match_reference(golden):
    for rec in golden("schedules")["grid"]:
        n, k, b = rec["n"], rec["k"], rec["b"]
        _, groups, sched, ordered, pipes, eps = plan_case(n, k, b)
        assert [[list(g.member_nodes), list(g.transfer_order)] for g in groups] == rec["groups"]
        steps = [[[t.step, t.sender, t.receiver, t.block_id] for t in row] for row in sched.steps]
        assert steps == rec["steps"], (n, k, b)          # including in-step order
        assert M.schedule_to_lines(sched) == rec["schedule_lines"]
        summ = M.schedule_summary(sched)
        assert summ["step_count"] == rec["summary"]["step_count"]
        assert [[a, c] for a, c in summ["completion_step"].items()] == rec["summary"]["completion_step"]
        assert [list(g.member_nodes) for g in ordered] == rec["ordered"]
        assert [[list(x) for x in p] for p in pipes] == rec["pipes"]
        assert P.pipelines_to_lines(eps) == rec["pipeline_lines"], (n, k, b)
        assert [list(ep.warnings) for ep in eps] == rec["warnings"]


def test_appendix_b_anchor_hashes():
    # SURVEY.md Appendix B (sources = nodes[:k])
    for n, k, b, steps, s16, p16 in [
            (8, 1, 16, 18, "534f3174b8377775", "65496538c2b49bbf"),
            (8, 2, 16, 17, "fdfe89aa10570ad6", "9ab8692375cfeeb5"),
            (8, 4, 16, 16, "a0055d46bb94b941", "ce30f8559f88e8d7"),
            (9, 1, 16, 20, "8778a59c79c2d462", "22a3da6394ecf253"),
            (8, 1, 80, 82, "fd8351e5650bc7e6", "4048d6e7b1381ea4"),
            (8, 2, 80, 81, "4080198c21156e5c", "53a8f58358bb63bc"),
            (4, 1, 2, 3, "045d6dad78364383", "86ce401ca2861d1f")]:
        _, _, sched, _, _, eps = plan_case(n, k, b)
        assert sched.step_count == steps
        assert sha16(M.schedule_to_lines(sched)) == s16
        assert sha16(P.pipelines_to_lines(eps)) == p16


@pytest.mark.parametrize("section", ["grid", "random_20250815", "random_7"])
def test_sweep_hashes_match_reference(golden, section):
    for n, k, b, steps, s16, p16 in golden("sweep")[section]:
        _, _, sched, _, _, eps = plan_case(n, k, b)
        assert sched.step_count == steps, (n, k, b)
        assert sha16(M.schedule_to_lines(sched)) == s16, (n, k, b)
        assert sha16(P.pipelines_to_lines(eps)) == p16, (n, k, b)


def test_two_source_fixture(golden):
    ref = golden("schedules")["two_source"]
    plan = M.partition_blocks(M.ModelSpec("m0", 8 * GB, 8), 4)
    groups = M.attach_orders(M.partition_subgroups([1, 2, 3, 4, 5, 6, 7, 8], [1, 2]), M.k_way_orders(4, 2))
    sched = M.compose_schedule(groups, plan)
    ordered = P.completion_ordered_groups(groups, sched)
    pipes = P.generate_pipelines(ordered)
    eps = [P.assign_blocks_to_stages(pn, [g.transfer_order for g in ordered], 4, sched, i)
           for i, pn in enumerate(pipes)]
    assert M.schedule_to_lines(sched) == ref["schedule_lines"]
    assert [list(g.member_nodes) for g in ordered] == ref["ordered"]
    assert pipes == [[tuple(x) for x in p] for p in ref["pipes"]]
    # the reference's own frozen lines (test_pipeline.py:46-60)
    assert P.pipelines_to_lines(eps) == ["0,0,4,0,0,1,2", "0,1,7,0,2,3,2", "1,0,5,0,0,1,2",
                                         "1,1,8,0,2,3,2", "2,0,3,0,0,1,3", "2,1,6,0,2,3,3"]
    assert P.pipelines_to_lines(eps) == ref["pipeline_lines"]


def test_custom_orders_through_builder(golden):
    for rec in golden("schedules")["custom_orders"]:
        order = tuple(rec["order"])
        plan = M.partition_blocks(M.ModelSpec("m", 26 * GB, 80), max(order) + 1)
        steps = M.build_binomial_schedule(M.SubGroup(0, tuple(rec["members"]), order), plan)
        assert [[[t.step, t.sender, t.receiver, t.block_id] for t in row] for row in steps] == rec["steps"]


def test_partition_blocks_match(golden):
    for name, size, layers, b, blocks in golden("plans")["partition"]:
        plan = M.partition_blocks(M.ModelSpec(name, size, layers), b)
        assert [[x.block_id, x.layer_lo, x.layer_hi, x.size_bytes] for x in plan.blocks] == blocks


def test_select_block_count_match(golden):
    for name, size, layers, n, ovh, bw, thr, want in golden("plans")["select_block_count"]:
        assert M.select_block_count(M.ModelSpec(name, size, layers), n, ovh, bw, thr) == want


def test_predicted_transfer_match(golden):
    for size, b, n, ovh, bw, want in golden("plans")["predicted"]:
        assert M.predicted_transfer_s(size, b, n, ovh, bw) == want   # bit-identical float


def test_k_way_and_subgroups_match(golden):
    misc = golden("misc")
    for b, k, orders in misc["k_way_orders"]:
        assert [list(o) for o in M.k_way_orders(b, k)] == orders
    for nodes, sources, groups in misc["partition_subgroups"]:
        got = M.partition_subgroups(nodes, sources)
        assert [[g.group_id, list(g.member_nodes)] for g in got] == groups


def test_validate_schedule_violations_match(golden):
    for name, case in golden("misc")["violations"].items():
        groups = tuple(M.SubGroup(g, tuple(m), tuple(o)) for g, m, o in case["groups"])
        steps = [[M.Transfer(*t) for t in row] for row in case["steps"]]
        got = M.validate_schedule(M.MulticastSchedule(groups, steps))
        assert [[v.kind, v.step, v.node, v.block_id, v.detail] for v in got] == case["violations"], name


def test_reference_quirks():
    # k=1 single-group pipeline with more stages than blocks: empty stage (SURVEY §0 finding 5)
    _, _, _, _, _, eps = plan_case(4, 1, 2)
    assert P.pipelines_to_lines(eps) == ["0,0,1,0,0,0,1", "0,1,2,0,1,1,1", "0,2,3,0,2,1,1"]
    # source re-sends its last block (finding 3): 1->8, b=4
    _, _, sched, _, _, _ = plan_case(8, 1, 4)
    src_blocks = [t.block_id for row in sched.steps for t in row if t.sender == 0]
    assert src_blocks == [0, 1, 2, 3, 3, 3]
