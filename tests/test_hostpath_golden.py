"""Host-side drop-in parity: residency, packing, 2D table, mode switch,
autoscale trigger, step-time model, metrics and the bursty trace generator —
all against fixtures dumped from the reference (tests/golden/make_golden.py)."""
import pytest

from paper_2502_09922_b200 import cluster as S
from paper_2502_09922_b200 import modelmgr
from paper_2502_09922_b200 import multicast as M
from paper_2502_09922_b200 import pipeline as P
from paper_2502_09922_b200 import workload as W
from paper_2502_09922_b200.errors import (CapacityError, IncompleteLogError, InvalidArgumentError,
                                          UnsatisfiableScalingError, UnsupportedConfigurationError)

GB = 10 ** 9


def test_startup_plan_matches(golden):
    for gpu_homes, mem_homes, ssd_homes, demand, kmax, want, lines in golden("misc")["startup_plan"]:
        tiers = modelmgr.TierMap()
        for n in gpu_homes:
            tiers.ensure(n, "m").gpu_blocks = set(range(16))
        for n in mem_homes:
            tiers.ensure(n, "m").mem_blocks = set(range(16))
        for n in ssd_homes:
            tiers.ensure(n, "m").ssd = True
        tiers.ensure(7, "m").gpu_blocks = {0, 1}
        if "error" in want:
            with pytest.raises(UnsatisfiableScalingError):
                modelmgr.startup_plan("m", 16, demand, tiers, kmax)
        else:
            sp = modelmgr.startup_plan("m", 16, demand, tiers, kmax)
            assert [[k, v] for k, v in sp.classes.items()] == want["classes"]
            assert sp.sources == want["sources"]
            assert sp.bootstrap_node == want["bootstrap"]
        assert tiers.to_lines() == lines


def test_pack_layout_matches(golden):
    for name, size, layers, b, ws, cap, want in golden("misc")["pack_layout"]:
        plan = M.partition_blocks(M.ModelSpec(name, size, layers), b)
        if "error" in want:
            with pytest.raises(CapacityError) as ei:
                modelmgr.pack_layout(plan, ws, cap)
            assert str(ei.value) == want["msg"]
        else:
            lay = modelmgr.pack_layout(plan, ws, cap)
            assert [[r.block_id, r.offset, r.length] for r in lay.regions] == want["regions"]
            assert (lay.activation_buffer_bytes, lay.staging_buffer_bytes, lay.total_bytes) == \
                (want["act"], want["staging"], want["total"])


def test_plan_2d_and_mode_switch_match(golden):
    misc = golden("misc")
    for s, b, ticks, waiting, util in misc["plan_2d"]:
        t = P.plan_2d_schedule(s, b)
        assert t.ticks == ticks and t.waiting == waiting
        assert [t.utilization(i) for i in range(len(t.ticks))] == util
    ep = P.ExecutionPipeline(0, (P.Stage(4, 0, 0, 1), P.Stage(7, 0, 2, 3), P.Stage(2, 1, 4, 5)))
    ms = P.plan_mode_switch(ep, [(f"r{i}", (i * 7) % 11) for i in range(8)], 0.5)
    assert [[a.request_id, a.node, a.recompute_cost_s] for a in ms.assignments] == misc["mode_switch"]
    with pytest.raises(InvalidArgumentError):
        P.plan_mode_switch(ep, [("x", -1)], 0.5)


def test_multi_gpu_strategy():
    m1 = M.ModelSpec("a", GB, 4)
    m4 = M.ModelSpec("b", GB, 4, gpus_per_replica=4)
    assert P.select_multi_gpu_strategy(m1, 8, 0) == P.CROSS_NODE_SINGLE_GPU
    assert P.select_multi_gpu_strategy(m1, 8, 3) == P.INTRA_NODE_REPLICATE
    assert P.select_multi_gpu_strategy(m4, 8, 0) == P.CROSS_NODE_MULTI_GPU
    with pytest.raises(UnsupportedConfigurationError):
        P.select_multi_gpu_strategy(m4, 2, 0)


def test_autoscale_and_step_time_match(golden):
    misc = golden("misc")
    for thr, cap, minr, q, a, idle, out, shrink in misc["autoscale"]:
        d = S.autoscale(S.AutoscalePolicy(threshold_hi=thr, capacity_per_replica=cap, min_replicas=minr),
                        q, a, idle)
        assert (d.scale_out, d.scale_in) == (out, shrink)
    for size, b, nic, ovh, want in misc["transfer_step_time"]:
        plan = M.partition_blocks(M.ModelSpec("m", size, 80), b)
        g = M.attach_orders(M.partition_subgroups(list(range(8)), [0]), M.k_way_orders(b, 1))
        sc = M.compose_schedule(g, plan)
        assert S.transfer_step_time(sc, plan, S.ClusterSpec(nic_Bps=nic, step_fixed_overhead_s=ovh)) == want


def test_aggregate_matches_reference_on_its_own_events(golden):
    agg = golden("misc")["aggregate"]
    events = [W.SimEvent(t, k, p) for t, k, p in agg["events"]]
    rep = W.aggregate(events, "lambda_scale", horizon_s=None)
    want = agg["report"]
    assert rep.requests_arrived == want["requests_arrived"]
    assert rep.requests_completed == want["requests_completed"]
    assert rep.total_tokens == want["total_tokens"]
    assert rep.ttft_samples == want["ttft_samples"]
    assert (rep.ttft_p50, rep.ttft_p90, rep.ttft_p99) == (want["ttft_p50"], want["ttft_p90"], want["ttft_p99"])
    assert [list(x) for x in rep.throughput_timeline] == want["throughput_timeline"]
    assert rep.gpu_seconds_cumulative == want["gpu_seconds_cumulative"]
    assert rep.first_token_s == want["first_token_s"]
    assert rep.ramp_first_serve_s == want["ramp_first_serve_s"]
    assert W.aggregate(events, "h", horizon_s=50.0).end_s == agg["horizon_report_end"]
    with pytest.raises(IncompleteLogError):
        W.aggregate([W.SimEvent(0.0, "request_arrival", {"request": "x"})])


def test_synth_burst_matches(golden):
    misc = golden("misc")
    tr = W.synth_burst(0.05, 6.0, [120.0, 800.0, 1500.0], 1800.0, seed=4, spike_duration_s=60.0,
                       output_tokens=(16, 32))
    assert len(tr) == misc["synth_burst_c5"]["count"] == 1151
    assert [[r.request_id, r.arrival_s, r.model_id, r.prompt_tokens, r.output_tokens]
            for r in tr[:5]] == misc["synth_burst_c5"]["head"]
    import hashlib
    s16 = hashlib.sha256("\n".join(f"{r.request_id},{r.arrival_s!r},{r.model_id},{r.prompt_tokens},"
                                   f"{r.output_tokens}" for r in tr).encode()).hexdigest()[:16]
    assert s16 == misc["synth_burst_c5"]["sha16"]
    tr2 = W.synth_burst(2.0, 10.0, [1.0], 5.0, seed=9, spike_duration_s=1.5, model_ids=("a", "b"),
                        prompt_tokens=(16, 64), output_tokens=(4, 9))
    assert [[r.request_id, r.arrival_s, r.model_id, r.prompt_tokens, r.output_tokens]
            for r in tr2] == misc["synth_burst_small"]
    for xs, p, want in misc["nearest_rank"]:
        assert W.nearest_rank(xs, p) == want


def test_baseline_schedules_match(golden):
    for strat, n, b, lines, deg, bound, delay, label, groups, steps in golden("misc")["baseline_schedule"]:
        plan = M.partition_blocks(M.ModelSpec("m", 26 * GB, 80), b)
        sc = S.baseline_schedule(strat, list(range(n)), plan, S.ClusterSpec())
        assert M.schedule_to_lines(sc) == lines, (strat, n, b)
        assert (sc.max_send_degree, sc.enforce_step_bound, sc.initial_delay_s, sc.label, sc.step_count) == \
            (deg, bound, delay, label, steps)
        assert [[g.group_id, list(g.member_nodes)] for g in sc.groups] == groups
    with pytest.raises(InvalidArgumentError):
        S.baseline_schedule("nope", [0, 1], M.partition_blocks(M.ModelSpec("m", GB, 4), 2), S.ClusterSpec())
