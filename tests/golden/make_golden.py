"""Dump golden fixtures from the reference planner (run HERE only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ``blockcast`` in place from ``/root/reference/pkg/src`` (read-only,
never copied) and writes JSON fixtures next to this script.  The GPU box
never runs this file; tests read the committed JSON only.

Fixtures:
  schedules.json   full schedule / pipeline lines, summaries, warnings for the
                   SURVEY.md Appendix-B grid + small cases (sources = nodes[:k]
                   as cli.py:308-309)
  sweep.json       sha256[:16] of schedule and pipeline lines over a wide
                   (n, k, b) grid and the reference's seed-20250815 random
                   grid (test_acceptance.py:56-70), plus 1000 more seeded cases
  plans.json       partition_blocks / select_block_count / predicted_transfer_s
  misc.json        k_way_orders, partition_subgroups, validate_schedule on
                   tampered schedules, startup_plan, pack_layout, plan_2d_schedule,
                   plan_mode_switch, autoscale, transfer_step_time, aggregate,
                   synth_burst (config C5 trace)
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from blockcast import modelmgr, pipeline as P, simengine as S, workload as W  # noqa: E402
from blockcast.multicast import (ModelSpec, MulticastSchedule, SubGroup, Transfer,  # noqa: E402
                                 attach_orders, build_binomial_schedule, compose_schedule,
                                 k_way_orders, partition_blocks, partition_subgroups,
                                 predicted_transfer_s, schedule_summary, schedule_to_lines,
                                 select_block_count, validate_schedule)

HERE = os.path.dirname(os.path.abspath(__file__))
GB = 10 ** 9


def sha16(lines):
    return hashlib.sha256("\n".join(lines).encode()).hexdigest()[:16]


def plan_case(n, k, b, layers=None, size=26 * GB):
    layers = layers or max(b, 80)
    plan = partition_blocks(ModelSpec("m", size, layers), b)
    nodes = list(range(n))
    groups = attach_orders(partition_subgroups(nodes, nodes[:k]), k_way_orders(b, k))
    sched = compose_schedule(groups, plan)
    ordered = completion_ordered_groups_safe(groups, sched)
    pipes = P.generate_pipelines(ordered) if any(g.receivers for g in ordered) else []
    orders = [g.transfer_order for g in ordered]
    eps = [P.assign_blocks_to_stages(pn, orders, b, sched, i) for i, pn in enumerate(pipes)]
    return plan, groups, sched, ordered, pipes, eps


def completion_ordered_groups_safe(groups, sched):
    return P.completion_ordered_groups(groups, sched)


def full_record(n, k, b, layers=None, size=26 * GB):
    plan, groups, sched, ordered, pipes, eps = plan_case(n, k, b, layers, size)
    summ = schedule_summary(sched)
    return {
        "n": n, "k": k, "b": b,
        "groups": [[list(g.member_nodes), list(g.transfer_order)] for g in groups],
        "steps": [[[t.step, t.sender, t.receiver, t.block_id] for t in row] for row in sched.steps],
        "schedule_lines": schedule_to_lines(sched),
        "summary": {"step_count": summ["step_count"],
                    "completion_step": [[n_, s_] for n_, s_ in summ["completion_step"].items()]},
        "ordered": [list(g.member_nodes) for g in ordered],
        "pipes": [[list(x) for x in p] for p in pipes],
        "pipeline_lines": P.pipelines_to_lines(eps),
        "warnings": [list(ep.warnings) for ep in eps],
    }


def make_schedules():
    grid = [
        # SURVEY.md Appendix B (schedules are size-independent; layers cover b)
        (4, 1, 4), (4, 2, 4), (4, 1, 2), (4, 2, 2),
        (8, 1, 16), (8, 1, 32), (8, 2, 16), (8, 4, 16), (8, 1, 14),
        (2, 1, 16), (3, 1, 16), (5, 1, 16), (9, 1, 16), (9, 1, 40),
        (8, 1, 80), (8, 2, 80),
        # eyeball cases and small shapes
        (8, 1, 4), (3, 1, 3), (2, 1, 1), (3, 1, 1), (5, 2, 3), (6, 1, 5), (7, 3, 7),
        (9, 2, 16), (9, 4, 16), (9, 1, 32), (9, 2, 40), (16, 1, 8), (16, 4, 32),
        (4, 4, 4), (5, 4, 2), (6, 4, 3), (12, 5, 6), (17, 2, 9), (1, 1, 4),
        (8, 8, 4),
    ]
    recs = [full_record(n, k, b) for n, k, b in grid]
    # the reference's frozen two-source fixture (test_pipeline.py:18-60)
    plan = partition_blocks(ModelSpec("m0", 8 * GB, 8), 4)
    groups = attach_orders(partition_subgroups([1, 2, 3, 4, 5, 6, 7, 8], [1, 2]), k_way_orders(4, 2))
    sched = compose_schedule(groups, plan)
    ordered = P.completion_ordered_groups(groups, sched)
    pipes = P.generate_pipelines(ordered)
    eps = [P.assign_blocks_to_stages(pn, [g.transfer_order for g in ordered], 4, sched, i)
           for i, pn in enumerate(pipes)]
    two_src = {"schedule_lines": schedule_to_lines(sched),
               "ordered": [list(g.member_nodes) for g in ordered],
               "pipes": [[list(x) for x in p] for p in pipes],
               "pipeline_lines": P.pipelines_to_lines(eps)}
    # non-identity transfer orders through the builder directly
    custom = []
    for members, order in [((0, 1), (3, 1, 0, 2)), ((0, 1, 2, 3, 4), (2, 0, 1)),
                           ((5, 9, 2), (1, 0)), ((0, 1, 2, 3, 4, 5, 6), (4, 3, 2, 1, 0, 5))]:
        plan = partition_blocks(ModelSpec("m", 26 * GB, 80), max(order) + 1)
        steps = build_binomial_schedule(SubGroup(0, members, order), plan)
        custom.append({"members": list(members), "order": list(order),
                       "steps": [[[t.step, t.sender, t.receiver, t.block_id] for t in row]
                                 for row in steps]})
    return {"grid": recs, "two_source": two_src, "custom_orders": custom}


def make_sweep():
    out = {"grid": [], "random_20250815": [], "random_7": []}
    for n in range(1, 19):
        for k in range(1, min(5, n) + 1):
            for b in (1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 13, 16, 24, 32):
                _, _, sched, _, _, eps = plan_case(n, k, b)
                out["grid"].append([n, k, b, sched.step_count,
                                    sha16(schedule_to_lines(sched)), sha16(P.pipelines_to_lines(eps))])
    rng = random.Random(20250815)
    for _ in range(1000):
        n = rng.randint(2, 16)
        k = rng.randint(1, min(4, n - 1))
        b = rng.randint(1, 32)
        _, _, sched, _, _, eps = plan_case(n, k, b)
        out["random_20250815"].append([n, k, b, sched.step_count, sha16(schedule_to_lines(sched)),
                                       sha16(P.pipelines_to_lines(eps))])
    rng = random.Random(7)
    for _ in range(600):
        n = rng.randint(2, 24)
        k = rng.randint(1, min(6, n - 1))
        b = rng.randint(1, 64)
        _, _, sched, _, _, eps = plan_case(n, k, b)
        out["random_7"].append([n, k, b, sched.step_count, sha16(schedule_to_lines(sched)),
                                sha16(P.pipelines_to_lines(eps))])
    return out


MODELS = {  # SURVEY.md §8 config table (bf16 bytes)
    "C1_tiny": (38_600_000, 4), "C2_llama3_8b": (16_060_522_496, 32),
    "C3_llama2_13b": (26_031_728_640, 40), "C4_llama3_70b": (141_107_412_992, 80),
    "C5_llama2_7b": (13_476_831_232, 32), "ref_13b": (26 * GB, 80),
}


def make_plans():
    parts = []
    for name, (size, layers) in MODELS.items():
        for b in sorted({1, 2, 3, 4, 7, 8, 14, 16, min(32, layers), min(40, layers), layers}):
            if b > layers:
                continue
            plan = partition_blocks(ModelSpec(name, size, layers), b)
            parts.append([name, size, layers, b,
                          [[x.block_id, x.layer_lo, x.layer_hi, x.size_bytes] for x in plan.blocks]])
    rng = random.Random(11)
    for _ in range(200):
        layers = rng.randint(1, 400)
        b = rng.randint(1, layers)
        size = rng.randint(1, 10 ** 13)
        plan = partition_blocks(ModelSpec("r", size, layers), b)
        parts.append(["r", size, layers, b,
                      [[x.block_id, x.layer_lo, x.layer_hi, x.size_bytes] for x in plan.blocks]])
    elbows = []
    for name, (size, layers) in MODELS.items():
        for n in (1, 2, 3, 4, 5, 8, 9, 16):
            for ovh in (0.0, 1e-6, 1e-5, 1e-4, 5e-3):
                for bw in (50e9, 64e9, 400e9, 900e9):
                    for thr in (0.01, 0.05):
                        elbows.append([name, size, layers, n, ovh, bw, thr,
                                       select_block_count(ModelSpec(name, size, layers), n, ovh, bw, thr)])
    preds = []
    for size in (26 * GB, 16_060_522_496, 141_107_412_992):
        for b in (1, 2, 7, 16, 32, 80):
            for n in (1, 2, 3, 8, 9):
                for ovh in (0.0, 1e-5, 5e-3):
                    for bw in (50e9, 900e9):
                        preds.append([size, b, n, ovh, bw, predicted_transfer_s(size, b, n, ovh, bw)])
    return {"partition": parts, "select_block_count": elbows, "predicted": preds}


def make_misc():
    m = {}
    m["k_way_orders"] = [[b, k, [list(o) for o in k_way_orders(b, k)]]
                         for b in range(1, 21) for k in range(1, 7)]
    m["partition_subgroups"] = []
    for nodes, sources in [(list(range(8)), [0]), (list(range(8)), [0, 1]),
                           ([1, 2, 3, 4, 5, 6, 7, 8], [1, 2]), (list(range(1, 8)), [1, 2]),
                           (list(range(9)), [0, 3, 7]), ([5, 3, 9, 1], [9]), (list(range(12)), [11, 4, 2, 0])]:
        gs = partition_subgroups(nodes, sources)
        m["partition_subgroups"].append([nodes, sources, [[g.group_id, list(g.member_nodes)] for g in gs]])
    # tampered schedules -> violation lists (validate_schedule returns data)
    plan = partition_blocks(ModelSpec("m0", 26 * GB, 80), 4)
    groups = attach_orders(partition_subgroups(list(range(4)), [0]), k_way_orders(4, 1))
    sched = compose_schedule(groups, plan)
    cases = {}
    bad = [list(r) for r in sched.steps]
    bad[0] = bad[0] + [Transfer(0, 3, 2, 3)]
    cases["causality"] = MulticastSchedule(sched.groups, bad)
    cases["truncated"] = MulticastSchedule(sched.groups, sched.steps[:-1])
    bad = [list(r) for r in sched.steps]
    bad[1] = [Transfer(5, t.sender, t.receiver, t.block_id) for t in bad[1]]
    cases["step_index"] = MulticastSchedule(sched.groups, bad)
    g2 = attach_orders(partition_subgroups(list(range(8)), [0, 1]), k_way_orders(4, 2))
    s2 = compose_schedule(g2, plan)
    bad = [list(r) for r in s2.steps]
    bad[2] = bad[2] + [Transfer(2, 0, 7, 1)]
    cases["membership"] = MulticastSchedule(s2.groups, bad)
    bad = [list(r) for r in sched.steps]
    bad[2] = bad[2] + [Transfer(2, 0, 1, 0), Transfer(2, 0, 2, 1)]
    cases["degrees"] = MulticastSchedule(sched.groups, bad)
    padded = [list(r) for r in sched.steps] + [[], [Transfer(len(sched.steps) + 1, 0, 1, 0)]]
    cases["step_bound"] = MulticastSchedule(sched.groups, padded)
    cases["not_perm"] = MulticastSchedule((SubGroup(0, (0, 1), (0, 0, 1)),), [[Transfer(0, 0, 1, 0)]])
    m["violations"] = {}
    for name, sc in cases.items():
        m["violations"][name] = {
            "groups": [[g.group_id, list(g.member_nodes), list(g.transfer_order)] for g in sc.groups],
            "steps": [[[t.step, t.sender, t.receiver, t.block_id] for t in row] for row in sc.steps],
            "violations": [[v.kind, v.step, v.node, v.block_id, v.detail] for v in validate_schedule(sc)],
        }
    # startup_plan scenarios (modelmgr.py:109-141)
    sp = []
    for gpu_homes, mem_homes, ssd_homes, demand, kmax in [
            ([0], [1], [], list(range(8)), 2), ([], [0, 1, 2, 3], [], list(range(8)), 4),
            ([3], [3, 5], [], [0, 1, 2, 3], 1), ([], [], [2, 4], [0, 1], 1), ([], [], [], [0], 1),
            ([0, 1], [], [], list(range(8)), 4), ([], [6], list(range(8)), list(range(8)), 3)]:
        tiers = modelmgr.TierMap()
        for n in gpu_homes:
            tiers.ensure(n, "m").gpu_blocks = set(range(16))
        for n in mem_homes:
            tiers.ensure(n, "m").mem_blocks = set(range(16))
        for n in ssd_homes:
            tiers.ensure(n, "m").ssd = True
        tiers.ensure(7, "m").gpu_blocks = {0, 1}  # partial copy never counts
        try:
            r = modelmgr.startup_plan("m", 16, demand, tiers, kmax)
            res = {"classes": [[k_, v_] for k_, v_ in r.classes.items()], "sources": r.sources,
                   "bootstrap": r.bootstrap_node}
        except Exception as e:  # noqa: BLE001
            res = {"error": type(e).__name__}
        sp.append([gpu_homes, mem_homes, ssd_homes, demand, kmax, res, tiers.to_lines()])
    m["startup_plan"] = sp
    lay = []
    for name, (size, layers) in MODELS.items():
        for b in (1, 4, 16, min(layers, 80)):
            if b > layers:
                continue
            plan = partition_blocks(ModelSpec(name, size, layers), b)
            for ws, cap in ((0, None), (2 * GB, 180 * GB), (0, 80 * GB)):
                try:
                    L = modelmgr.pack_layout(plan, ws, cap)
                    res = {"regions": [[r.block_id, r.offset, r.length] for r in L.regions],
                           "act": L.activation_buffer_bytes, "staging": L.staging_buffer_bytes,
                           "total": L.total_bytes}
                except Exception as e:  # noqa: BLE001
                    res = {"error": type(e).__name__, "msg": str(e)}
                lay.append([name, size, layers, b, ws, cap, res])
    m["pack_layout"] = lay
    m["plan_2d"] = []
    for s_ in range(1, 6):
        for b_ in range(0, 8):
            t = P.plan_2d_schedule(s_, b_)
            m["plan_2d"].append([s_, b_, t.ticks, t.waiting, [t.utilization(i) for i in range(len(t.ticks))]])
    ep = P.ExecutionPipeline(0, (P.Stage(4, 0, 0, 1), P.Stage(7, 0, 2, 3), P.Stage(2, 1, 4, 5)))
    reqs = [(f"r{i}", (i * 7) % 11) for i in range(8)]
    ms = P.plan_mode_switch(ep, reqs, 0.5)
    m["mode_switch"] = [[a.request_id, a.node, a.recompute_cost_s] for a in ms.assignments]
    m["autoscale"] = []
    for pol in (S.AutoscalePolicy(), S.AutoscalePolicy(threshold_hi=1.0, capacity_per_replica=2, min_replicas=1)):
        for q in (0, 1, 3, 4, 9, 17, 40):
            for a in (0, 1, 2, 5):
                for idle in (0.0, 20.0):
                    d = S.autoscale(pol, q, a, idle)
                    m["autoscale"].append([pol.threshold_hi, pol.capacity_per_replica, pol.min_replicas,
                                           q, a, idle, d.scale_out, d.scale_in])
    m["baseline_schedule"] = []
    for strat in ("binary_tree", "broadcast_groups", "ssd_only", "ideal"):
        for n, b in ((1, 4), (2, 4), (3, 5), (8, 16), (9, 7), (5, 1)):
            plan = partition_blocks(ModelSpec("m", 26 * GB, 80), b)
            sc = S.baseline_schedule(strat, list(range(n)), plan, S.ClusterSpec())
            m["baseline_schedule"].append([strat, n, b, schedule_to_lines(sc), sc.max_send_degree,
                                           sc.enforce_step_bound, sc.initial_delay_s, sc.label,
                                           [[g.group_id, list(g.member_nodes)] for g in sc.groups],
                                           sc.step_count])
    m["transfer_step_time"] = []
    for size, b in ((26 * GB, 16), (16_060_522_496, 16), (141_107_412_992, 80)):
        plan = partition_blocks(ModelSpec("m", size, 80), b)
        g = attach_orders(partition_subgroups(list(range(8)), [0]), k_way_orders(b, 1))
        sc = compose_schedule(g, plan)
        for cl in (S.ClusterSpec(), S.ClusterSpec(nic_Bps=900e9, step_fixed_overhead_s=1e-5)):
            m["transfer_step_time"].append([size, b, cl.nic_Bps, cl.step_fixed_overhead_s,
                                            S.transfer_step_time(sc, plan, cl)])
    # aggregate over the reference simulator's own event stream (50-request burst)
    trace = [W.TraceRecord(f"r{i}", 0.001 * i, "m0", 128, 16) for i in range(50)]
    res = S.run(S.ClusterSpec(), [ModelSpec("m0", 26 * GB, 80)], "lambda_scale", trace,
                S.AutoscalePolicy(), block_count=16, k=2, initial_memory={"m0": [0, 1]})
    ev = [[e.time_s, e.kind, e.payload] for e in res.events]
    ev_json = json.loads(json.dumps(ev, default=lambda o: sorted(o) if isinstance(o, set) else str(o)))
    rep = res.report
    m["aggregate"] = {"events": ev_json, "report": {
        "requests_arrived": rep.requests_arrived, "requests_completed": rep.requests_completed,
        "requests_in_flight": rep.requests_in_flight, "total_tokens": rep.total_tokens,
        "ttft_samples": rep.ttft_samples, "ttft_p50": rep.ttft_p50, "ttft_p90": rep.ttft_p90,
        "ttft_p99": rep.ttft_p99, "throughput_timeline": rep.throughput_timeline,
        "gpu_seconds_cumulative": rep.gpu_seconds_cumulative, "first_token_s": rep.first_token_s,
        "ramp_first_serve_s": rep.ramp_first_serve_s, "end_s": rep.end_s},
        "horizon_report_end": W.aggregate(res.events, "h", horizon_s=50.0).end_s}
    tr = W.synth_burst(0.05, 6.0, [120.0, 800.0, 1500.0], 1800.0, seed=4,
                       spike_duration_s=60.0, output_tokens=(16, 32))
    m["synth_burst_c5"] = {"count": len(tr),
                           "sha16": sha16([f"{r.request_id},{r.arrival_s!r},{r.model_id},{r.prompt_tokens},{r.output_tokens}" for r in tr]),
                           "head": [[r.request_id, r.arrival_s, r.model_id, r.prompt_tokens, r.output_tokens] for r in tr[:5]]}
    tr2 = W.synth_burst(2.0, 10.0, [1.0], 5.0, seed=9, spike_duration_s=1.5, model_ids=("a", "b"),
                        prompt_tokens=(16, 64), output_tokens=(4, 9))
    m["synth_burst_small"] = [[r.request_id, r.arrival_s, r.model_id, r.prompt_tokens, r.output_tokens] for r in tr2]
    m["nearest_rank"] = [[xs, p, W.nearest_rank(xs, p)] for xs in ([3.0, 1.0, 2.0], [5.0] * 7 + [1.0, 9.0], list(map(float, range(100))))
                         for p in (1, 50, 90, 99, 100)]
    return m


def main():
    for name, fn in (("schedules", make_schedules), ("sweep", make_sweep),
                     ("plans", make_plans), ("misc", make_misc)):
        data = fn()
        with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print(name, os.path.getsize(os.path.join(HERE, f"{name}.json")), "bytes")


if __name__ == "__main__":
    main()
