"""Reactive autoscaling with repeated λPipe scale-outs (config C5 machinery)
on one GPU (three nodes emulated on cuda:0): a burst makes the reference
autoscaler add replicas by multicast from the hot node, idle replicas are
released after the keep-alive, every request completes and every token of
every request equals the oracle's greedy continuation (committed prompts,
tests/parity.py)."""
import pytest

pytestmark = pytest.mark.gpu


def test_autoscale_burst_tiny():
    from paper_2502_09922_b200.autoscaler import AutoscaleServer
    from paper_2502_09922_b200.cluster import AutoscalePolicy
    from paper_2502_09922_b200.workload import TraceRecord, aggregate

    policy = AutoscalePolicy(threshold_hi=1.0, keep_alive_s=0.3, min_replicas=1, capacity_per_replica=2,
                             eval_interval_s=0.01)
    srv = AutoscaleServer("tiny", [0, 0, 0], block_count=4, k=1, hot=(0,), policy=policy, local_slots=2,
                          max_len=64, seed=7)
    try:
        from parity import assert_tokens, entries
        ids = [f"r{i}" for i in range(24)] + [f"s{i}" for i in range(12)]
        es = dict(zip(ids, entries(len(ids), max_prompt=32)))
        prompts = {rid: e["prompt"] for rid, e in es.items()}
        trace = [TraceRecord(rid, 0.0 if rid[0] == "r" else 1.5, "tiny", len(prompts[rid]), 12) for rid in ids]
        ev = srv.run(trace, prompts, timeout_s=60)
        kinds = [e.kind for e in ev]
        rep = aggregate(ev, "t")
        assert rep.requests_completed == len(trace)
        assert kinds.count("scale_out") >= 1 and kinds.count("mode_switch") >= 1, srv.decisions[:20]
        assert kinds.count("scale_in") >= 1
        compared = sum(assert_tokens(srv.requests[rid].out, es[rid], 12, what=f"autoscale {rid}") for rid in ids)
        assert compared == 12 * len(ids)
    finally:
        srv.close()


def test_autoscale_from_host_copy_tiers():
    """No GPU holds the model at start, only the box's pinned host copy: the
    first scale-out's startup plan picks the host copy as its (MEMORY-tier)
    source; later ones use the then-hot GPUs first and the host copy after
    them (k = 2).  Every token of every request equals the oracle's."""
    from paper_2502_09922_b200.autoscaler import AutoscaleServer
    from paper_2502_09922_b200.cluster import AutoscalePolicy
    from paper_2502_09922_b200.workload import TraceRecord, aggregate
    from parity import assert_tokens, entries

    policy = AutoscalePolicy(threshold_hi=1.0, keep_alive_s=5.0, min_replicas=0, capacity_per_replica=2,
                             eval_interval_s=0.01)
    srv = AutoscaleServer("tiny", [0, 0, 0], block_count=4, k=2, hot=(), policy=policy, local_slots=2,
                          max_len=64, seed=7, host_copy=True)
    try:
        ids = [f"r{i}" for i in range(4)] + [f"s{i}" for i in range(12)]
        es = dict(zip(ids, entries(len(ids), max_prompt=32)))
        prompts = {rid: e["prompt"] for rid, e in es.items()}
        trace = [TraceRecord(rid, 0.0 if rid[0] == "r" else 0.8, "tiny", len(prompts[rid]), 12) for rid in ids]
        ev = srv.run(trace, prompts, timeout_s=60)
        outs = [e for e in ev if e.kind == "scale_out"]
        assert outs and outs[0].payload["sources"] == [srv.host_id], outs[0].payload
        assert all(c == "cold" for c in outs[0].payload["classes"].values())
        if len(outs) > 1:           # GPU copies rank ahead of the host copy
            assert outs[1].payload["sources"][0] != srv.host_id
        rep = aggregate(ev, "t")
        assert rep.requests_completed == len(trace)
        compared = sum(assert_tokens(srv.requests[rid].out, es[rid], 12, what=f"autoscale {rid}") for rid in ids)
        assert compared == 12 * len(ids)
    finally:
        srv.close()
