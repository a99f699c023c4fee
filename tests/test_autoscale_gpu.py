"""Reactive autoscaling with repeated λPipe scale-outs (config C5 machinery)
on one GPU (three nodes emulated on cuda:0): a burst makes the reference
autoscaler add replicas by multicast from the hot node, idle replicas are
released after the keep-alive, every request completes and its tokens equal
the fp32 oracle's greedy continuation (margin-gated)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_autoscale_burst_tiny():
    from oracle import dataplane as D
    from oracle import llama as OL
    from paper_2502_09922_b200.autoscaler import AutoscaleServer
    from paper_2502_09922_b200.cluster import AutoscalePolicy
    from paper_2502_09922_b200.workload import TraceRecord, aggregate

    policy = AutoscalePolicy(threshold_hi=1.0, keep_alive_s=0.3, min_replicas=1, capacity_per_replica=2,
                             eval_interval_s=0.01)
    srv = AutoscaleServer("tiny", [0, 0, 0], block_count=4, k=1, hot=(0,), policy=policy, local_slots=2,
                          max_len=64, seed=7)
    try:
        rng = np.random.default_rng(3)
        trace = [TraceRecord(f"r{i}", 0.0, "tiny", 12, 12) for i in range(24)]
        trace += [TraceRecord(f"s{i}", 1.5, "tiny", 12, 12) for i in range(12)]
        prompts = {r.request_id: rng.integers(0, srv.cfg.vocab, r.prompt_tokens).tolist() for r in trace}
        ev = srv.run(trace, prompts, timeout_s=60)
        kinds = [e.kind for e in ev]
        rep = aggregate(ev, "t")
        assert rep.requests_completed == len(trace)
        assert kinds.count("scale_out") >= 1 and kinds.count("mode_switch") >= 1, srv.decisions[:20]
        assert kinds.count("scale_in") >= 1
        W = OL.weights(srv.lay, D.fill_image(srv.lay, 7))
        for rid in ("r0", "r20", "s3"):
            ref, margins = OL.greedy(srv.cfg, W, prompts[rid], 12)
            got = srv.requests[rid].out
            for i, (a, b) in enumerate(zip(got, ref)):
                if margins[i] < 0.16:
                    break
                assert a == b, (rid, got, ref)
    finally:
        srv.close()
