"""Execute-while-load fed by a host-memory source:
the tier-driven plan (startup_plan: GPU copies first, then the box's pinned
host copy) with k = 2 multicasts from GPU node 0 AND the host copy, so one of
the two sub-groups is fed over PCIe; the λPipe pipeline built from it serves
tokens before the mode switch, the receivers end byte-exact, and every token
equals the oracle's greedy continuation (committed prompts, tests/parity.py).
All nodes emulated on cuda:0."""
import pytest

pytestmark = pytest.mark.gpu


def test_execute_while_load_gpu_plus_host_source_k2():
    import torch
    from paper_2502_09922_b200 import engine as E
    from paper_2502_09922_b200 import scaleout as SO
    from paper_2502_09922_b200.serving import Server
    from paper_2502_09922_b200.workload import TraceRecord, aggregate
    from parity import assert_tokens, doc

    tm = SO.box_tiers("tiny", 4, gpu_resident=(0,), host_copy=True, host_id=4)
    tp = SO.plan_from_tiers("tiny", [1, 2, 3], tm, k=2, block_count=4, host_id=4)
    assert tp.sources == [0, 4] and tp.plan.host_nodes == (1,)
    assert tp.plan.pipelines
    so = SO.TieredScaleOut(tp, node_devices={0: 0, 1: 0, 2: 0, 3: 0}, seed=7, tile_bytes=64 * 1024)
    try:
        so.load_sources()
        assert so.cluster.node(1).kind == E.LP_NODE_HOST
        assert so.plan is tp.plan or so.plan.pipelines == tp.plan.pipelines   # no warm nodes here
        srv = Server(so.plan, so.cluster, local_slots=4, max_len=64, switch_hold_tokens=6)
        es = {f"r{i}": e for i, e in enumerate(e for e in doc()["prompts"] if len(e["prompt"]) in (13, 14, 15))}
        prompts = {rid: e["prompt"] for rid, e in es.items()}
        trace = [TraceRecord(rid, 0.0, "tiny", len(p), 16) for rid, p in prompts.items()]
        ev = srv.run(trace, prompts, {0: torch.cuda.Stream(device=0)}, pull_ctas=4)
        kinds = [e.kind for e in ev]
        first_switch = kinds.index("mode_switch")
        pre = sum(e.kind == "token_emitted" for e in ev[:first_switch])
        assert pre >= 6, pre                           # the host-fed pipeline served before the switch
        rep = aggregate(ev, "t")
        assert rep.requests_completed == 3 and rep.total_tokens == 48
        compared = sum(assert_tokens(r.out, es[rid], what=f"host-fed serving {rid}")
                       for rid, r in srv.requests.items())
        assert compared == 48
        want = E.block_checksums(so.cluster.node(0).image, tp.plan.layout.block_offsets,
                                 tp.plan.layout.block_lengths)
        got = so.checksums()
        assert sorted(got) == [1, 2, 3] and all(v == want for v in got.values())
    finally:
        so.close()


def test_scale_out_tiered_warm_and_cold():
    """scale_out(): hot node kept, warm node loaded from host memory over its
    own link, cold nodes fed by the GPU + host k = 2 multicast; every demand
    node ends byte-exact."""
    from oracle import dataplane as D
    from paper_2502_09922_b200 import scaleout as SO
    tm = SO.box_tiers("tiny", 4, gpu_resident=(0,), host_copy=True, host_id=5, warm=(2,))
    so, epoch = SO.scale_out("tiny", [0, 1, 2, 3, 4], tm, k=2, block_count=4, host_id=5,
                             node_devices={n: 0 for n in range(5)}, seed=7)
    try:
        tp = so.tp
        assert tp.hot == [0] and tp.warm == [2] and tp.cold == [1, 3, 4]
        assert tp.sources == [0, 2]                  # the warm node's host copy doubles as the 2nd source
        lay = tp.plan.layout
        want = D.block_checksums(D.fill_image(lay, 7), lay.block_offsets, lay.block_lengths)
        got = so.checksums()
        assert sorted(got) == [1, 2, 3, 4]
        assert all(v == want for v in got.values())
    finally:
        so.close()


def test_warm_nodes_pipeline_before_full_load():
    """Warm-node pipelines (SPEC.md:371, :416 — specified, not implemented by
    the reference simulator): two warm GPUs load from the host copy in k-way
    order (warm node i takes chunk i first) and form one pipeline among
    themselves that serves before either holds the whole model; every token
    equals the oracle's."""
    import torch
    from paper_2502_09922_b200 import scaleout as SO
    from paper_2502_09922_b200.serving import Server
    from paper_2502_09922_b200.workload import TraceRecord, aggregate
    from parity import assert_tokens, doc

    tm = SO.box_tiers("tiny", 4, gpu_resident=(), host_copy=True, host_id=4, warm=(1, 2))
    tp = SO.warm_pipeline_plan(SO.plan_from_tiers("tiny", [1, 2], tm, k=2, block_count=4, host_id=4), "tiny", 4)
    assert tp.cold == [] and tp.warm == [1, 2] and tp.plan is None
    ep = tp.exec_plan.pipelines[-1]
    assert [(st.block_lo, st.block_hi) for st in ep.stages] == [(0, 1), (2, 3)] and ep.activation_step == 1
    so = SO.TieredScaleOut(tp, node_devices={1: 0, 2: 0}, seed=7, tile_bytes=64 * 1024)
    try:
        so.load_sources()
        srv = Server(so.plan, so.cluster, local_slots=4, max_len=64, switch_hold_tokens=6)
        es = {f"r{i}": e for i, e in enumerate(e for e in doc()["prompts"] if len(e["prompt"]) in (9, 16, 20))}
        prompts = {rid: e["prompt"] for rid, e in es.items()}
        trace = [TraceRecord(rid, 0.0, "tiny", len(p), 16) for rid, p in prompts.items()]
        ev = srv.run(trace, prompts, {0: torch.cuda.Stream(device=0)}, pull_ctas=4)
        kinds = [x.kind for x in ev]
        first_switch = kinds.index("mode_switch")
        assert sum(x.kind == "token_emitted" for x in ev[:first_switch]) >= 6
        rep = aggregate(ev, "t")
        assert rep.requests_completed == 3 and rep.total_tokens == 48
        compared = sum(assert_tokens(r.out, es[rid], what=f"warm pipeline {rid}") for rid, r in srv.requests.items())
        assert compared == 48
        got = so.checksums()
        assert sorted(got) == [1, 2] and got[1] == got[2]
    finally:
        so.close()
