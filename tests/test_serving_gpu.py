"""Execute-while-load serving on one GPU (all nodes emulated on cuda:0):
pipelines over partial replicas serve, mode switch moves requests to local
replicas with KV recompute, and every generated token — the pipelined ones
before the switch and the local ones after it — equals the oracle's greedy
continuation at every position (committed prompts, tests/parity.py): i.e.
pipelined, switched and local execution produce the same model outputs."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pipeline_batch,prefill_tokens", [(1, 256), (2, 256), (2, 1)])
def test_execute_while_load_tiny_matches_oracle(pipeline_batch, prefill_tokens):
    """prefill_tokens = 1: one prefill per pipeline pass, the other admitted
    requests wait in their slots while the first one decodes."""
    import torch
    from paper_2502_09922_b200 import engine as E
    from paper_2502_09922_b200 import scaleout as SO
    from paper_2502_09922_b200.serving import Server
    from paper_2502_09922_b200.workload import TraceRecord, aggregate

    plan = SO.plan_scale_out("tiny", 4, k=2, block_count=4)
    assert len(plan.pipelines) == 1 and len(plan.pipelines[0].stages) == 2
    lay = plan.layout
    cl = E.Cluster.devices([0, 0, 0, 0], lay.block_offsets, lay.block_lengths, lay.weights_bytes,
                           tile_bytes=64 * 1024)
    try:
        for s in plan.sources:
            E.load_source_image(cl, s, lay, 7)
        cl.set_schedule_all(plan.schedule, plan.sources)
        srv = Server(plan, cl, local_slots=4, max_len=64, switch_hold_tokens=6, pipeline_batch=pipeline_batch,
                     pipeline_prefill_tokens=prefill_tokens)
        assert srv.units[0].slots == 2 * pipeline_batch
        from parity import assert_tokens, doc
        es = {f"r{i}": e for i, e in enumerate(e for e in doc()["prompts"] if len(e["prompt"]) in (10, 11, 12))}
        prompts = {rid: e["prompt"] for rid, e in es.items()}
        trace = [TraceRecord(rid, 0.0, "tiny", len(p), 16) for rid, p in prompts.items()]
        ev = srv.run(trace, prompts, {0: torch.cuda.Stream(device=0)}, pull_ctas=4)
        kinds = [e.kind for e in ev]
        assert "mode_switch" in kinds
        # tokens were served by the pipeline unit before the switch and by
        # the local replicas after it
        first_switch = kinds.index("mode_switch")
        pre = sum(e.kind == "token_emitted" for e in ev[:first_switch])
        post = sum(e.kind == "token_emitted" for e in ev[first_switch:])
        assert pre >= 6 and post >= 6, (pre, post)
        rep = aggregate(ev, "t")
        assert rep.requests_completed == 3 and rep.total_tokens == 48
        compared = sum(assert_tokens(r.out, es[rid], what=f"serving {rid}") for rid, r in srv.requests.items())
        assert compared == 48
        # receivers hold the full image byte-exactly after the run
        want = E.block_checksums(cl.node(0).image, lay.block_offsets, lay.block_lengths)
        for n in plan.receivers:
            assert E.block_checksums(cl.node(n).image, lay.block_offsets, lay.block_lengths) == want
    finally:
        cl.close()
