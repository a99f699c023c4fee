"""Multi-GPU parity of the multicast engine, one process per GPU (torchrun,
NCCL rendezvous on 127.0.0.1): every executor and source tier delivers the
source's bytes to every rank.  Skipped on boxes with fewer than 2 GPUs."""
import json
import os
import subprocess
import sys

import pytest

from conftest import gpu_count

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(gpu_count() < 2, reason="needs >= 2 GPUs")
def test_distributed_multicast_all_executors():
    n = min(gpu_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + os.getpid() % 200),
           os.path.join(ROOT, "tools", "mc_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=280, cwd=ROOT)
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert res.returncode == 0 and line, res.stdout[-2000:] + res.stderr[-2000:]
    out = json.loads(line[-1])
    assert out["ok"] and len(out["results"]) == 5, out


@pytest.mark.skipif(gpu_count() < 3, reason="needs >= 3 GPUs for cross-device relays")
@pytest.mark.parametrize("executor", ["ce", "kernel"])
def test_single_process_relays(executor):
    """One process driving several GPUs (as serving and the autoscaler do)
    through a schedule whose relays wait on each other across devices: the
    copy-engine executor must not deadlock (it runs in the push direction in
    this mode) and every receiver ends byte-exact.  Run in a subprocess with
    a timeout, since a stream-level deadlock has no watchdog."""
    n = min(gpu_count(), 4)
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "relay_check.py"), str(n), "1", "4", executor],
                         capture_output=True, text=True, timeout=150, cwd=ROOT, env=env)
    assert res.returncode == 0 and "byte-exact" in res.stdout, res.stdout[-2000:] + res.stderr[-2000:]


@pytest.mark.skipif(gpu_count() < 2, reason="needs >= 2 GPUs")
def test_stage_split_across_gpus_handoff_matches_local():
    """A two-stage pipeline over two GPUs (layers 0-1 + vocab ops on cuda:0,
    layers 2-3 on cuda:1), hidden states handed over NVLink by lp_handoff (SM
    stores into the peer's buffer) both ways, gives the logits of one local
    executor (tolerance: split-K order) and the oracle's greedy tokens."""
    import numpy as np
    import torch
    from paper_2502_09922_b200 import _native as N
    from paper_2502_09922_b200 import engine as E
    from paper_2502_09922_b200 import image as I
    from paper_2502_09922_b200.llama import LlamaExecutor
    from parity import doc

    cfg = I.CONFIGS["tiny"]
    lay = I.build_layout(cfg, 4)
    for a, b in ((0, 1), (1, 0)):
        N.call("lp_enable_peer", a, b)
    p0, p1 = E.dev_malloc(0, lay.weights_bytes), E.dev_malloc(1, lay.weights_bytes)
    try:
        with E.on_device(0):
            E.fill_image(p0, lay, 7)
        with E.on_device(1):
            E.fill_image(p1, lay, 7)
        e = next(x for x in doc()["prompts"] if len(x["prompt"]) == 20)
        T = len(e["prompt"])

        def ints(v, dev):
            return torch.as_tensor(v, dtype=torch.int32, device=f"cuda:{dev}")

        with torch.cuda.device(0):
            local = LlamaExecutor(lay, p0, 0, max_seqs=1, max_len=64)
            _, ref = local.forward(tokens=ints(e["prompt"], 0), pos=ints(list(range(T)), 0), seq=ints([0] * T, 0))
        s0 = LlamaExecutor(lay, p0, 0, 0, 1, max_seqs=1, max_len=64)
        s1 = LlamaExecutor(lay, p1, 1, 2, 3, max_seqs=1, max_len=64, vocab_ops=False)

        def hop(x, src, dst):
            out = torch.empty(x.shape, dtype=x.dtype, device=f"cuda:{dst}")
            torch.cuda.synchronize(dst)
            with torch.cuda.device(src):
                N.check(N.lib().lp_handoff(N.C.c_void_p(x.data_ptr()), N.C.c_void_p(out.data_ptr()),
                                           x.numel() * x.element_size(), None, 0, None,
                                           N.C.c_void_p(torch.cuda.current_stream(src).cuda_stream)))
            torch.cuda.synchronize(src)
            return out

        toks, ctx = [], list(e["prompt"])
        pos0 = 0
        for step in range(len(e["greedy"])):
            new = ctx[pos0:]
            n = len(new)
            pos = list(range(pos0, pos0 + n))
            with torch.cuda.device(0):
                x, _ = s0.forward(tokens=ints(new, 0), pos=ints(pos, 0), seq=ints([0] * n, 0), want_logits=False)
            x = hop(x, 0, 1)
            with torch.cuda.device(1):
                x, _ = s1.forward(x=x, pos=ints(pos, 1), seq=ints([0] * n, 1), want_logits=False)
            x = hop(x, 1, 0)
            with torch.cuda.device(0):
                lg = s0.head(x[-1:].contiguous() if step else x)
                if step == 0:
                    err = (lg - ref).abs().max().item()
                    assert err < 1e-2, err
                    lg = lg[-1:]
                tok, _ = s0.greedy(lg)
            toks.append(int(tok.item()))
            pos0 += n
            ctx.append(toks[-1])
        assert toks == e["greedy"], (toks, e["greedy"])
    finally:
        E.dev_free(0, p0)
        E.dev_free(1, p1)


@pytest.mark.skipif(gpu_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("executor", ["kernel", "ce"])
def test_serving_two_gpus_token_parity(executor):
    """Execute-while-load with real cross-device pipelines: sources on both
    GPUs, receivers 2 (cuda:0) and 3 (cuda:1) form a two-stage pipeline whose
    hand-offs cross NVLink; pre-switch pipeline tokens and post-switch local
    tokens all equal the oracle's (every position)."""
    import torch
    from paper_2502_09922_b200 import engine as E
    from paper_2502_09922_b200 import scaleout as SO
    from paper_2502_09922_b200.serving import Server
    from paper_2502_09922_b200.workload import TraceRecord, aggregate
    from parity import assert_tokens, doc

    plan = SO.plan_scale_out("tiny", 4, k=2, block_count=4)
    lay = plan.layout
    cl = E.Cluster.devices([0, 1, 0, 1], lay.block_offsets, lay.block_lengths, lay.weights_bytes,
                           tile_bytes=64 * 1024)
    try:
        for s in plan.sources:
            E.load_source_image(cl, s, lay, 7)
        cl.set_schedule_all(plan.schedule, plan.sources)
        stage_devs = {cl.node_device(st.node) for ep in plan.pipelines for st in ep.stages}
        assert stage_devs == {0, 1}, "the pipeline must span both GPUs"
        srv = Server(plan, cl, local_slots=4, max_len=64, switch_hold_tokens=6)
        es = {f"r{i}": e for i, e in enumerate(e for e in doc()["prompts"] if len(e["prompt"]) in (8, 16, 32))}
        prompts = {rid: e["prompt"] for rid, e in es.items()}
        trace = [TraceRecord(rid, 0.0, "tiny", len(p), 16) for rid, p in prompts.items()]
        streams = {0: torch.cuda.Stream(device=0), 1: torch.cuda.Stream(device=1)}
        ev = srv.run(trace, prompts, streams, pull_ctas=4, executor=executor)
        kinds = [x.kind for x in ev]
        first_switch = kinds.index("mode_switch")
        assert sum(x.kind == "token_emitted" for x in ev[:first_switch]) >= 6
        rep = aggregate(ev, "t")
        assert rep.requests_completed == 3 and rep.total_tokens == 48
        compared = sum(assert_tokens(r.out, es[rid], what=f"2-GPU serving {rid}") for rid, r in srv.requests.items())
        assert compared == 48
        want = E.block_checksums(cl.node(0).image, lay.block_offsets, lay.block_lengths)
        for n in plan.receivers:
            with E.on_device(cl.node_device(n)):
                assert E.block_checksums(cl.node(n).image, lay.block_offsets, lay.block_lengths) == want
    finally:
        cl.close()
