"""Execute-while-load serving benchmark (single process driving N GPUs).

  python tools/serve_bench.py --gpus 4 [--model llama3-8b] [--k 2] [--requests 16]

GPU nodes 0..k-1 hold the model (sources); the rest are cold receivers.  At
t = 0 the λPipe multicast starts and a burst of requests arrives (1 ms apart,
prompt 128 / output 32 tokens: the reference defaults, workload.py:126-127);
only cold capacity (pipelines, then post-switch local replicas) serves them.
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # see paper_2502_09922_b200/__init__.py

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run_serving(n_gpus: int, model: str = "llama3-8b", k: int = 2, blocks: int = 16, requests: int = 16,
                prompt_len: int = 128, out_tokens: int = 32, spacing_s: float = 0.001, pull_ctas: int = 32,
                local_slots: int = 16, seed: int = 20250815, executor: str = "ce", outdir: str | None = None,
                node_devices: list | None = None, host_source: bool = False, pipeline_batch: int | None = None,
                pipeline_prefill_tokens: int | None = None):
    """host_source: the tier-driven plan (scaleout.plan_from_tiers) with GPU 0
    holding the model and the box's pinned host copy as the second source
    (k = 2): one sub-group is fed over PCIe, GPUs 1..n-1 are cold."""
    import numpy as np
    import torch

    from paper_2502_09922_b200 import engine as E
    from paper_2502_09922_b200 import scaleout as SO
    from paper_2502_09922_b200.serving import Server
    from paper_2502_09922_b200.workload import TraceRecord, aggregate, write_result

    # node_devices: schedule node i on GPU node_devices[i] (default one node per
    # GPU); e.g. 8 nodes on 4 GPUs exercises the 8-node plan on a 4-GPU box
    node_devices = list(node_devices) if node_devices else list(range(n_gpus))
    if host_source:
        tm = SO.box_tiers(model, blocks, gpu_resident=(0,), host_copy=True, host_id=n_gpus)
        tp = SO.plan_from_tiers(model, list(range(1, n_gpus)), tm, k=k, block_count=blocks, host_id=n_gpus)
        plan = tp.plan
        node_devices = [-1 if i in plan.host_nodes else n for i, n in enumerate(tp.ref_nodes)]
    else:
        plan = SO.plan_scale_out(model, len(node_devices), k=k, block_count=blocks)
    devs = sorted(set(d for d in node_devices if d >= 0))
    lay = plan.layout
    tile = SO.CE_TILE if executor == "ce" else 2 << 20
    cl = E.Cluster.devices(node_devices, lay.block_offsets, lay.block_lengths, lay.weights_bytes,
                           tile_bytes=tile)
    try:
        for s in plan.sources:
            E.load_source_image(cl, s, lay, seed)
        cl.set_schedule_all(plan.schedule, plan.sources)
        for d in devs:
            cl.per_device[d].configure(1, 0, 0, 16384, 3)
        graphs = not os.environ.get("LP_NO_GRAPHS")
        pb = local_slots if pipeline_batch is None else pipeline_batch
        srv = Server(plan, cl, local_slots=local_slots, max_len=prompt_len + out_tokens + 8, use_graphs=graphs,
                     pipeline_batch=pb, pipeline_prefill_tokens=pipeline_prefill_tokens)
        rng = np.random.default_rng(seed)
        prompts = {f"r{i}": rng.integers(0, plan.config.vocab, prompt_len).tolist() for i in range(requests)}
        trace = [TraceRecord(f"r{i}", spacing_s * i, model, prompt_len, out_tokens) for i in range(requests)]
        streams = {d: torch.cuda.Stream(device=d) for d in devs}
        # warm-up (kernels, allocator, tensor maps): a tiny burst on a second epoch is not needed;
        # run one short pass first and report the second
        srv.run(trace[:2], prompts, streams, pull_ctas=pull_ctas, executor=executor)
        srv2 = Server(plan, cl, local_slots=local_slots, max_len=prompt_len + out_tokens + 8, use_graphs=graphs,
                      pipeline_batch=pb, pipeline_prefill_tokens=pipeline_prefill_tokens)
        ev = srv2.run(trace, prompts, streams, pull_ctas=pull_ctas, executor=executor)
        rep = aggregate(ev, "lambda_scale")
        if outdir:   # the reference's result files: `blockcast report <outdir>` re-aggregates them
            write_result(outdir, "lambda_scale", ev, rep)
        first_full = min(srv2.block_complete_s.values()) if srv2.block_complete_s else None
        all_full = max(srv2.block_complete_s.values()) if srv2.block_complete_s else None
        t_switch = next((e.time_s for e in ev if e.kind == "mode_switch"), None)
        pipe_tokens = sum(1 for e in ev if e.kind == "token_emitted" and (t_switch is None or e.time_s < t_switch))
        busy = [x for x in rep.throughput_timeline if x[1] > 0]
        if os.environ.get("LP_SERVE_PROFILE"):
            import time as _t
            for n, u in srv2.local_units.items():
                if u.graph is None:
                    continue
                d = u.stages[0].device
                with torch.cuda.device(d):
                    torch.cuda.synchronize(d)
                    t0 = _t.perf_counter()
                    for _ in range(5):
                        u.graph.graph.replay()
                    torch.cuda.synchronize(d)
                    print(f"replay node {n} dev {d}: {(_t.perf_counter() - t0) / 5 * 1e3:.2f} ms", file=sys.stderr)
            for row in srv2.profile_detail or []:
                print("detail %s unit=%d cap=%d %.4f s" % row, file=sys.stderr)
            for row in srv2.profile:
                print("iter t=%.4f enq=%.4f dev=%.4f tokens=%d batches=%d" % row, file=sys.stderr)
        return {
            "multicast_executor": executor + (" (push direction: one process drives every GPU, DESIGN §5.1)" if executor == "ce" else ""),
            "workload": f"{model} bf16, sources {plan.sources} (HOST positions {list(plan.host_nodes)}), "
                        f"receivers {plan.receivers}, b={blocks}, k={k}, pipeline capacity stages x {pb}, "
                        f"local replicas {local_slots} slots; "
                        f"{requests} requests x (prompt {prompt_len}, out {out_tokens}), {spacing_s * 1e3:.0f} ms apart at t=0",
            "pipelines": [[(st.node, st.block_lo, st.block_hi) for st in ep.stages] for ep in plan.pipelines],
            "pipeline_activation_s": sorted(srv2.activation_s.values()),
            "first_token_s": rep.first_token_s, "first_receiver_full_model_s": first_full,
            "all_receivers_full_s": all_full, "mode_switch_s": t_switch,
            "tokens_before_switch": pipe_tokens,
            "first_token_before_any_full_replica": (rep.first_token_s is not None and first_full is not None
                                                    and rep.first_token_s < first_full),
            "ttft_p50_s": rep.ttft_p50, "ttft_p90_s": rep.ttft_p90, "ttft_p99_s": rep.ttft_p99,
            "tokens_total": rep.total_tokens, "end_s": rep.end_s,
            "tokens_per_s": rep.total_tokens / rep.end_s if rep.end_s else None,
            "peak_window_tokens_per_s": max((x[1] for x in busy), default=0.0),
            "requests_completed": rep.requests_completed,
        }
    finally:
        cl.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--blocks", type=int, default=16)
    ap.add_argument("--requests", type=int, default=16)
    ap.add_argument("--out-tokens", type=int, default=32)
    ap.add_argument("--executor", default="ce")
    ap.add_argument("--pull-ctas", type=int, default=32)
    ap.add_argument("--outdir", default=None, help="write the reference's result files (cli.py:268-281) here")
    ap.add_argument("--node-devices", default="", help="comma list: GPU of each schedule node (default 0..gpus-1)")
    ap.add_argument("--host-source", action="store_true", help="GPU 0 + the pinned host copy as the k = 2 sources")
    ap.add_argument("--pipeline-batch", type=int, default=None,
                    help="requests per pipeline slot (default = local slots; 1 = the reference's capacity)")
    ap.add_argument("--pipeline-prefill-tokens", type=int, default=None,
                    help="prompt tokens one pipeline pass prefills (default: serving.Server's FLOP budget)")
    a = ap.parse_args()
    print(json.dumps(run_serving(a.gpus, a.model, a.k, a.blocks, a.requests, out_tokens=a.out_tokens,
                                 executor=a.executor, pull_ctas=a.pull_ctas, outdir=a.outdir,
                                 node_devices=[int(x) for x in a.node_devices.split(",")] if a.node_devices else None,
                                 host_source=a.host_source, pipeline_batch=a.pipeline_batch,
                                 pipeline_prefill_tokens=a.pipeline_prefill_tokens)))
