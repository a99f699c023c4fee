"""Config C5: bursty trace with repeated λPipe scale-outs (single process, N GPUs).

  python tools/burst_bench.py --gpus 4 [--compress 30]

The reference's own trace (test_acceptance.py:205-206): synth_burst(0.05, 6.0,
[120, 800, 1500], 1800, seed=4, spike_duration_s=60, output_tokens=(16, 32)),
1151 requests, replayed time-compressed by --compress (arrivals, spike length,
keep-alive and the autoscaler period all divided by it).  Llama-2-7B bf16,
one hot replica at t=0; the reference autoscaler adds replicas by λPipe
scale-out from hot GPUs (copy-engine multicast, k = 2) and releases them
after the keep-alive.
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # see paper_2502_09922_b200/__init__.py

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run_burst(n_gpus: int, compress: float = 30.0, model: str = "llama2-7b", k: int = 2, blocks: int = 16,
              local_slots: int = 16, limit_requests: int | None = None, seed: int = 4, outdir: str | None = None):
    import numpy as np

    from paper_2502_09922_b200.autoscaler import AutoscaleServer
    from paper_2502_09922_b200.cluster import AutoscalePolicy
    from paper_2502_09922_b200.workload import TraceRecord, aggregate, synth_burst, write_result

    raw = synth_burst(0.05, 6.0, [120.0, 800.0, 1500.0], 1800.0, seed=seed, spike_duration_s=60.0,
                      output_tokens=(16, 32))
    if limit_requests:
        raw = raw[:limit_requests]
    trace = [TraceRecord(r.request_id, r.arrival_s / compress, r.model_id, r.prompt_tokens, r.output_tokens)
             for r in raw]
    ref_policy = AutoscalePolicy()
    policy = AutoscalePolicy(threshold_hi=ref_policy.threshold_hi, keep_alive_s=ref_policy.keep_alive_s / compress,
                             min_replicas=1, capacity_per_replica=local_slots,
                             eval_interval_s=ref_policy.eval_interval_s / compress)
    srv = AutoscaleServer(model, list(range(n_gpus)), block_count=blocks, k=k, hot=(0,), policy=policy,
                          local_slots=local_slots, max_len=128 + 40)
    try:
        rng = np.random.default_rng(1)
        vocab = srv.cfg.vocab
        prompts = {r.request_id: rng.integers(0, vocab, r.prompt_tokens).tolist() for r in trace}
        ev = srv.run(trace, prompts)
        rep = aggregate(ev, "lambda_scale")
        if outdir:   # the reference's result files: `blockcast report <outdir>` re-aggregates them
            write_result(outdir, "lambda_scale", ev, rep)
        outs = sum(1 for e in ev if e.kind == "scale_out")
        busy = [x[1] for x in rep.throughput_timeline if x[1] > 0]
        return {"workload": f"{model} bf16, reference C5 trace ({len(trace)} requests) compressed {compress:g}x, "
                            f"{n_gpus} GPUs, 1 hot replica at t=0, k={k}, b={blocks}",
                "requests_completed": rep.requests_completed, "tokens": rep.total_tokens,
                "ttft_p50_s": rep.ttft_p50, "ttft_p90_s": rep.ttft_p90, "ttft_p99_s": rep.ttft_p99,
                "tokens_per_s_mean_busy": sum(busy) / len(busy) if busy else 0.0,
                "tokens_per_s_peak_window": max(busy) if busy else 0.0,
                "scale_outs": outs, "scale_ins": sum(1 for e in ev if e.kind == "scale_in"),
                "gpu_seconds": rep.gpu_seconds_cumulative, "end_s": rep.end_s}
    finally:
        srv.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--compress", type=float, default=30.0)
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--outdir", default=None, help="write the reference's result files (cli.py:268-281) here")
    a = ap.parse_args()
    print(json.dumps(run_burst(a.gpus, a.compress, limit_requests=a.limit or None, outdir=a.outdir)))
