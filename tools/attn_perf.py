"""Attention kernel timing (dev tool): decode rows (one per sequence, CUDA-core
path) and prefill tiles (tensor-core path), Llama-3-8B / 70B head shapes,
CUDA events over 200 warm launches."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import _native as N  # noqa: E402

lib = N.lib()
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def run(H, KV, hd, seqs, ctx, prefill, max_len=None):
    max_len = max_len or ctx + 8
    kc = (torch.randn(seqs, KV, max_len, hd, device="cuda") * 0.5).to(torch.bfloat16)
    vc = torch.randn(seqs, KV, max_len, hd, device="cuda").to(torch.float16)
    if prefill:   # every position of every sequence
        pos = torch.arange(ctx, dtype=torch.int32, device="cuda").repeat(seqs)
        seq = torch.arange(seqs, dtype=torch.int32, device="cuda").repeat_interleave(ctx)
    else:         # one new token per sequence at position ctx - 1
        pos = torch.full((seqs,), ctx - 1, dtype=torch.int32, device="cuda")
        seq = torch.arange(seqs, dtype=torch.int32, device="cuda")
    T = pos.numel()
    q = torch.randn(T, H, hd, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    f = lambda: N.check(lib.lp_attention(P(q), P(kc), P(vc), P(pos), P(seq), T, H, KV, hd, max_len,  # noqa: E731
                                         C.c_float(1 / math.sqrt(hd)), P(out), None))
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(int(os.environ.get("ATTN_ITERS", 200))):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / int(os.environ.get("ATTN_ITERS", 200)) * 1e3
    kv_bytes = (seqs * KV * ctx * hd * 2 * 2) if not prefill else seqs * KV * ctx * hd * 2 * 2
    flops = 4.0 * hd * H * seqs * ctx * (ctx + 1) / 2 if prefill else 4.0 * hd * H * seqs * ctx
    print(f"{'prefill' if prefill else 'decode '} H={H} KV={KV} seqs={seqs:3d} ctx={ctx:5d} max_len={max_len:5d} rows={T:6d}: "
          f"{us:8.1f} us  (K/V {kv_bytes / us / 1e3:7.1f} GB/s, {flops / us / 1e6:7.1f} TFLOP/s causal)", flush=True)


if len(sys.argv) > 1 and sys.argv[1] == "one":     # one decode config (ncu target): one SEQS CTX [MAX_LEN]
    run(32, 8, 128, int(sys.argv[2]), int(sys.argv[3]), False, int(sys.argv[4]) if len(sys.argv) > 4 else None)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "split":   # decode rows vs the cluster key split (cache capacity 2048)
    for H, KV in ((32, 8), (64, 8)):
        for seqs, ctx in ((16, 160), (16, 1024), (16, 2000), (8, 160), (8, 2000), (4, 2000), (32, 1024), (1, 160)):
            run(H, KV, 128, seqs, ctx, False, 2048)
    sys.exit(0)

if len(sys.argv) > 1 and sys.argv[1] == "pone":      # one prefill config (ncu target): pone H KV SEQS CTX
    run(int(sys.argv[2]), int(sys.argv[3]), 128, int(sys.argv[4]), int(sys.argv[5]), True)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "prefill":   # prefill only (LP_ATTN_TC=0/1 A/B)
    for H, KV in ((32, 8), (64, 8), (40, 40)):
        for seqs, ctx in ((16, 128), (8, 512), (1, 2048), (2, 4096)):
            run(H, KV, 128, seqs, ctx, True)
    sys.exit(0)

for H, KV in ((32, 8), (64, 8)):
    for seqs, ctx in ((16, 160), (16, 1024), (64, 160), (1, 4096), (4, 2048), (1, 32768)):
        run(H, KV, 128, seqs, ctx, False)
    for seqs, ctx in ((16, 128), (8, 512), (1, 2048)):
        run(H, KV, 128, seqs, ctx, True)
