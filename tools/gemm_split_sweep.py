"""Split-K sweep for decode-shaped GEMMs (dev tool): weight-streaming GB/s per split."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import _native as N  # noqa: E402

P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
lib = N.lib()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(iters):
        flush.zero_()                      # evict L2: weights stream from HBM
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / iters


for T in (1, 8):
    for name, n, k in [("qkv", 6144, 4096), ("wo", 4096, 4096), ("gate_up_cat", 28672, 4096), ("down", 4096, 14336),
                       ("lm_head", 128256, 4096)]:
        w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn(T, k, device="cuda").to(torch.bfloat16)
        out = torch.zeros(T, n, device="cuda")
        res = []
        for split in (1, 2, 3, 4, 5, 6, 8, 9, 12, 16):
            if split > k // 64:
                continue
            ms = timeit(lambda: N.check(lib.lp_gemm_bf16(P(w), n, k, P(x), T, P(out), n, 0, split, None)))
            res.append((split, 2 * n * k / ms / 1e6))
        best = max(res, key=lambda r: r[1])
        print(f"T={T} {name:12s} tiles={-(-n // 128):4d} " + " ".join(f"s{s}:{g:5.0f}" for s, g in res)
              + f"  best s{best[0]} {best[1]:.0f} GB/s", flush=True)
    wg = (torch.randn(14336, 4096, device="cuda") * 0.02).to(torch.bfloat16)
    wu = (torch.randn(14336, 4096, device="cuda") * 0.02).to(torch.bfloat16)
    x = torch.randn(T, 4096, device="cuda").to(torch.bfloat16)
    act = torch.empty(T, 14336, dtype=torch.bfloat16, device="cuda")
    ms = timeit(lambda: N.check(lib.lp_gemm_swiglu(P(wg), P(wu), 14336, 4096, P(x), T, P(act), 14336, None)))
    print(f"T={T} swiglu fused (112 CTAs): {2 * 2 * 14336 * 4096 / ms / 1e6:.0f} GB/s", flush=True)
