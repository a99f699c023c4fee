"""tcgen05 GEMM perf (dev tool): weight-streaming GB/s (decode) and TFLOP/s
(prefill) for Llama-3-8B layer shapes, cuBLAS (torch.matmul) beside it."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import _native as N  # noqa: E402
from paper_2502_09922_b200.llama import gemm_split  # noqa: E402

P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
lib = N.lib()


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


SHAPES = {
    "llama3-8b": [("qkv", 6144, 4096), ("wo", 4096, 4096), ("gate_up", 14336, 4096), ("down", 4096, 14336)],
    "llama3-70b": [("qkv", 10240, 8192), ("wo", 8192, 8192), ("gate_up", 28672, 8192), ("down", 8192, 28672)],
}
shapes = SHAPES[sys.argv[2] if len(sys.argv) > 2 else "llama3-8b"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for T in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,16,64,256,1024,4096").split(",")]:
    for name, n, k in shapes:
        w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
        w2 = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn(T, k, device="cuda").to(torch.bfloat16)
        if name == "gate_up":
            out = torch.empty(T, n, dtype=torch.bfloat16, device="cuda")
            f = lambda: N.check(lib.lp_gemm_swiglu(P(w), P(w2), n, k, P(x), T, P(out), n, None))  # noqa: E731
            flops, wbytes = 4 * T * n * k, 2 * 2 * n * k
            ref = lambda: torch.matmul(x, torch.cat([w, w2]).T)  # noqa: E731
        else:
            out = torch.zeros(T, n, device="cuda")
            split = gemm_split(n, k, T)        # the executor's policy (llama.gemm_split)
            f = lambda: N.check(lib.lp_gemm_bf16(P(w), n, k, P(x), T, P(out), n, 0, split, None))  # noqa: E731
            flops, wbytes = 2 * T * n * k, 2 * n * k
            ref = lambda: torch.matmul(x, w.T)  # noqa: E731
        ms = timeit(f)
        ms_ref = timeit(ref)
        split_s = f"split={split}" if name != "gate_up" else "       "
        print(f"T={T:5d} {name:8s} N={n:6d} K={k:6d} {split_s} ours {ms*1e3:8.1f} us  {wbytes/ms/1e6:7.0f} GB/s(w)  "
              f"{flops/ms/1e9:7.1f} TF/s | cuBLAS {ms_ref*1e3:8.1f} us {flops/ms_ref/1e9:7.1f} TF/s", flush=True)
