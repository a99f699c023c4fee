"""ncu target (dev tool): one lp_gemm_bf16 launch at a decode / prefill shape
after an L2 flush, e.g. ``ncu --set full -k regex:gemm_ -s 2 -c 1 python
tools/gemm_ncu_target.py 6144 4096 16``  (N K T; split from llama.gemm_split)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import _native as N  # noqa: E402
from paper_2502_09922_b200.llama import gemm_split  # noqa: E402

n, k, T = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (6144, 4096, 16)))
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
lib = N.lib()
w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
x = torch.randn(T, k, device="cuda").to(torch.bfloat16)
out = torch.zeros(T, n, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(4):
    flush.zero_()
    N.check(lib.lp_gemm_bf16(P(w), n, k, P(x), T, P(out), n, 0, gemm_split(n, k, T), None))
torch.cuda.synchronize()
