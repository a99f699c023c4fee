"""Decode-step timing of one local replica (dev tool): eager vs CUDA graph."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import engine as E  # noqa: E402
from paper_2502_09922_b200 import image as I  # noqa: E402
from paper_2502_09922_b200.llama import DecodeGraph, LlamaExecutor  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = I.CONFIGS[model]
lay = I.build_layout(cfg, 16 if cfg.n_layers >= 16 else cfg.n_layers)
ptr = E.dev_malloc(0, lay.weights_bytes)
E.fill_image(ptr, lay, 1)
ex = LlamaExecutor(lay, ptr, 0, max_seqs=B, max_len=256)
P = 128
toks = torch.randint(0, cfg.vocab, (B * P,), dtype=torch.int32, device="cuda")
pos = torch.arange(P, dtype=torch.int32, device="cuda").repeat(B)
seq = torch.arange(B, dtype=torch.int32, device="cuda").repeat_interleave(P)
torch.cuda.synchronize()
t0 = time.perf_counter()
_, lg = ex.forward(tokens=toks, pos=pos, seq=seq)
torch.cuda.synchronize()
print(f"prefill {B}x{P}: {1e3 * (time.perf_counter() - t0):.1f} ms (first call, incl. warm-up)")
ts = []
for _ in range(5):   # eager launches: host jitter, so the median of 5
    t0 = time.perf_counter()
    _, lg = ex.forward(tokens=toks, pos=pos, seq=seq)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"prefill {B}x{P}: {1e3 * sorted(ts)[2]:.1f} ms (median of 5, min {1e3 * min(ts):.1f})")
tok = torch.zeros(B, dtype=torch.int32, device="cuda")
p1 = torch.full((B,), P, dtype=torch.int32, device="cuda")
s1 = torch.arange(B, dtype=torch.int32, device="cuda")
for it in range(3):
    ex.forward(tokens=tok, pos=p1, seq=s1)
torch.cuda.synchronize()
t0 = time.perf_counter()
n = 10
for it in range(n):
    _, lg = ex.forward(tokens=tok, pos=p1, seq=s1)
    t, _ = ex.greedy(lg)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / n
print(f"eager decode step B={B}: {dt * 1e3:.2f} ms -> {B / dt:.0f} tok/s, weights {lay.weights_bytes / dt / 1e9:.0f} GB/s")
g = DecodeGraph(ex, B)
g.capture()
for it in range(3):
    g.graph.replay()
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(n):
    g.graph.replay()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / n
print(f"graph decode step B={B}: {dt * 1e3:.2f} ms -> {B / dt:.0f} tok/s, weights {lay.weights_bytes / dt / 1e9:.0f} GB/s")
t0 = time.perf_counter()
for it in range(n):
    out = g.step([1] * B, [P] * B, list(range(B)))
    out.cpu()
dt = (time.perf_counter() - t0) / n
print(f"graph step() incl. host copies+sync: {dt * 1e3:.2f} ms")
