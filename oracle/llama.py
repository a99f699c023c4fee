"""ORACLE (test infrastructure): CPU fp32 Llama decoder on a packed image.

The paper's inference module ("extends Meta's Llama framework",
PAPER.md:580) is not vendored, so logits parity is anchored on
transformers 5.5 ``LlamaForCausalLM`` (fp32) instead: tests/golden/
make_llama_golden.py runs it on the same bf16 weights and this restatement is
checked against its logits (tests/test_llama_oracle.py).

Math (HF modeling_llama): RMSNorm in fp32 (x * rsqrt(mean(x^2)+eps) * w),
RoPE rotate_half with inv_freq = theta^(-2j/hd), GQA causal softmax
attention with scale 1/sqrt(hd), SwiGLU MLP, untied LM head.

``bf16=True`` is the bf16-faithful mode: the same network, but every tensor
the CUDA path stores in bf16 is rounded to bf16 at the same point — the
RMSNorm outputs (GEMM inputs), q/k after RoPE (the bf16 K cache), the
attention output and the SwiGLU product — v is rounded to fp16 (the fp16 V
cache), while the residual stream, GEMM accumulation, softmax and logits stay
fp32 (paper_2502_09922_b200/llama.py module doc).  RoPE angles follow the kernel's fp32 recipe
(inv = 2^(-2j/hd * log2 theta), angle = float(pos) * inv).  What remains
between the two is accumulation order and the kernels' fp16 rounding of the
softmax probabilities inside attention, so greedy tokens agree wherever the
oracle's top-1/top-2 margin clears a small gate (tests/golden/prompts_tiny.json
holds prompts whose margins clear it at every generated position).
"""

from __future__ import annotations

import numpy as np


def weights(layout, image: np.ndarray) -> dict:
    """name -> fp32 torch tensor of every packed bf16 tensor."""
    import torch
    out = {}
    for t in layout.tensors:
        raw = np.ascontiguousarray(image[t.offset:t.offset + t.nbytes]).view(np.int16)
        bf = torch.from_numpy(raw.copy()).view(torch.bfloat16)
        out[t.name] = bf.to(torch.float32).reshape(t.shape)
    return out


def _bf(t, on: bool):
    """Round to bf16 and back when the CUDA path stores ``t`` in bf16."""
    import torch
    return t.to(torch.bfloat16).to(torch.float32) if on else t


def _h(t, on: bool):
    """Round to fp16 and back (the V cache) when faithful."""
    import torch
    return t.to(torch.float16).to(torch.float32) if on else t


def _rms(x, w, eps):
    import torch
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _rope(x, pos, theta, kernel_angles: bool = False):
    import math
    import torch
    hd = x.shape[-1]
    if kernel_angles:   # lp_llama.cu rope_kv_kernel: exp2f(-2j/hd * log2f(theta)) in fp32
        j = torch.arange(0, hd // 2, dtype=torch.float32)
        inv = torch.exp2(-2.0 * j / hd * torch.tensor(math.log2(theta), dtype=torch.float32))
    else:
        inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    ang = pos.float()[:, None] * inv[None, :]
    emb = torch.cat([ang, ang], dim=-1)
    cos, sin = emb.cos()[:, None, :], emb.sin()[:, None, :]
    x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
    rot = torch.cat([-x2, x1], dim=-1)
    return x * cos + rot * sin


def forward(cfg, W: dict, tokens, layers=None, x=None, head: bool = True, bf16: bool = False):
    """Full-sequence causal forward.  Returns (hidden fp32 [T,d], logits or None).
    ``bf16``: round where the CUDA path stores bf16 (module doc)."""
    import torch
    toks = torch.as_tensor(tokens, dtype=torch.int64)
    T = toks.numel()
    pos = torch.arange(T)
    H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    G = H // KV
    if x is None:
        x = W["embed"][toks].clone()
    lo, hi = (0, cfg.n_layers - 1) if layers is None else layers
    mask = torch.full((T, T), float("-inf")).triu(1)
    for l in range(lo, hi + 1):
        p = f"layers.{l}."
        h = _bf(_rms(x, W[p + "attn_norm"], cfg.norm_eps), bf16)
        q = (h @ W[p + "wq"].T).view(T, H, hd)
        k = (h @ W[p + "wk"].T).view(T, KV, hd)
        v = _h((h @ W[p + "wv"].T).view(T, KV, hd), bf16)
        q = _bf(_rope(q, pos, cfg.rope_theta, bf16), bf16)
        k = _bf(_rope(k, pos, cfg.rope_theta, bf16), bf16)
        k = k.repeat_interleave(G, dim=1)
        v = v.repeat_interleave(G, dim=1)
        att = torch.einsum("thd,shd->hts", q, k) / (hd ** 0.5) + mask
        o = _bf(torch.einsum("hts,shd->thd", att.softmax(-1), v).reshape(T, H * hd), bf16)
        x = x + o @ W[p + "wo"].T
        h = _bf(_rms(x, W[p + "ffn_norm"], cfg.norm_eps), bf16)
        g, u = h @ W[p + "w_gate"].T, h @ W[p + "w_up"].T
        a = _bf(g / (1.0 + torch.exp(-g)) * u, bf16) if bf16 else torch.nn.functional.silu(g) * u
        x = x + a @ W[p + "w_down"].T
    logits = None
    if head and hi == cfg.n_layers - 1:
        logits = _bf(_rms(x, W["final_norm"], cfg.norm_eps), bf16) @ W["lm_head"].T
    return x, logits


def greedy(cfg, W: dict, prompt, steps: int, bf16: bool = False):
    """Greedy continuation by full recompute (small models only).  Returns
    (tokens, top-1/top-2 logit margin at each generated position)."""
    toks = list(prompt)
    margins = []
    for _ in range(steps):
        _, logits = forward(cfg, W, toks, bf16=bf16)
        last = logits[-1]
        top = last.topk(2)
        margins.append(float(top.values[0] - top.values[1]))
        toks.append(int(top.indices[0]))
    return toks[len(prompt):], margins
