"""Per-kernel parity probe of one decoder layer (GPU vs the bf16-faithful
oracle math applied to the GPU's own inputs), to locate where logits drift.

  python tools/parity_probe.py [tiny|llama3-8b] [T]
"""
import ctypes as C
import dataclasses
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import llama as OL  # noqa: E402
from paper_2502_09922_b200 import _native as N  # noqa: E402
from paper_2502_09922_b200 import engine as E  # noqa: E402
from paper_2502_09922_b200 import image as I  # noqa: E402
from paper_2502_09922_b200.llama import LlamaExecutor  # noqa: E402


def vp(t):
    return C.c_void_p(t.data_ptr())


def bf(t):
    return t.to(torch.bfloat16).float()


def report(name, got, ref):
    got, ref = got.float().cpu(), ref.float().cpu()
    d = (got - ref).abs()
    mism = (bf(got) != bf(ref)).float().mean().item()
    print(f"{name:28s} max|d| {d.max().item():.3e}  rel {d.max().item() / (ref.abs().max().item() + 1e-30):.2e}"
          f"  bf16-mismatch {mism * 100:.3f}%  |ref|max {ref.abs().max().item():.3e}")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    cfg = I.CONFIGS[name]
    if name != "tiny":
        cfg = dataclasses.replace(cfg, n_layers=1)
    lay = I.build_layout(cfg, 1 if name != "tiny" else 4)
    ptr = E.dev_malloc(0, lay.weights_bytes)
    E.fill_image(ptr, lay, 7)
    torch.cuda.synchronize()
    img = E.device_view(ptr, lay.weights_bytes, 0).cpu().numpy()
    W = OL.weights(lay, img)
    ex = LlamaExecutor(lay, ptr, 0, max_seqs=1, max_len=T + 8)
    lib = N.lib()
    dev = "cuda:0"
    H, KV, hd, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_model
    toks = np.random.default_rng(1).integers(0, cfg.vocab, T)
    tt = torch.as_tensor(toks, dtype=torch.int32, device=dev)
    pos = torch.arange(T, dtype=torch.int32, device=dev)
    seq = torch.zeros(T, dtype=torch.int32, device=dev)
    x = ex.embed(tt)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    l = 0
    p = f"layers.{l}."
    h = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
    nq = (H + 2 * KV) * hd
    qkv = torch.empty((T, nq), dtype=torch.float32, device=dev)
    N.check(lib.lp_rmsnorm_zero(vp(x), C.c_void_p(ex.ptr(p + "attn_norm")), T, d, cfg.norm_eps, vp(h), vp(qkv),
                                nq, s))
    torch.cuda.synchronize()
    xc = x.cpu()
    report("rmsnorm h", h, bf(OL._rms(xc, W[p + "attn_norm"], cfg.norm_eps)))
    ex._gemm_add(ex.ptr(p + "wq"), nq, d, h, T, qkv, nq, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    hc = h.float().cpu()
    wqkv = torch.cat([W[p + "wq"], W[p + "wk"], W[p + "wv"]], 0)
    report("qkv gemm", qkv, hc @ wqkv.T)
    q = torch.empty((T, H * hd), dtype=torch.bfloat16, device=dev)
    N.check(lib.lp_rope_kv(vp(qkv), T, H, KV, hd, vp(pos), vp(seq), cfg.rope_theta, vp(q), vp(ex.cache.k[l]),
                           vp(ex.cache.v[l]), ex.cache.max_len, s))
    torch.cuda.synchronize()
    qk = qkv.cpu()
    qr = OL._rope(qk[:, :H * hd].view(T, H, hd), pos.cpu(), cfg.rope_theta, True)
    report("rope q", q.view(T, H, hd), bf(qr))
    kr = OL._rope(qk[:, H * hd:(H + KV) * hd].view(T, KV, hd), pos.cpu(), cfg.rope_theta, True)
    report("rope k (cache)", ex.cache.k[l][0, :, :T].transpose(0, 1), bf(kr))
    vr = qk[:, (H + KV) * hd:].view(T, KV, hd)
    report("v (fp16 cache)", ex.cache.v[l][0, :, :T].transpose(0, 1), vr.half().float())
    o = torch.empty((T, H * hd), dtype=torch.bfloat16, device=dev)
    N.check(lib.lp_attention(vp(q), vp(ex.cache.k[l]), vp(ex.cache.v[l]), vp(pos), vp(seq), T, H, KV, hd,
                             ex.cache.max_len, 1.0 / math.sqrt(hd), vp(o), s))
    torch.cuda.synchronize()
    qg = q.float().cpu().view(T, H, hd)
    kg = ex.cache.k[l][0, :, :T].float().cpu().transpose(0, 1).repeat_interleave(H // KV, 1)
    vg = ex.cache.v[l][0, :, :T].float().cpu().transpose(0, 1).repeat_interleave(H // KV, 1)
    mask = torch.full((T, T), float("-inf")).triu(1)
    att = torch.einsum("thd,shd->hts", qg, kg) / math.sqrt(hd) + mask
    oref = torch.einsum("hts,shd->thd", att.softmax(-1), vg).reshape(T, H * hd)
    report("attention o", o, bf(oref))
    report("attention o (unrounded)", o, oref)
    xo = x.clone()
    ex._gemm_add(ex.ptr(p + "wo"), d, H * hd, o, T, x, d, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    report("wo + residual", x, xo.cpu() + o.float().cpu() @ W[p + "wo"].T)
    h2 = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
    N.check(lib.lp_rmsnorm(vp(x), C.c_void_p(ex.ptr(p + "ffn_norm")), T, d, cfg.norm_eps, vp(h2), s))
    act = torch.empty((T, cfg.ffn), dtype=torch.bfloat16, device=dev)
    N.check(lib.lp_gemm_swiglu(C.c_void_p(ex.ptr(p + "w_gate")), C.c_void_p(ex.ptr(p + "w_up")), cfg.ffn, d, vp(h2),
                               T, vp(act), cfg.ffn, s))
    torch.cuda.synchronize()
    h2c = h2.float().cpu()
    g, u = h2c @ W[p + "w_gate"].T, h2c @ W[p + "w_up"].T
    report("swiglu act", act, bf(g / (1 + torch.exp(-g)) * u))
    xd = x.clone()
    ex._gemm_add(ex.ptr(p + "w_down"), d, cfg.ffn, act, T, x, d, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    report("down + residual", x, xd.cpu() + act.float().cpu() @ W[p + "w_down"].T)
    # whole-model logits
    ex2 = LlamaExecutor(lay, ptr, 0, max_seqs=1, max_len=T + 8)
    _, lg = ex2.forward(tokens=tt, pos=pos, seq=seq)
    _, ref = OL.forward(cfg, W, toks, bf16=True)
    report("logits (full model)", lg, ref)
    E.dev_free(0, ptr)


if __name__ == "__main__":
    main()
