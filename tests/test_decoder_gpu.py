"""GPU parity of the decoder kernels.

* tcgen05 GEMM vs a torch fp32 matmul of the same bf16 operands
  (tolerance: |err| <= 1e-3 * sqrt(K) * rms(x) * rms(w) * 4, fp32 accumulation);
* the whole tiny Llama (prefill + KV-cache decode) vs the CPU oracle:
  logits within LOGIT_TOL of the bf16-faithful oracle (and LOGIT_TOL_FP32 of
  the transformers-pinned fp32 one); greedy tokens identical at EVERY
  generated position of the committed prompts (tests/golden/prompts_tiny.json,
  whose oracle margins clear the gate everywhere).
"""
import math

import numpy as np
import pytest

from paper_2502_09922_b200 import _native as N
from paper_2502_09922_b200 import image as I

pytestmark = pytest.mark.gpu

# absolute logit tolerances (logit std ~1.15).  Measured on B200: 0.035-0.038 vs the
# bf16-faithful oracle, 0.050 vs the fp32 one.  The floor is set by bf16 itself:
# rounding points amplify accumulation-order noise (a 1e-7 relative weight
# perturbation moves the bf16 oracle's own logits by 0.02, tests/test_prompts_golden.py),
# so the committed prompts' margins clear 0.1 at every position instead.
import os as _os
TESTS_DIR = _os.path.dirname(_os.path.abspath(__file__))
ROOT_DIR = _os.path.dirname(TESTS_DIR)
LOGIT_TOL = 0.06
LOGIT_TOL_FP32 = 0.1


def _ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


@pytest.mark.parametrize("n,k,t,epi,split", [
    (128, 64, 16, 1, 1), (256, 256, 1, 1, 1), (300, 688, 5, 1, 1), (1024, 1024, 33, 0, 4),
    (4096, 512, 100, 0, 2), (384, 4096, 300, 1, 1), (640, 1536, 256, 0, 1), (32000, 256, 24, 1, 1),
    (512, 4096, 7, 0, 8),
    # CTA-pair stream-K tail (> 1 wave of 74 pair tiles, tail <= 80 %): 192 tiles, 8 k-blocks each;
    # 160 ragged tiles whose tail spans are 1-2 k-blocks
    (6144, 512, 2048, 0, 1), (5000, 640, 1900, 0, 1)])
def test_gemm_matches_fp32(n, k, t, epi, split):
    import torch
    g = torch.Generator(device="cuda").manual_seed(n * 7 + k)
    w = (torch.randn(n, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(t, k, device="cuda", generator=g).to(torch.bfloat16)
    ref = x.float() @ w.float().T
    out = torch.full((t, n), 0.5, device="cuda") if epi == 0 else torch.empty((t, n), device="cuda")
    N.check(N.lib().lp_gemm_bf16(_ptr(w), n, k, _ptr(x), t, _ptr(out), n, epi, split, None))
    torch.cuda.synchronize()
    if epi == 0:
        ref = ref + 0.5
    tol = 4e-3 * math.sqrt(k) * 0.05
    assert (out - ref).abs().max().item() < tol


@pytest.mark.parametrize("n,k,t", [(688, 256, 24), (1536, 512, 1), (640, 1024, 130), (1408, 512, 600),
                                   (384, 4096, 257),
                                   # > 1 wave of 256 x 256 pair tiles: the partial last wave's rows go
                                   # to a 64-token-tile launch (224 tiles; ragged 90 tiles at T = 1100)
                                   (14336, 256, 1024), (4608, 128, 1100)])
def test_gemm_swiglu_matches_fp32(n, k, t):
    import torch
    g = torch.Generator(device="cuda").manual_seed(n + k)
    wg = (torch.randn(n, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    wu = (torch.randn(n, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(t, k, device="cuda", generator=g).to(torch.bfloat16)
    ref = torch.nn.functional.silu(x.float() @ wg.float().T) * (x.float() @ wu.float().T)
    out = torch.empty((t, n), dtype=torch.bfloat16, device="cuda")
    N.check(N.lib().lp_gemm_swiglu(_ptr(wg), _ptr(wu), n, k, _ptr(x), t, _ptr(out), n, None))
    torch.cuda.synchronize()
    assert ((out.float() - ref).abs() / (ref.abs() + 0.1)).max().item() < 0.05


@pytest.mark.parametrize("hd,H,KV,ctx,run", [(128, 32, 8, [1, 150, 37, 300], 40), (64, 4, 2, [5, 129, 64], 40),
                                              (128, 64, 8, [200, 17], 40), (128, 8, 8, [33, 96], 40),
                                              (128, 64, 8, [300, 5], 200), (64, 4, 2, [600], 520),
                                              (128, 32, 8, [150, 100, 3], 150), (64, 16, 4, [300, 7], 299)])
def test_attention_matches_fp32(hd, H, KV, ctx, run):
    """Ragged causal GQA attention (decode rows at arbitrary positions and a
    prefill-style run of ``run`` consecutive positions) vs a torch fp32
    softmax.  T x KV >= 1024 selects the prefill variants: smem-staged row
    tiles when max_len's K/V fit (the last two cases; mixed-sequence tiles
    read global memory), else a warp per row."""
    _check_attention(hd, H, KV, ctx, run, max(ctx) + 8)


@pytest.mark.parametrize("dbuf", ["1", "0"])
def test_attention_decode_single_cta_double_buffer(dbuf, monkeypatch):
    """The single-CTA double-buffered decode variant (no key split: T x KV in
    [75, 148], cache >= 1024 keys — the 8B B = 10 x 1100-key case) and, as an
    A/B, the single-buffered kernel (LP_DEC_DBUF=0, read once per process, so
    run in a subprocess)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r); import test_decoder_gpu as t; "
            "t._check_attention(128, 32, 8, [1100] * 10, 0, 1200)") % (ROOT_DIR, TESTS_DIR)
    env = dict(__import__("os").environ, LP_DEC_DBUF=dbuf)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=240)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]


@pytest.mark.parametrize("hd,H,KV,ctx,max_len", [(128, 32, 8, [4000], 4096), (64, 4, 2, [1, 1500, 700], 1536),
                                                  (128, 64, 8, [2048, 30], 2056), (128, 32, 8, [1, 5], 2048),
                                                  (128, 8, 8, [1100, 257, 64, 1], 1200),
                                                  (64, 4, 2, [1, 3000, 4100], 4200), (128, 64, 8, [20000], 20480)])
def test_attention_long_context_cluster_split(hd, H, KV, ctx, max_len):
    """Few decode rows over a long-context cache: the keys of a row are split
    over a thread-block cluster (8, or 16 non-portable when it fits) and
    merged through distributed shared memory (CTAs that get no keys carry an
    empty softmax state)."""
    _check_attention(hd, H, KV, ctx, 0, max_len)


def _check_attention(hd, H, KV, ctx, run, max_len):
    import torch
    g = torch.Generator(device="cuda").manual_seed(hd + H + len(ctx))
    seqs = len(ctx)
    kc = torch.randn(seqs, KV, max_len, hd, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn(seqs, KV, max_len, hd, device="cuda", generator=g).to(torch.float16)
    pos = [c - 1 for c in ctx] + list(range(ctx[0] - 1, max(ctx[0] - run, -1), -1))
    seq = list(range(seqs)) + [0] * (len(pos) - seqs)
    T = len(pos)
    q = torch.randn(T, H, hd, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty(T, H, hd, dtype=torch.bfloat16, device="cuda")
    p_t = torch.tensor(pos, dtype=torch.int32, device="cuda")
    s_t = torch.tensor(seq, dtype=torch.int32, device="cuda")
    scale = 1.0 / math.sqrt(hd)
    N.check(N.lib().lp_attention(_ptr(q), _ptr(kc), _ptr(vc), _ptr(p_t), _ptr(s_t), T, H, KV, hd, max_len,
                                 N.C.c_float(scale), _ptr(out), None))
    torch.cuda.synchronize()
    G = H // KV
    for t in range(T):
        L = pos[t] + 1
        k = kc[seq[t], :, :L].float().repeat_interleave(G, 0)      # [H, L, hd]
        v = vc[seq[t], :, :L].float().repeat_interleave(G, 0)
        w = torch.softmax(torch.einsum("hd,hld->hl", q[t].float() * scale, k), -1)
        ref = torch.einsum("hl,hld->hd", w, v)
        assert (out[t].float() - ref).abs().max().item() < 2e-2, f"token {t} (pos {pos[t]})"


@pytest.fixture(scope="module")
def tiny():
    import torch
    from oracle import dataplane as D
    from oracle import llama as OL
    from paper_2502_09922_b200 import engine as E
    cfg = I.CONFIGS["tiny"]
    lay = I.build_layout(cfg, 4)
    img = D.fill_image(lay, 7)
    W = OL.weights(lay, img)
    dev_img = torch.from_numpy(img).cuda()          # the product fills its own image below
    ptr = E.dev_malloc(0, lay.weights_bytes)
    E.fill_image(ptr, lay, 7)
    torch.cuda.synchronize()
    got = E.device_view(ptr, lay.weights_bytes, 0)
    assert torch.equal(got, dev_img)                  # GPU generator == oracle generator, byte-exact
    yield cfg, lay, W, ptr
    E.dev_free(0, ptr)


def test_tiny_prefill_and_decode_match_oracle(tiny):
    import torch
    from oracle import llama as OL
    from paper_2502_09922_b200.llama import LlamaExecutor
    from parity import assert_tokens, entries
    cfg, lay, W, ptr = tiny
    e = next(x for x in entries(12) if len(x["prompt"]) == 24)
    prompt = np.asarray(e["prompt"], dtype=np.int64)
    ex = LlamaExecutor(lay, ptr, 0, max_seqs=2, max_len=64)
    toks = torch.as_tensor(prompt, dtype=torch.int32, device="cuda")
    pos = torch.arange(len(prompt), dtype=torch.int32, device="cuda")
    seq = torch.zeros(len(prompt), dtype=torch.int32, device="cuda")
    _, logits = ex.forward(tokens=toks, pos=pos, seq=seq)
    _, ref = OL.forward(cfg, W, prompt, bf16=True)
    _, ref32 = OL.forward(cfg, W, prompt)
    err = (logits.cpu() - ref).abs().max().item()
    err32 = (logits.cpu() - ref32).abs().max().item()
    print(f"tiny prefill logits: max |gpu - bf16 oracle| {err:.5f}, |gpu - fp32 oracle| {err32:.5f}")
    assert err < LOGIT_TOL, err
    assert err32 < LOGIT_TOL_FP32, err32
    # greedy decode through the KV cache: all 16 positions
    tok, _ = ex.greedy(logits[-1:])
    out = [int(tok.item())]
    for step in range(len(e["greedy"]) - 1):
        p = torch.tensor([len(prompt) + step], dtype=torch.int32, device="cuda")
        _, lg = ex.forward(tokens=tok, pos=p, seq=seq[:1])
        tok, _ = ex.greedy(lg)
        out.append(int(tok.item()))
    assert assert_tokens(out, e, what="tiny KV-cache decode") == 16
    # teacher-forced logits of the decode steps: one causal oracle pass
    full = list(prompt) + out[:-1]
    _, ref_all = OL.forward(cfg, W, full, bf16=True)
    ex2 = LlamaExecutor(lay, ptr, 0, max_seqs=2, max_len=64)
    n = len(full)
    _, lg_all = ex2.forward(tokens=torch.as_tensor(full, dtype=torch.int32, device="cuda"),
                            pos=torch.arange(n, dtype=torch.int32, device="cuda"),
                            seq=torch.zeros(n, dtype=torch.int32, device="cuda"))
    err_all = (lg_all.cpu() - ref_all).abs().max().item()
    print(f"tiny prefill {n} tokens: max |gpu - bf16 oracle| {err_all:.5f}")
    assert err_all < LOGIT_TOL


def test_stage_split_equals_local(tiny):
    """Two stages (layers 0-1 with vocab ops, 2-3) hand hidden states over and
    produce the same logits as one local executor (tolerance: split-K order)."""
    import torch
    from paper_2502_09922_b200.llama import LlamaExecutor
    cfg, lay, W, ptr = tiny
    prompt = torch.as_tensor(np.random.default_rng(3).integers(0, cfg.vocab, 16), dtype=torch.int32,
                             device="cuda")
    pos = torch.arange(16, dtype=torch.int32, device="cuda")
    seq = torch.zeros(16, dtype=torch.int32, device="cuda")
    local = LlamaExecutor(lay, ptr, 0, max_seqs=1, max_len=32)
    _, ref = local.forward(tokens=prompt, pos=pos, seq=seq)
    s0 = LlamaExecutor(lay, ptr, 0, 0, 1, max_seqs=1, max_len=32)
    s1 = LlamaExecutor(lay, ptr, 0, 2, 3, max_seqs=1, max_len=32)
    x, _ = s0.forward(tokens=prompt, pos=pos, seq=seq, want_logits=False)
    x, _ = s1.forward(x=x.clone(), pos=pos, seq=seq, want_logits=False)
    lg = s0.head(x)
    assert (lg - ref).abs().max().item() < 1e-2


def test_generate_api_matches_oracle(tiny):
    """serving.generate(): batched prefill + graph decode == oracle greedy at
    every one of 16 positions for three prompts of different lengths."""
    from paper_2502_09922_b200.llama import LlamaExecutor
    from paper_2502_09922_b200.serving import generate
    from parity import assert_tokens, doc
    cfg, lay, W, ptr = tiny
    es = [e for e in doc()["prompts"] if len(e["prompt"]) in (9, 12, 15)]
    assert len(es) == 3
    ex = LlamaExecutor(lay, ptr, 0, max_seqs=4, max_len=48)
    outs = generate(ex, [e["prompt"] for e in es], 16)
    compared = sum(assert_tokens(got, e, what=f"generate prompt {len(e['prompt'])}") for got, e in zip(outs, es))
    assert compared == 48


@pytest.mark.parametrize("hd,H,KV,lens,cap", [(128, 32, 8, [1024], 0), (128, 64, 8, [700, 300], 0),
                                               (128, 8, 8, [517], 0), (64, 4, 2, [600, 1, 33], 0),
                                               (128, 32, 8, [64] * 9 + [130], 400),
                                               # 70B groups (G = 8, 16-token tiles, 32 per CTA) with
                                               # ragged lengths; MHA at head_dim 64
                                               (128, 64, 8, [37, 250, 5, 301], 0), (64, 8, 8, [300, 77], 0)])
def test_prefill_attention_tcgen05_causal(hd, H, KV, lens, cap):
    """Prompts laid out as consecutive rows (the serving layout: one or more
    sequences back to back, positions 0..len-1) through the tcgen05/TMEM
    prefill kernel (lp_attn_tc.cu), vs a torch fp32 causal softmax over the
    same bf16 K / fp16 V caches."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(sum(lens) + hd + H)
    seqs, max_len = len(lens), max(max(lens) + 16, cap)     # caches > 256 keys take the tcgen05 kernel
    kc = torch.randn(seqs, KV, max_len, hd, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn(seqs, KV, max_len, hd, device="cuda", generator=g).to(torch.float16)
    pos = [p for n in lens for p in range(n)]
    seq = [s for s, n in enumerate(lens) for _ in range(n)]
    T = len(pos)
    assert T * KV >= 1024
    q = torch.randn(T, H, hd, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty(T, H, hd, dtype=torch.bfloat16, device="cuda")
    p_t = torch.tensor(pos, dtype=torch.int32, device="cuda")
    s_t = torch.tensor(seq, dtype=torch.int32, device="cuda")
    scale = 1.0 / math.sqrt(hd)
    N.check(N.lib().lp_attention(_ptr(q), _ptr(kc), _ptr(vc), _ptr(p_t), _ptr(s_t), T, H, KV, hd, max_len,
                                 N.C.c_float(scale), _ptr(out), None))
    torch.cuda.synchronize()
    G = H // KV
    row = 0
    for s, n in enumerate(lens):
        k = kc[s, :, :n].float().repeat_interleave(G, 0)            # [H, n, hd]
        v = vc[s, :, :n].float().repeat_interleave(G, 0)
        qs = q[row:row + n].float().transpose(0, 1) * scale           # [H, n, hd]
        att = torch.einsum("hid,hjd->hij", qs, k)
        att = att.masked_fill(torch.ones(n, n, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
        ref = torch.einsum("hij,hjd->hid", att.softmax(-1), v).transpose(0, 1)
        err = (out[row:row + n].float() - ref).abs().max().item()
        assert err < 2e-2, (s, n, err)
        row += n


@pytest.mark.parametrize("seed", range(6))
def test_prefill_attention_random_ragged_batches(seed):
    """Random ragged prompt batches (1-6 prompts of 1-700 tokens, GQA groups
    of 1-8 heads, head_dim 64 / 128) through whichever prefill kernel the
    dispatch picks (tcgen05 FA layout for GQA >= 4 or caches > 256 keys,
    mma.sync otherwise), vs a torch fp32 causal softmax."""
    import random
    rnd = random.Random(1000 + seed)
    hd = rnd.choice([64, 128])
    KV = rnd.choice([2, 4, 8])
    G = rnd.choice([1, 2, 4, 8])
    lens = [rnd.randint(1, 700) for _ in range(rnd.randint(1, 6))]
    while sum(lens) * KV < 1024:          # the prefill (many-row) path
        lens.append(rnd.randint(64, 700))
    test_prefill_attention_tcgen05_causal(hd, G * KV, KV, lens, 0)


@pytest.mark.parametrize("seed", range(6))
def test_gemm_random_shapes(seed):
    """Random prefill / decode shapes through the residual-add GEMM (split-K,
    CTA pairs, the stream-K tail) and the fused SwiGLU (incl. its tail
    launch), vs torch fp32."""
    import random
    rnd = random.Random(2000 + seed)
    n = 128 * rnd.randint(1, 96) + rnd.choice([0, 0, 16, 48])
    k = 64 * rnd.randint(1, 48)
    t = rnd.choice([rnd.randint(1, 64), rnd.randint(65, 700), rnd.randint(700, 2500)])
    test_gemm_matches_fp32(n, k, t, 0, 1)
    if k % 64 == 0:
        test_gemm_swiglu_matches_fp32(n, k, t)
