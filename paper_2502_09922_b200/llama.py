"""Llama decoder on the packed image, executed by the sm_100a kernels.

:class:`LlamaExecutor` runs any contiguous layer range of a model whose
weights live in a packed image (``image.build_layout``) on one GPU: that is
both a λPipe pipeline *stage* (layers of its resident blocks; the stage
holding block 0 also owns embedding + final norm + LM head, see image.py)
and, with all layers, the local full-model replica after mode switch.

Per layer (fp32 residual stream ``x``, bf16 GEMM inputs, fp32 accumulation):

    h   = rmsnorm(x) * attn_norm                      lp_rmsnorm
    qkv = h @ [Wq;Wk;Wv]^T          (one GEMM: wq/wk/wv are contiguous)
    q,k,v <- RoPE(qkv); k,v appended to the KV cache  lp_rope_kv
    o   = causal GQA attention(q, cache)              lp_attention
    x  += o @ Wo^T                  (GEMM, split-K, residual-add epilogue)
    h   = rmsnorm(x) * ffn_norm
    a   = silu(h @ Wg^T) * (h @ Wu^T)  (one GEMM, two TMEM accumulators)
    x  += a @ Wd^T                  (GEMM, split-K, residual-add epilogue)

The GEMMs are ``lp_gemm_bf16`` / ``lp_gemm_swiglu`` (tcgen05 + TMEM + TMA).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time

from . import _native as N
from .engine import device_view
from .image import ImageLayout

def _vp(x):
    return C.c_void_p(x if isinstance(x, int) else x.data_ptr())


def _cur_stream(stream):
    """Kernels go to torch's current stream unless told otherwise (so they
    are captured by ``torch.cuda.graph``)."""
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


SMS = 148
GEMM_PAIR = os.environ.get("LP_GEMM_PAIR", "1") != "0"   # mirrors lp_gemm.cu's switches
GEMM_PAIR_STREAMK = os.environ.get("LP_GEMM_PAIR_STREAMK", "1") != "0"


def gemm_token_tile(tokens: int) -> int:
    """Token tile lp_gemm_bf16 dispatches for ``tokens`` (lp_gemm.cu dispatch())."""
    for bt in (16, 32, 64, 128):
        if tokens <= bt:
            return bt
    return 256


def gemm_split(n_rows: int, k: int, tokens: int) -> int:
    """K splits for the accumulating (residual-add) GEMM.

    Decode (T <= 64, one CTA per work item, 2 per SM): ~160 CTAs measured
    best (profiles/gemm_split_sweep_r01.txt).  Prefill (persistent, one CTA
    per SM): the split maximising wave efficiency (work items / 148-SM
    slots), discounted 2 % per extra split — e.g. QKV at T = 256 has only 48 tiles of 128 x 256, so
    48 of 148 SMs would work without a 3-way split.  Each split keeps >= 8
    k-blocks of 64."""
    kb = -(-k // 64)
    if tokens <= 64:
        tiles = -(-n_rows // 128) * -(-tokens // gemm_token_tile(tokens))
        return max(1, min(round(160 / max(tiles, 1)), max(1, kb // 4)))
    # prefill runs on CTA pairs (lp_gemm.cu gemm_pair_kernel): 256-row tiles
    # over SMS / 2 cluster slots
    slots = SMS // 2 if GEMM_PAIR else SMS
    rows = 256 if GEMM_PAIR else 128
    tiles = -(-n_rows // rows) * -(-tokens // gemm_token_tile(tokens))
    if GEMM_PAIR and GEMM_PAIR_STREAMK and tiles > slots and (tiles % slots) * 10 <= 8 * slots:
        # more than one wave: the kernel's stream-K tail balances the last
        # partial wave itself (same condition as lp_gemm.cu; profiles/r02/gemm_streamk_ab.txt)
        return 1
    if tiles >= 2 * slots:
        # >= 2 waves: tiles finish at staggered times, so quantisation costs
        # less than modelled, while shorter K per item exposes the red.add
        # epilogue (T = 4096 QKV: 167 us unsplit vs 192 us at 3 splits)
        return 1
    best, best_score = 1, 0.0
    for split in range(1, 9):
        if split > 1 and kb // split < 8:
            break
        items = tiles * split
        eff = items / (-(-items // slots) * slots)
        score = eff * (1.0 - 0.02 * (split - 1))    # each split re-adds T x N partial sums
        if score > best_score + 1e-9:
            best, best_score = split, score
    return best


def _upload(graph):
    """Replay a freshly captured graph once (its static inputs still point
    every row at the scratch sequence slot, so nothing live is touched): the
    first launch of an instantiated graph uploads it to the device, which
    measured 30+ ms for a 32-layer prefill graph — paid here, before the
    serving clock, instead of by the first request after the mode switch."""
    import torch
    graph.replay()
    torch.cuda.current_stream().synchronize()


class KVCache:
    """K (bf16) and V (fp16) caches per layer: [max_seqs, n_kv, max_len, head_dim].
    V is fp16 because attention's P V product runs in fp16 (lp_llama.cu)."""

    def __init__(self, cfg, layers, max_seqs: int, max_len: int, device):
        import torch
        self.max_seqs, self.max_len = max_seqs, max_len
        shape = (max_seqs, cfg.n_kv_heads, max_len, cfg.head_dim)
        self.k = {l: torch.zeros(shape, dtype=torch.bfloat16, device=device) for l in layers}
        self.v = {l: torch.zeros(shape, dtype=torch.float16, device=device) for l in layers}


class LlamaExecutor:
    """Runs layers [layer_lo, layer_hi] (+ vocab ops if it holds block 0)."""

    def __init__(self, layout: ImageLayout, image_ptr: int, device: int, layer_lo: int = 0,
                 layer_hi: int | None = None, max_seqs: int = 8, max_len: int = 512, vocab_ops: bool = True):
        import torch
        self.lay = layout
        self.cfg = layout.config
        self.base = image_ptr
        self.device = device
        self.layer_lo = layer_lo
        self.layer_hi = self.cfg.n_layers - 1 if layer_hi is None else layer_hi
        self.vocab_ops = vocab_ops
        self.torch_device = torch.device(f"cuda:{device}")
        # one extra sequence slot: scratch for padded rows of captured decode graphs
        self.cache = KVCache(self.cfg, range(self.layer_lo, self.layer_hi + 1), max_seqs + 1, max_len,
                             self.torch_device)
        self.scratch_seq = max_seqs
        self.lib = N.lib()

    # -- weights ----------------------------------------------------------------
    def ptr(self, name: str) -> int:
        return self.base + self.lay.by_name[name].offset

    def weight(self, name: str):
        """A torch bf16 view of one packed tensor (no copy)."""
        import torch
        t = self.lay.by_name[name]
        return device_view(self.base + t.offset, t.nbytes, self.device, torch.bfloat16, t.shape)

    # -- kernels ------------------------------------------------------------------
    def _gemm_add(self, w: int, n_rows: int, k: int, x, tokens: int, out, ldo: int, stream: int):
        split = gemm_split(n_rows, k, tokens)
        N.check(self.lib.lp_gemm_bf16(C.c_void_p(w), n_rows, k, _vp(x), tokens, _vp(out), ldo, 0, split,
                                      C.c_void_p(stream)), "lp_gemm_bf16")

    def embed(self, tokens, stream=None):
        stream = _cur_stream(stream)
        import torch
        T = tokens.numel()
        x = torch.empty((T, self.cfg.d_model), dtype=torch.float32, device=self.torch_device)
        N.check(self.lib.lp_embed(C.c_void_p(self.ptr("embed")), self.cfg.d_model, _vp(tokens), T, _vp(x),
                                  C.c_void_p(stream)), "lp_embed")
        return x

    def layer(self, l: int, x, pos, seq, stream=None):
        stream = _cur_stream(stream)
        import torch
        cfg = self.cfg
        T, d = x.shape
        H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        s = C.c_void_p(stream)
        dev = self.torch_device
        h = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
        nq = (H + 2 * KV) * hd
        qkv = torch.empty((T, nq), dtype=torch.float32, device=dev)    # zeroed by the norm kernel
        N.check(self.lib.lp_rmsnorm_zero(_vp(x), C.c_void_p(self.ptr(f"layers.{l}.attn_norm")), T, d, cfg.norm_eps,
                                         _vp(h), _vp(qkv), nq, s), "lp_rmsnorm_zero")
        self._gemm_add(self.ptr(f"layers.{l}.wq"), nq, d, h, T, qkv, nq, stream)
        q = torch.empty((T, H * hd), dtype=torch.bfloat16, device=dev)
        N.check(self.lib.lp_rope_kv(_vp(qkv), T, H, KV, hd, _vp(pos), _vp(seq), cfg.rope_theta, _vp(q),
                                    _vp(self.cache.k[l]), _vp(self.cache.v[l]), self.cache.max_len, s),
                "lp_rope_kv")
        o = torch.empty((T, H * hd), dtype=torch.bfloat16, device=dev)
        N.check(self.lib.lp_attention(_vp(q), _vp(self.cache.k[l]), _vp(self.cache.v[l]), _vp(pos), _vp(seq), T,
                                      H, KV, hd, self.cache.max_len, 1.0 / math.sqrt(hd), _vp(o), s),
                "lp_attention")
        self._gemm_add(self.ptr(f"layers.{l}.wo"), d, H * hd, o, T, x, d, stream)
        N.check(self.lib.lp_rmsnorm(_vp(x), C.c_void_p(self.ptr(f"layers.{l}.ffn_norm")), T, d, cfg.norm_eps,
                                    _vp(h), s), "lp_rmsnorm")
        act = torch.empty((T, cfg.ffn), dtype=torch.bfloat16, device=dev)
        N.check(self.lib.lp_gemm_swiglu(C.c_void_p(self.ptr(f"layers.{l}.w_gate")),
                                        C.c_void_p(self.ptr(f"layers.{l}.w_up")), cfg.ffn, d, _vp(h), T, _vp(act),
                                        cfg.ffn, s), "lp_gemm_swiglu")
        self._gemm_add(self.ptr(f"layers.{l}.w_down"), d, cfg.ffn, act, T, x, d, stream)
        return x

    def head(self, x, stream=None):
        """Final norm + LM head -> fp32 logits [T, V]."""
        stream = _cur_stream(stream)
        import torch
        cfg = self.cfg
        T, d = x.shape
        h = torch.empty((T, d), dtype=torch.bfloat16, device=self.torch_device)
        N.check(self.lib.lp_rmsnorm(_vp(x), C.c_void_p(self.ptr("final_norm")), T, d, cfg.norm_eps, _vp(h),
                                    C.c_void_p(stream)), "lp_rmsnorm")
        logits = torch.empty((T, cfg.vocab), dtype=torch.float32, device=self.torch_device)
        N.check(self.lib.lp_gemm_bf16(C.c_void_p(self.ptr("lm_head")), cfg.vocab, d, _vp(h), T, _vp(logits),
                                      cfg.vocab, 1, 1, C.c_void_p(stream)), "lp_gemm_bf16")
        return logits

    def greedy(self, logits, stream=None):
        stream = _cur_stream(stream)
        import torch
        T = logits.shape[0]
        tok = torch.empty((T,), dtype=torch.int32, device=self.torch_device)
        top2 = torch.empty((T, 2), dtype=torch.float32, device=self.torch_device)
        N.check(self.lib.lp_argmax(_vp(logits), T, self.cfg.vocab, _vp(tok), _vp(top2), C.c_void_p(stream)),
                "lp_argmax")
        return tok, top2

    def forward(self, tokens=None, x=None, pos=None, seq=None, stream=None, want_logits: bool = True):
        """Embed (if tokens) -> layers [lo, hi] -> head (if this stage owns it)."""
        if x is None:
            x = self.embed(tokens, stream)
        for l in range(self.layer_lo, self.layer_hi + 1):
            x = self.layer(l, x, pos, seq, stream)
        if want_logits and self.vocab_ops and self.layer_hi == self.cfg.n_layers - 1:
            return x, self.head(x, stream)
        return x, None


class DecodeGraph:
    """A CUDA graph of one batched decode step (embed -> all layers -> head ->
    argmax) for a full-model executor, ``batch`` rows wide.  Rows past the
    live batch are padded onto the executor's scratch sequence slot, so a
    fixed-shape graph serves any batch <= ``batch``; one replay replaces
    ~10 kernel launches per layer."""

    def __init__(self, ex: LlamaExecutor, batch: int):
        import torch
        self.ex, self.batch = ex, batch
        dev = ex.torch_device
        self.tokens = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.pos = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.seq = torch.full((batch,), ex.scratch_seq, dtype=torch.int32, device=dev)
        self.graph = None
        self.out = None
        # pinned staging: one H2D copy of [tokens | pos | seq], one D2H of the result
        self.h_in = torch.zeros(3 * batch, dtype=torch.int32).pin_memory()
        self.d_in = torch.zeros(3 * batch, dtype=torch.int32, device=dev)
        self.d_in[2 * batch:] = ex.scratch_seq   # warm-up/capture rows must only touch the scratch slot
        self.h_out = torch.zeros(batch, dtype=torch.int32).pin_memory()

    def _body(self):
        b = self.batch
        self.tokens.copy_(self.d_in[:b])
        self.pos.copy_(self.d_in[b:2 * b])
        self.seq.copy_(self.d_in[2 * b:])
        _, logits = self.ex.forward(tokens=self.tokens, pos=self.pos, seq=self.seq)
        tok, _ = self.ex.greedy(logits)
        return tok

    def capture(self):
        import torch
        with torch.cuda.device(self.ex.device):
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self._body()                      # warm-up: tensor maps, attributes, allocator
            torch.cuda.current_stream().wait_stream(s)
            self.graph = torch.cuda.CUDAGraph()
            # explicit per-device capture stream: torch.cuda.graph's default side
            # stream is created once, on whichever device captured first
            N.lib().lp_set_pdl(1)
            try:
                with torch.cuda.graph(self.graph, stream=torch.cuda.Stream(device=self.ex.device)):
                    self.out = self._body()
            finally:
                N.lib().lp_set_pdl(0)
            _upload(self.graph)

    def step(self, tokens, pos, seq):
        """Decode one token for each live row; returns the int32 device tensor."""
        import torch
        n = len(tokens)
        if n > self.batch:
            raise ValueError("batch larger than the captured graph")
        if self.graph is None:
            self.capture()
        b = self.batch
        pad = b - n
        vals = list(tokens) + [0] * pad + list(pos) + [0] * pad + list(seq) + [self.ex.scratch_seq] * pad
        self.h_in.numpy()[:] = vals
        with torch.cuda.device(self.ex.device):
            self.d_in.copy_(self.h_in, non_blocking=True)
            self.graph.replay()
            self.h_out.copy_(self.out, non_blocking=True)
        return self.h_out[:n]


class PrefillGraph:
    """A CUDA graph of one ragged prefill (embed -> all layers -> head on the
    last row of every request -> argmax) padded to ``tokens`` rows and
    ``rows`` requests.  Padded token rows sit on the scratch sequence slot at
    position 0; padded request rows read row 0 and are ignored."""

    def __init__(self, ex: LlamaExecutor, tokens: int, rows: int):
        import torch
        self.ex, self.cap, self.rows = ex, tokens, rows
        dev = ex.torch_device
        self.d_in = torch.zeros(3 * tokens + rows, dtype=torch.int32, device=dev)
        self.h_in = torch.zeros(3 * tokens + rows, dtype=torch.int32).pin_memory()
        self.h_out = torch.zeros(rows, dtype=torch.int32).pin_memory()
        self.graph = None
        self.out = None

    def _body(self):
        c, r = self.cap, self.rows
        toks, pos, seq = self.d_in[:c], self.d_in[c:2 * c], self.d_in[2 * c:3 * c]
        last = self.d_in[3 * c:3 * c + r].long()
        x = self.ex.embed(toks)
        for l in range(self.ex.layer_lo, self.ex.layer_hi + 1):
            x = self.ex.layer(l, x, pos, seq)
        logits = self.ex.head(x.index_select(0, last).contiguous())
        tok, _ = self.ex.greedy(logits)
        return tok

    def capture(self):
        import torch
        c = self.cap
        self.d_in[2 * c:3 * c].fill_(self.ex.scratch_seq)
        with torch.cuda.device(self.ex.device):
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self._body()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = torch.cuda.CUDAGraph()
            N.lib().lp_set_pdl(1)
            try:
                with torch.cuda.graph(self.graph, stream=torch.cuda.Stream(device=self.ex.device)):
                    self.out = self._body()
            finally:
                N.lib().lp_set_pdl(0)
            _upload(self.graph)

    def step(self, tokens, pos, seq, last):
        """Prefill; returns the next token of each request (pinned host tensor,
        valid after the device is synchronised)."""
        import torch
        c, r = self.cap, self.rows
        n, m = len(tokens), len(last)
        if n > c or m > r:
            raise ValueError("prefill larger than the captured graph")
        if self.graph is None:
            self.capture()
        t0 = time.perf_counter()
        buf = self.h_in.numpy()
        buf[:n] = tokens
        buf[n:c] = 0
        buf[c:c + n] = pos
        buf[c + n:2 * c] = 0
        buf[2 * c:2 * c + n] = seq
        buf[2 * c + n:3 * c] = self.ex.scratch_seq
        buf[3 * c:3 * c + m] = last
        buf[3 * c + m:] = 0
        with torch.cuda.device(self.ex.device):
            t1 = time.perf_counter()
            self.d_in.copy_(self.h_in, non_blocking=True)
            t2 = time.perf_counter()
            self.graph.replay()
            t3 = time.perf_counter()
            self.h_out.copy_(self.out, non_blocking=True)
        self.last_timing = (t1 - t0, t2 - t1, t3 - t2, time.perf_counter() - t3)   # host s: fill, h2d, replay, d2h
        return self.h_out[:m]


class SegmentGraph:
    """One captured piece of a pipeline stage, with static device I/O:

    * ``embed``: tokens -> x (vocab stage only),
    * layers [ex.layer_lo, ex.layer_hi] on x,
    * ``head``: rows ``last`` of x -> final norm -> LM head -> argmax,

    padded to ``cap`` token rows and ``rows`` requests (padding on the
    executor's scratch sequence slot).  ``x_in`` / ``x_out`` are the fixed
    hand-off buffers the previous / next stage reads and writes."""

    def __init__(self, ex: LlamaExecutor, cap: int, rows: int, embed: bool, layers: bool, head: bool):
        import torch
        self.ex, self.cap, self.rows = ex, cap, rows
        self.embed_, self.layers_, self.head_ = embed, layers, head
        dev = ex.torch_device
        d = ex.cfg.d_model
        self.d_in = torch.zeros(3 * cap + rows, dtype=torch.int32, device=dev)
        self.h_in = torch.zeros(3 * cap + rows, dtype=torch.int32).pin_memory()
        self.x_in = torch.zeros((cap, d), dtype=torch.float32, device=dev)
        self.x_out = torch.zeros((cap, d), dtype=torch.float32, device=dev)
        self.h_out = torch.zeros(rows, dtype=torch.int32).pin_memory()
        self.graph = None
        self.tok = None

    def _body(self):
        c, r = self.cap, self.rows
        toks, pos, seq = self.d_in[:c], self.d_in[c:2 * c], self.d_in[2 * c:3 * c]
        x = self.ex.embed(toks) if self.embed_ else self.x_in.clone()
        if self.layers_:
            for l in range(self.ex.layer_lo, self.ex.layer_hi + 1):
                x = self.ex.layer(l, x, pos, seq)
        if self.head_:
            last = self.d_in[3 * c:3 * c + r].long()
            logits = self.ex.head(x.index_select(0, last).contiguous())
            tok, _ = self.ex.greedy(logits)
            return tok
        self.x_out.copy_(x)
        return None

    def capture(self):
        import torch
        c = self.cap
        self.d_in[2 * c:3 * c].fill_(self.ex.scratch_seq)
        with torch.cuda.device(self.ex.device):
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self._body()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = torch.cuda.CUDAGraph()
            N.lib().lp_set_pdl(1)
            try:
                with torch.cuda.graph(self.graph, stream=torch.cuda.Stream(device=self.ex.device)):
                    self.tok = self._body()
            finally:
                N.lib().lp_set_pdl(0)
            _upload(self.graph)

    def stage_inputs(self, tokens, pos, seq, last):
        c = self.cap
        n, m = len(tokens), len(last)
        buf = self.h_in.numpy()
        buf[:n] = tokens
        buf[n:c] = 0
        buf[c:c + n] = pos
        buf[c + n:2 * c] = 0
        buf[2 * c:2 * c + n] = seq
        buf[2 * c + n:3 * c] = self.ex.scratch_seq
        buf[3 * c:3 * c + m] = last
        buf[3 * c + m:] = 0
        self.d_in.copy_(self.h_in, non_blocking=True)


class PipelineGraph:
    """Graph-replayed forward of an execution pipeline: one SegmentGraph per
    stage (the vocab stage embeds; a separate head segment on the vocab
    device closes the ring) with NVLink hand-offs (``lp_handoff``) between
    devices, ordered by CUDA events — no host round trip inside a step."""

    def __init__(self, stage_execs: list, vocab_exec: LlamaExecutor, cap: int, rows: int):
        self.cap, self.rows = cap, rows
        self.segs = []
        for i, ex in enumerate(stage_execs):
            self.segs.append(SegmentGraph(ex, cap, rows, embed=(i == 0), layers=ex.layer_lo <= ex.layer_hi,
                                          head=False))
        self.head = SegmentGraph(vocab_exec, cap, rows, embed=False, layers=False, head=True)

    def capture(self):
        for g in self.segs + [self.head]:
            g.capture()

    def _handoff(self, src, dst):
        import torch
        sdev, ddev = src.device.index, dst.device.index
        if sdev == ddev:
            with torch.cuda.device(sdev):
                dst.copy_(src)
            return
        with torch.cuda.device(sdev):
            N.check(N.lib().lp_handoff(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                                       src.numel() * src.element_size(), None, 0, None,
                                       C.c_void_p(torch.cuda.current_stream(sdev).cuda_stream)), "lp_handoff")
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(sdev))
        torch.cuda.current_stream(ddev).wait_event(ev)

    def step(self, tokens, pos, seq, last):
        """One ragged batch through the ring; returns the next token per
        request (pinned host tensor, valid once the vocab device is synced)."""
        import torch
        if len(tokens) > self.cap or len(last) > self.rows:
            raise ValueError("batch larger than the captured pipeline graph")
        if self.head.graph is None:
            self.capture()
        prev = None
        for g in self.segs:
            with torch.cuda.device(g.ex.device):
                g.stage_inputs(tokens, pos, seq, last)
                if prev is not None:
                    self._handoff(prev, g.x_in)
                g.graph.replay()
            prev = g.x_out
        h = self.head
        with torch.cuda.device(h.ex.device):
            h.stage_inputs(tokens, pos, seq, last)
            self._handoff(prev, h.x_in)
            h.graph.replay()
            h.h_out.copy_(h.tok, non_blocking=True)
        return h.h_out[:len(last)]
