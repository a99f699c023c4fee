"""Llama model shapes and the packed per-GPU weight image.

The reference moves abstract blocks whose byte sizes are layer-proportional
(``partition_blocks``, multicast.py:153-173) and packs them back to back with a
staging buffer (``pack_layout``, modelmgr.py:238-259).  Here the blocks hold
real bf16 tensors of a Llama decoder, laid out so that

* block ``i`` covers exactly the decoder layers of ``partition_blocks``'s
  block ``i`` (``layer_lo..layer_hi``) — execution stages index it directly;
* the vocabulary tensors (token embedding, final RMSNorm, LM head) are packed
  into block 0 ahead of its layers.  Block 0 is injected first by every k=1
  source and is the stage that closes the cyclic pipeline (embedding in,
  logits out), while the last block — the one the binomial schedule's source
  re-sends ``ceil(log2 L) - 1`` extra times (multicast.py:360-364) — stays a
  plain layer block;
* every tensor starts 256-byte aligned, so blocks are 16-byte-vector and
  TMA-friendly and a block lands with one contiguous copy.

The image is one device allocation per GPU: ``[blocks | working set |
staging]`` in ``pack_layout`` order, followed by the multicast signal area.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .multicast import BlockPlan, ModelSpec, partition_blocks

ALIGN = 256


@dataclass(frozen=True)
class LlamaConfig:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    def layer_params(self) -> int:
        d, f, kv = self.d_model, self.ffn, self.kv_dim
        return 2 * d + d * d + 2 * d * kv + d * d + 3 * d * f

    def param_count(self) -> int:
        return self.n_layers * self.layer_params() + 2 * self.vocab * self.d_model + self.d_model

    def bf16_bytes(self) -> int:
        return 2 * self.param_count()


# SURVEY.md §8 config table (standard architectures; bf16 = 2 B/param)
CONFIGS = {
    "tiny": LlamaConfig("tiny", 4, 256, 4, 2, 688, 32000, 10000.0),
    "llama3-8b": LlamaConfig("llama3-8b", 32, 4096, 32, 8, 14336, 128256, 500000.0),
    "llama2-13b": LlamaConfig("llama2-13b", 40, 5120, 40, 40, 13824, 32000, 10000.0),
    "llama3-70b": LlamaConfig("llama3-70b", 80, 8192, 64, 8, 28672, 128256, 500000.0),
    "llama2-7b": LlamaConfig("llama2-7b", 32, 4096, 32, 32, 11008, 32000, 10000.0),
}

KIND_RANDOM, KIND_ONES, KIND_ZEROS = 0, 1, 2
LAYER_TENSORS = ("attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")


@dataclass(frozen=True)
class TensorSlot:
    index: int          # generator tensor id (canonical order)
    name: str           # e.g. "layers.3.wq", "embed", "lm_head"
    layer: int          # -1 for vocabulary tensors
    block: int
    offset: int         # bytes from the image base
    shape: tuple        # (rows, cols) row-major, or (n,)
    kind: int
    scale_exp: int

    @property
    def numel(self) -> int:
        return math.prod(self.shape)

    @property
    def nbytes(self) -> int:
        return 2 * self.numel


@dataclass
class ImageLayout:
    config: LlamaConfig
    plan: BlockPlan
    tensors: list
    block_offsets: list
    block_lengths: list
    weights_bytes: int
    by_name: dict = field(default_factory=dict)

    def block_of_layer(self, layer: int) -> int:
        for blk in self.plan.blocks:
            if blk.layer_lo <= layer <= blk.layer_hi:
                return blk.block_id
        raise KeyError(layer)


def _align(x: int) -> int:
    return (x + ALIGN - 1) // ALIGN * ALIGN


def _scale_exp(fan_in: int) -> int:
    """Uniform[-2^e, 2^e) has std 2^e/sqrt(3); pick e so std ~ 1/sqrt(fan_in)."""
    return round(math.log2(math.sqrt(3.0 / fan_in)))


def model_spec(cfg: LlamaConfig, **kw) -> ModelSpec:
    """The reference ModelSpec of a config (size = real bf16 bytes)."""
    return ModelSpec(cfg.name, cfg.bf16_bytes(), cfg.n_layers, **kw)


def layer_tensor_shapes(cfg: LlamaConfig) -> list:
    d, f, kv = cfg.d_model, cfg.ffn, cfg.kv_dim
    # weights are stored [out_features, in_features] (y = x @ W^T)
    return [("attn_norm", (d,), KIND_ONES, 0), ("wq", (d, d), KIND_RANDOM, _scale_exp(d)),
            ("wk", (kv, d), KIND_RANDOM, _scale_exp(d)), ("wv", (kv, d), KIND_RANDOM, _scale_exp(d)),
            ("wo", (d, d), KIND_RANDOM, _scale_exp(d)), ("ffn_norm", (d,), KIND_ONES, 0),
            ("w_gate", (f, d), KIND_RANDOM, _scale_exp(d)), ("w_up", (f, d), KIND_RANDOM, _scale_exp(d)),
            ("w_down", (d, f), KIND_RANDOM, _scale_exp(f))]


def build_layout(cfg: LlamaConfig, block_count: int) -> ImageLayout:
    """Pack a config's tensors into ``block_count`` blocks (see module doc)."""
    spec = model_spec(cfg)
    plan = partition_blocks(spec, block_count)
    # generator ids follow the canonical order: embed, layers..., norm, lm_head
    ids = {"embed": 0}
    nxt = 1
    for layer in range(cfg.n_layers):
        for name in LAYER_TENSORS:
            ids[f"layers.{layer}.{name}"] = nxt
            nxt += 1
    ids["final_norm"] = nxt
    ids["lm_head"] = nxt + 1
    d, v = cfg.d_model, cfg.vocab
    tensors = []
    offsets, lengths = [], []
    cursor = 0
    for blk in plan.blocks:
        start = cursor
        if blk.block_id == 0:
            for name, shape, kind, e in (("embed", (v, d), KIND_RANDOM, 0),
                                         ("final_norm", (d,), KIND_ONES, 0),
                                         ("lm_head", (v, d), KIND_RANDOM, _scale_exp(d))):
                tensors.append(TensorSlot(ids[name], name, -1, 0, cursor, shape, kind, e))
                cursor = _align(cursor + 2 * math.prod(shape))
        for layer in range(blk.layer_lo, blk.layer_hi + 1):
            for name, shape, kind, e in layer_tensor_shapes(cfg):
                full = f"layers.{layer}.{name}"
                tensors.append(TensorSlot(ids[full], full, layer, blk.block_id, cursor, shape, kind, e))
                cursor = _align(cursor + 2 * math.prod(shape))
        offsets.append(start)
        lengths.append(cursor - start)
    lay = ImageLayout(cfg, plan, tensors, offsets, lengths, cursor)
    lay.by_name = {t.name: t for t in tensors}
    return lay


def fill_args(layout: ImageLayout):
    """Columns for ``lp_fill_tensors``: offsets, numels, kinds, scale exps, generator ids."""
    ts = sorted(layout.tensors, key=lambda t: t.index)
    return ([t.offset for t in ts], [t.numel for t in ts], [t.kind for t in ts],
            [t.scale_exp for t in ts], [t.index for t in ts])
