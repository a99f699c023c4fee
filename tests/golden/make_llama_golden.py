"""Pin the logits oracle against transformers' LlamaForCausalLM (run HERE).

    python tests/golden/make_llama_golden.py

Builds the tiny config's packed image with the oracle generator (seed 7),
loads the same bf16 weights (as fp32) into transformers 5.5
LlamaForCausalLM, and stores its logits + greedy continuation in
tests/golden/llama_tiny.npz.  The GPU box never runs this script.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

SEED = 7
PROMPT_LEN = 24
STEPS = 12


def main():
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    from oracle import dataplane as D
    from oracle import llama as OL
    from paper_2502_09922_b200 import image as I

    cfg = I.CONFIGS["tiny"]
    lay = I.build_layout(cfg, 4)
    img = D.fill_image(lay, SEED)
    W = OL.weights(lay, img)
    hf_cfg = LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model, intermediate_size=cfg.ffn,
                         num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
                         num_key_value_heads=cfg.n_kv_heads, rms_norm_eps=cfg.norm_eps, rope_theta=cfg.rope_theta,
                         max_position_embeddings=2048, tie_word_embeddings=False, attention_bias=False,
                         mlp_bias=False, torch_dtype="float32")
    model = LlamaForCausalLM(hf_cfg).float().eval()
    sd = {"model.embed_tokens.weight": W["embed"], "model.norm.weight": W["final_norm"], "lm_head.weight": W["lm_head"]}
    names = {"attn_norm": "input_layernorm", "ffn_norm": "post_attention_layernorm", "wq": "self_attn.q_proj",
             "wk": "self_attn.k_proj", "wv": "self_attn.v_proj", "wo": "self_attn.o_proj",
             "w_gate": "mlp.gate_proj", "w_up": "mlp.up_proj", "w_down": "mlp.down_proj"}
    for l in range(cfg.n_layers):
        for ours, theirs in names.items():
            sd[f"model.layers.{l}.{theirs}.weight"] = W[f"layers.{l}.{ours}"]
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and all("rotary" in m for m in missing), (missing, unexpected)
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, PROMPT_LEN).astype(np.int64)
    with torch.no_grad():
        hf_logits = model(torch.as_tensor(prompt)[None]).logits[0].float().numpy()
        gen = model.generate(torch.as_tensor(prompt)[None], max_new_tokens=STEPS, do_sample=False,
                             pad_token_id=0)[0, PROMPT_LEN:].numpy()
    _, ours = OL.forward(cfg, W, prompt)
    print("oracle vs transformers max |dlogit|:", float(np.abs(ours.numpy() - hf_logits).max()))
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "llama_tiny.npz"),
                        prompt=prompt, seed=SEED, last_logits=hf_logits[-4:].astype(np.float32),
                        top8_idx=np.argsort(-hf_logits, axis=1)[:, :8].astype(np.int32),
                        top8_val=np.sort(hf_logits, axis=1)[:, ::-1][:, :8].astype(np.float32),
                        greedy=gen.astype(np.int32))
    print("greedy:", gen.tolist())


if __name__ == "__main__":
    main()
