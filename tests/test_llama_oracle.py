"""Pin the logits oracle (oracle/llama.py) against transformers'
LlamaForCausalLM fp32 outputs stored by tests/golden/make_llama_golden.py."""
import os

import numpy as np

from oracle import dataplane as D
from oracle import llama as OL
from paper_2502_09922_b200 import image as I

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "llama_tiny.npz")


def test_oracle_matches_transformers_logits_and_greedy():
    g = np.load(GOLD)
    cfg = I.CONFIGS["tiny"]
    lay = I.build_layout(cfg, 4)
    W = OL.weights(lay, D.fill_image(lay, int(g["seed"])))
    _, logits = OL.forward(cfg, W, g["prompt"])
    logits = logits.numpy()
    assert np.abs(logits[-4:] - g["last_logits"]).max() < 1e-4
    assert (np.argsort(-logits, axis=1)[:, :1] == g["top8_idx"][:, :1]).all()
    gen, margins = OL.greedy(cfg, W, g["prompt"], 4)
    assert gen == g["greedy"][:4].tolist()
    assert len(set(g["greedy"].tolist())) > 6          # non-degenerate continuation
