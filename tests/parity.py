"""Greedy-token parity helpers shared by the GPU tests and the smoke.

The prompts come from tests/golden/prompts_tiny.json (make_prompts.py): for
each of them the bf16-faithful oracle's top-1/top-2 margin clears the gate
at EVERY generated position, so every position is compared — no margin-gated
early exit — and :func:`assert_tokens` fails a check that compares nothing.
"""
from __future__ import annotations

import json
import os

FIXTURE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "prompts_tiny.json")
_DOC = None


def doc() -> dict:
    global _DOC
    if _DOC is None:
        with open(FIXTURE) as fh:
            _DOC = json.load(fh)
    return _DOC


def entries(n: int, max_prompt: int = 1 << 30) -> list:
    """``n`` fixture entries (cycled), prompts at most ``max_prompt`` tokens."""
    pool = [e for e in doc()["prompts"] if len(e["prompt"]) <= max_prompt]
    assert pool, "no fixture prompt fits"
    return [pool[i % len(pool)] for i in range(n)]


def assert_tokens(got, entry, n: int | None = None, what: str = "") -> int:
    """Every one of the first ``n`` generated tokens equals the oracle's
    (all of them when n is None).  Returns the number of positions compared."""
    want = entry["greedy"] if n is None else entry["greedy"][:n]
    assert len(want) > 0, "a parity check must compare at least one token"
    assert len(got) >= len(want), f"{what}: generated {len(got)} tokens, expected {len(want)}"
    got = list(got)[:len(want)]
    assert got == want, f"{what}: greedy tokens differ from the oracle\n got  {got}\n want {want}\n " \
                        f"margins {entry['margins'][:len(want)]}"
    return len(want)
