"""ORACLE — test infrastructure, never part of the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_2502_09922_b200`` never
imports it (tests/test_boundary.py enforces that).

Contents
  dataplane    ctypes binding of oracle/dataplane.c (generator, checksum,
               schedule execution on host buffers)
  planner      pure-Python restatement of the reference planner
               (multicast.py / pipeline.py), pinned against tests/golden/
  llama        CPU fp32 Llama decoder (logits oracle), pinned against
               transformers' LlamaForCausalLM via tests/golden/llama_*.npz

Pinning status: planner = pinned (reference-generated
golden fixtures); dataplane = schedule pinned, bytes self-consistent (the
paper's RDMC transfer module is not vendored: "parity unpinned" for raw
bytes beyond receiver == source); logits = pinned to transformers, not to the
paper's unvendored inference module.
"""
