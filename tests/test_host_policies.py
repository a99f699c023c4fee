"""Host-side serving and kernel-launch policies (CPU only).

* ``Server._admit``: FIFO admission into the active unit with the most free
  slots — with the reference's one slot per unit (simengine.py:236,
  ``batch_slots = 1``) this is exactly its unit-order fill
  (simengine.py:356-368); with multi-slot replicas a burst is spread.
* ``llama.gemm_split``: K splits for the residual-add GEMM (decode as
  measured, prefill by wave efficiency over the 148-SM / 74-pair grid).
"""
from collections import deque

import pytest

from paper_2502_09922_b200 import llama as L
from paper_2502_09922_b200.serving import Request, Server, Unit
from paper_2502_09922_b200.workload import TraceRecord


def _server(unit_slots):
    srv = object.__new__(Server)          # admission needs only the unit table
    srv.units = {i: Unit(i, "local", [], s, True, active=True) for i, s in enumerate(unit_slots)}
    return srv


def _queue(n):
    return deque(Request(TraceRecord(f"r{i}", 0.001 * i, "m", 4, 2), [1, 2, 3, 4]) for i in range(n))


def test_admission_single_slot_units_follow_unit_order():
    srv = _server([1, 1, 1])
    q = _queue(5)
    srv._admit(q)
    assert [srv.units[u].busy[0].rid for u in range(3)] == ["r0", "r1", "r2"]
    assert [r.rid for r in q] == ["r3", "r4"]            # the rest wait, FIFO


def test_admission_spreads_a_burst_over_replicas():
    srv = _server([16, 16])
    q = _queue(20)
    srv._admit(q)
    assert len(srv.units[0].busy) == 10 and len(srv.units[1].busy) == 10
    assert not q
    srv.units[0].retired = True                        # retired units take nothing
    q = _queue(3)
    srv._admit(q)
    assert len(srv.units[0].busy) == 10 and len(srv.units[1].busy) == 13


def test_admission_respects_capacity_and_inactive_units():
    srv = _server([2, 2])
    srv.units[1].active = False
    q = _queue(5)
    srv._admit(q)
    assert len(srv.units[0].busy) == 2 and not srv.units[1].busy and len(q) == 3
    for r in srv.units[0].busy.values():
        assert r.unit == 0 and r.needs_prefill and r.kv_len == 0


def test_gemm_split_policy(monkeypatch):
    # decode: ~160 CTAs of one wave (profiles/gemm_split_sweep_r01.txt), >= 4 k-blocks per split
    assert L.gemm_split(6144, 4096, 16) == 3
    assert L.gemm_split(4096, 14336, 1) == 5
    assert L.gemm_split(32000, 256, 8) == 1
    # prefill beyond one wave of pair tiles with the kernel's stream-K tail
    # (default): no split (WO T = 2048: 128 tiles for 74 slots)
    assert L.GEMM_PAIR_STREAMK
    for n, k, t in ((4096, 4096, 2048), (4096, 14336, 4096), (10240, 8192, 1024)):
        assert L.gemm_split(n, k, t) == 1
    assert L.gemm_split(6144, 4096, 256) == 3      # below one wave: split-K as before
    monkeypatch.setattr(L, "GEMM_PAIR_STREAMK", False)   # LP_GEMM_PAIR_STREAMK=0: wave-efficiency split
    # prefill: QKV at T = 256 has 24 pair tiles for 74 cluster slots -> split
    assert L.gemm_split(6144, 4096, 256) == 3
    # >= 2 waves of tiles: never split (T = 4096, 8B shapes)
    for n, k in ((6144, 4096), (4096, 4096), (4096, 14336)):
        assert L.gemm_split(n, k, 4096) == 1
    # every split keeps >= 8 k-blocks of 64
    for n, k, t in ((1536, 512, 300), (640, 1024, 130), (10240, 8192, 256)):
        s = L.gemm_split(n, k, t)
        assert s == 1 or (k // 64) // s >= 8
    assert L.gemm_token_tile(1) == 16 and L.gemm_token_tile(65) == 128 and L.gemm_token_tile(129) == 256


def test_fit_ctas_shares_one_device(monkeypatch):
    """Several schedule nodes on one device (tests, host-fed boxes): the
    per-node CTA counts shrink so every CTA of the dataflow is co-resident."""
    import torch
    from paper_2502_09922_b200 import engine as E

    class Props:
        multi_processor_count = 148
    monkeypatch.setattr(torch.cuda, "get_device_properties", lambda d: Props())
    assert E._fit_ctas(0, 4, 0, 32) == (0, 32)            # fits: unchanged
    assert E._fit_ctas(0, 5, 0, 32) == (0, 29)            # 160 > 148
    push, pull = E._fit_ctas(0, 5, 16, 16)
    assert push >= 1 and pull >= 1 and 5 * (push + pull) <= 148
    assert E._fit_ctas(0, 74, 1, 1) == (1, 1)
    with pytest.raises(ValueError):
        E._fit_ctas(0, 200, 0, 1)


def test_pipeline_prefill_budget():
    """Pipeline passes prefill ~8.2 TFLOP of prompt: 510 tokens for
    Llama-3-8B, fewer than one 128-token prompt for 70B (so one request per
    pass); an explicit budget wins.  AutoscaleServer sets the same budget
    (it does not run Server.__init__)."""
    import inspect
    from paper_2502_09922_b200 import autoscaler as A
    from paper_2502_09922_b200 import image as I
    from paper_2502_09922_b200.serving import Server
    assert Server.prefill_budget(I.build_layout(I.CONFIGS["llama3-8b"], 16)) == 510
    assert Server.prefill_budget(I.build_layout(I.CONFIGS["llama3-70b"], 16)) < 128
    assert Server.prefill_budget(I.build_layout(I.CONFIGS["llama3-8b"], 16), 64) == 64
    src = inspect.getsource(A.AutoscaleServer.__init__)
    assert "pipeline_prefill_tokens" in src and "pipeline_batch" in src


def test_pipeline_pass_prefill_budget():
    """A pipeline pass runs every decode and prefills in slot order while they
    fit the token budget, at least one (Server._pipeline_pass)."""
    from types import SimpleNamespace
    from paper_2502_09922_b200.serving import Server

    def req(n, prefill):
        return SimpleNamespace(prompt=[0] * n, out=[], needs_prefill=prefill)
    srv = SimpleNamespace(pipeline_prefill_tokens=300)
    reqs = [req(128, True), req(128, True), req(10, False), req(128, True), req(40, True)]
    got = Server._pipeline_pass(srv, reqs)
    assert got == [reqs[0], reqs[1], reqs[2], reqs[4]]       # 128 + 128 + 40 <= 300; the third 128 waits
    srv.pipeline_prefill_tokens = 64
    got = Server._pipeline_pass(srv, [req(500, True), req(10, True), req(1, False)])
    assert [len(r.prompt) for r in got] == [500, 1]           # one over-budget prompt still runs alone


def test_split_executor_tiles():
    from paper_2502_09922_b200 import scaleout as SO
    t = SO.split_tiles(5, 2 << 20)
    assert t == [SO.SPLIT_CE_TILE, 2 << 20, SO.SPLIT_CE_TILE, 2 << 20, SO.SPLIT_CE_TILE]
