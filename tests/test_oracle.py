"""Oracle pinning + CPU data-plane parity (no GPU).

* the C generator/checksum equal an independent numpy restatement;
* executing the reference's own golden schedule lines on host buffers
  delivers every block byte-exactly to every receiver;
* the reference test-suite oracles (BFS optimality, replayed arrivals) agree
  with the drop-in planner.
"""
import numpy as np
import pytest

from oracle import dataplane as D
from oracle import planner_checks as O
from paper_2502_09922_b200 import image as I
from paper_2502_09922_b200 import multicast as M

MASK = np.uint64(0xFFFFFFFFFFFFFFFF)


def np_mix64(z):
    with np.errstate(over="ignore"):
        z = (z + np.uint64(0x9E3779B97F4A7C15)) & MASK
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & MASK
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & MASK
        return z ^ (z >> np.uint64(31))


def np_fill(numel, tid, seed, e):
    i = np.arange(numel, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np_mix64(np.uint64(seed) + (np.uint64(tid + 1) << np.uint64(40)) + i)
    v = (z >> np.uint64(48)).astype(np.int64) - 32768
    f = (v.astype(np.float32) * np.float32(2.0 ** (e - 15))).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    return ((u + (((u >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF))) >> np.uint64(16)).astype(np.uint16)


def test_generator_matches_numpy_restatement():
    for tid, seed, e in [(0, 0, 0), (5, 123, -4), (77, 2**40 + 3, -7)]:
        got = D.fill_tensor(10007, tid, seed, 0, e)
        assert np.array_equal(got, np_fill(10007, tid, seed, e))
    assert (D.fill_tensor(9, 1, 0, 1, 0) == 0x3F80).all()
    assert (D.fill_tensor(9, 1, 0, 2, 0) == 0).all()


def test_checksum_matches_numpy_restatement():
    buf = np.random.default_rng(0).integers(0, 256, 1 << 16, dtype=np.uint8)
    w = buf.view(np.uint64)
    k = np.arange(w.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        want = int(np_mix64(w ^ (k * np.uint64(0x9E3779B97F4A7C15))).sum(dtype=np.uint64))
    assert D.checksum(buf) == want
    buf2 = buf.copy()
    buf2[1234] ^= 1
    assert D.checksum(buf2) != want


@pytest.mark.parametrize("n,k,b", [(4, 1, 4), (4, 2, 4), (5, 1, 4), (8, 2, 4), (3, 1, 2)])
def test_cpu_execution_of_golden_schedule_is_byte_exact(golden, n, k, b):
    rec = next(r for r in golden("schedules")["grid"] if (r["n"], r["k"], r["b"]) == (n, k, b)) \
        if any((r["n"], r["k"], r["b"]) == (n, k, b) for r in golden("schedules")["grid"]) else None
    lay = I.build_layout(I.CONFIGS["tiny"], b)
    src = D.fill_image(lay, seed=0)
    if rec is None:
        pl = M.partition_blocks(M.ModelSpec("m", 26 * 10**9, 80), b)
        g = M.attach_orders(M.partition_subgroups(list(range(n)), list(range(k))), M.k_way_orders(b, k))
        lines = M.schedule_to_lines(M.compose_schedule(g, pl))
    else:
        lines = rec["schedule_lines"]
    images = [src.copy() if i < k else np.zeros_like(src) for i in range(n)]
    D.execute(images, lay.block_offsets, lay.block_lengths, lines, list(range(k)), threads=4)
    want = D.block_checksums(src, lay.block_offsets, lay.block_lengths)
    for i in range(n):
        assert D.block_checksums(images[i], lay.block_offsets, lay.block_lengths) == want
        assert np.array_equal(images[i], src)


def test_cpu_execution_rejects_causality_breach():
    lay = I.build_layout(I.CONFIGS["tiny"], 2)
    imgs = [np.zeros(lay.weights_bytes, np.uint8) for _ in range(3)]
    with pytest.raises(RuntimeError):
        D.execute(imgs, lay.block_offsets, lay.block_lengths, ["0,1,2,0"], [0])


def test_builder_is_optimal_by_exhaustive_search():
    # reference acceptance criterion 3 (test_acceptance.py:73-81)
    for size in (2, 3, 4):
        for b in (1, 2, 3):
            plan = M.partition_blocks(M.ModelSpec("m", 26 * 10**9, 80), b)
            built = len(M.build_binomial_schedule(M.SubGroup(0, tuple(range(size)), tuple(range(b))), plan))
            assert built == O.min_multicast_steps(size, b)


def test_arrivals_agree_with_replay_and_zero_redundancy():
    for n, k, b in [(8, 1, 16), (9, 1, 16), (8, 2, 16), (7, 3, 5), (16, 4, 32)]:
        plan = M.partition_blocks(M.ModelSpec("m", 26 * 10**9, 80), b)
        g = M.attach_orders(M.partition_subgroups(list(range(n)), list(range(k))), M.k_way_orders(b, k))
        s = M.compose_schedule(g, plan)
        rep = O.arrivals_by_replay(s.steps)
        arr = s.arrival_steps()
        for node, blocks in rep.items():
            assert blocks == {bk: st for bk, st in arr[node].items() if st >= 0}
        # every receiver gets every block exactly once (SURVEY §0 finding 2)
        seen = set()
        for row in s.steps:
            for t in row:
                assert (t.receiver, t.block_id) not in seen
                seen.add((t.receiver, t.block_id))
        assert len(seen) == (n - k) * b


def test_image_layout_covers_partition_blocks():
    for name in ("tiny", "llama3-8b", "llama2-13b", "llama3-70b"):
        cfg = I.CONFIGS[name]
        for b in sorted({1, 4, min(16, cfg.n_layers), cfg.n_layers}):
            lay = I.build_layout(cfg, b)
            assert lay.block_offsets[0] == 0
            for o, n, o2 in zip(lay.block_offsets, lay.block_lengths, lay.block_offsets[1:] + [lay.weights_bytes]):
                assert o + n == o2 and o % 256 == 0 and n % 256 == 0
            assert sum(t.numel for t in lay.tensors) == cfg.param_count()
            for t in lay.tensors:
                if t.layer >= 0:
                    blk = lay.plan.blocks[t.block]
                    assert blk.layer_lo <= t.layer <= blk.layer_hi
    assert I.CONFIGS["llama3-8b"].param_count() == 8_030_261_248
    assert I.CONFIGS["llama2-13b"].param_count() == 13_015_864_320
    assert I.CONFIGS["llama3-70b"].param_count() == 70_553_706_496
    assert I.CONFIGS["llama2-7b"].param_count() == 6_738_415_616
