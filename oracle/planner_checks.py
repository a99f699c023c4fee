"""ORACLE (test infrastructure): the reference test-suite's independent
planner oracles, restated (pkg/tests/oracles.py).  Deliberately different
algorithms from the planner: exhaustive search and plain replays."""

from __future__ import annotations


def min_multicast_steps(group_size: int, block_count: int) -> int:
    """Fewest lockstep steps for a 1->L multicast by breadth-first search
    (oracles.py:14-73): per step every node sends <= 1 block it held at step
    start, receives <= 1, no self-sends; non-source nodes are interchangeable."""
    full = (1 << block_count) - 1
    start = (full,) + (0,) * (group_size - 1)

    def canon(state):
        return (state[0],) + tuple(sorted(state[1:]))

    def successors(state):
        found = set()

        def assign(sender, taken, nxt):
            if sender == group_size:
                found.add(canon(tuple(nxt)))
                return
            assign(sender + 1, taken, nxt)
            have = state[sender]
            if not have:
                return
            for r in range(group_size):
                if r == sender or r in taken:
                    continue
                useful = have & ~state[r]
                while useful:
                    low = useful & -useful
                    useful ^= low
                    saved = nxt[r]
                    nxt[r] |= low
                    assign(sender + 1, taken | {r}, nxt)
                    nxt[r] = saved

        assign(0, frozenset(), list(state))
        return found

    goal = (full,) * group_size
    frontier, seen, steps = {canon(start)}, {canon(start)}, 0
    while goal not in frontier:
        nxt = set()
        for st in frontier:
            nxt |= successors(st)
        frontier = nxt - seen
        seen |= frontier
        steps += 1
        if steps > block_count * group_size + 8:
            raise RuntimeError("search runaway")
    return steps


def arrivals_by_replay(steps) -> dict:
    """Per-node last-write arrival replay (oracles.py:127-133)."""
    out: dict = {}
    for idx, row in enumerate(steps):
        for t in row:
            out.setdefault(t.receiver, {})[t.block_id] = idx
    return out


def balanced_contiguous_sizes(total: int, parts: int) -> list:
    base, extra = divmod(total, parts)
    return [base + 1] * extra + [base] * (parts - extra)
