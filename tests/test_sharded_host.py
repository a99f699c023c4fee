"""Host-side properties of the sharded host-load schedule (CPU)."""
import pytest

from paper_2502_09922_b200 import multicast as M
from paper_2502_09922_b200 import scaleout as SO


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 9])
@pytest.mark.parametrize("b", [1, 3, 16, 40])
def test_sharded_host_schedule_properties(n, b):
    plan = SO.plan_scale_out("llama2-13b", n, 1, b, host_source=True, strategy="sharded_host")
    sched = plan.schedule
    assert M.validate_schedule(sched) == []
    G = n - 1
    rows = [t for row in sched.steps for t in row]
    # every GPU receives every block exactly once, the host sends each block once
    for gpu in range(1, n):
        got = sorted(t.block_id for t in rows if t.receiver == gpu)
        assert got == list(range(b))
    host = [t for t in rows if t.sender == 0]
    assert sorted(t.block_id for t in host) == list(range(b))
    # block j comes from the host to its owner 1 + j % G; owners relay only their own blocks
    for t in host:
        assert t.receiver == 1 + t.block_id % G
    for t in rows:
        if t.sender != 0:
            assert t.sender == 1 + t.block_id % G
    # each GPU sends and receives at most one block per step
    for row in sched.steps:
        rcv = [t.receiver for t in row]
        snd = [t.sender for t in row if t.sender != 0]
        assert len(rcv) == len(set(rcv)) and len(snd) == len(set(snd))
    assert plan.pipelines == [] and plan.strategy == "sharded_host"


def test_strategy_policy_and_errors():
    assert SO.choose_strategy(True, 1) == "lambda"
    assert SO.choose_strategy(True, 4) == "sharded_host"
    assert SO.choose_strategy(False, 8) == "lambda"
    with pytest.raises(ValueError):
        SO.plan_scale_out("tiny", 4, strategy="sharded_host")
    with pytest.raises(ValueError):
        SO.plan_scale_out("tiny", 4, host_source=True, strategy="tree")
