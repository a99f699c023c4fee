"""Cluster shape, the scale-out trigger and the step-time model — the
hot-path subset of ``blockcast.simengine`` (pkg/src/blockcast/simengine.py).

On one B200 box a reference *node* is one GPU:
``ClusterSpec(node_count=8, gpus_per_node=1, nic_Bps=900e9, h2d_Bps=64e9)``
is the NVLink-5 / PCIe-Gen5 instance of the reference's cost constants.
The discrete-event loop itself is replaced by real execution
(:mod:`.scaleout`, :mod:`.serving`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import InvalidArgumentError
from .multicast import BlockPlan, MulticastSchedule, SubGroup, Transfer

STRATEGIES = ("lambda_scale", "binary_tree", "broadcast_groups", "ssd_only", "ideal")


@dataclass(frozen=True)
class ClusterSpec:
    """Hardware shape and cost constants (simengine.py:40-60)."""

    node_count: int = 8
    gpus_per_node: int = 1
    gpu_mem_bytes: float = 80e9
    host_mem_bytes: float = 1e12
    nic_Bps: float = 50e9
    nvlink_Bps: float = 400e9
    h2d_Bps: float = 64e9
    ssd_Bps: float = 5e9
    step_fixed_overhead_s: float = 0.005
    baseline_group_init_s: float = 0.6

    def __post_init__(self):
        if self.node_count < 1 or self.gpus_per_node < 1:
            raise InvalidArgumentError("cluster needs at least one node and one device")
        for attr in ("nic_Bps", "nvlink_Bps", "h2d_Bps", "ssd_Bps"):
            if getattr(self, attr) <= 0:
                raise InvalidArgumentError(f"{attr} must be positive")


def b200_box(**overrides) -> ClusterSpec:
    """One 8×B200 HGX box in reference terms: a node per GPU, NVLink as the fabric."""
    spec = dict(node_count=8, gpus_per_node=1, gpu_mem_bytes=180e9, nic_Bps=900e9,
                nvlink_Bps=900e9, h2d_Bps=64e9, step_fixed_overhead_s=1e-5)
    spec.update(overrides)
    return ClusterSpec(**spec)


@dataclass(frozen=True)
class AutoscalePolicy:
    threshold_hi: float = 2.0
    keep_alive_s: float = 15.0
    min_replicas: int = 0
    capacity_per_replica: int = 4
    eval_interval_s: float = 0.1


@dataclass(frozen=True)
class ScaleDecision:
    scale_out: int = 0
    scale_in: int = 0


def autoscale(policy: AutoscalePolicy, queue_depth: int, active_replicas: int,
              idle_s: float = 0.0) -> ScaleDecision:
    """Grow on backlog per replica, shrink on idleness (simengine.py:78-92)."""
    per = max(1, policy.capacity_per_replica)
    grow = 0
    if active_replicas == 0:
        if queue_depth > 0:
            grow = math.ceil(queue_depth / per)
    elif queue_depth / active_replicas > policy.threshold_hi:
        grow = max(0, math.ceil((queue_depth - active_replicas * per) / per))
    shrink = int(queue_depth == 0 and idle_s >= policy.keep_alive_s
                 and active_replicas > policy.min_replicas)
    return ScaleDecision(grow, shrink)


def transfer_step_time(schedule: MulticastSchedule, plan: BlockPlan, cluster: ClusterSpec) -> float:
    """Modelled seconds per lockstep step: ovh + mean block × degree / fabric BW."""
    return cluster.step_fixed_overhead_s + \
        plan.mean_block_bytes() * schedule.max_send_degree / cluster.nic_Bps


def baseline_schedule(strategy: str, nodes: list, plan: BlockPlan, cluster: ClusterSpec) -> MulticastSchedule:
    """Comparator schedules of the reference (simengine.py:106-151), executed
    for real by the multicast engine (tools/compare_strategies.py):

    * ``binary_tree`` — static breadth-first tree (FaaSNet-style), block j
      crosses into node i at step j + depth(i) - 1, parents feed both children
      in the same step (``max_send_degree = 2``);
    * ``broadcast_groups`` — per-block recursive-doubling broadcast behind a
      one-time group-formation delay (NCCL-style), no step bound;
    * ``ssd_only`` / ``ideal`` — no network plan, one group per node.
    """
    order = tuple(bl.block_id for bl in plan.blocks)
    nblk = len(order)
    n = len(nodes)
    if strategy == "binary_tree":
        depth = [0] * n
        for i in range(1, n):
            depth[i] = depth[(i - 1) // 2] + 1
        horizon = nblk + max(depth) - 1 if n > 1 else 0
        steps = []
        for st in range(horizon):
            steps.append([Transfer(st, nodes[(i - 1) // 2], nodes[i], order[st - depth[i] + 1])
                          for i in range(1, n) if 0 <= st - depth[i] + 1 < nblk])
        return MulticastSchedule((SubGroup(0, tuple(nodes), order),), steps, max_send_degree=2, label=strategy)
    if strategy == "broadcast_groups":
        rounds = max(1, math.ceil(math.log2(n))) if n > 1 else 0
        steps = []
        for blk in order:
            for d in range(rounds):
                idx = len(steps)
                steps.append([Transfer(idx, nodes[p], nodes[p + (1 << d)], blk)
                              for p in range(1 << d) if p + (1 << d) < n])
        return MulticastSchedule((SubGroup(0, tuple(nodes), order),), steps, enforce_step_bound=False,
                                 initial_delay_s=cluster.baseline_group_init_s, label=strategy)
    if strategy in ("ssd_only", "ideal"):
        return MulticastSchedule(tuple(SubGroup(i, (x,), order) for i, x in enumerate(nodes)), [], label=strategy)
    raise InvalidArgumentError(f"unknown strategy {strategy!r}")
