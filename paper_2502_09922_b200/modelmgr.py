"""Tier residency and packed-image layout — the hot-path subset of
``blockcast.modelmgr`` (pkg/src/blockcast/modelmgr.py).

* :func:`startup_plan` picks multicast sources by tier (GPU copies first, then
  host-memory copies, SSD bootstrap last) — modelmgr.py:109-141.
* :func:`pack_layout` lays blocks back to back plus a staging buffer of the
  largest block and a working set — modelmgr.py:238-259.  The CUDA engine
  allocates exactly this layout per GPU (one contiguous image, so each block
  lands with one copy and pipeline stages index it by offset).

Eviction and the cache-replay study (modelmgr.py:144-220) are out of scope
for the scaling hot path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import CapacityError, InvalidArgumentError, UnsatisfiableScalingError
from .multicast import BlockPlan

GPU = "gpu"
MEMORY = "memory"
SSD = "ssd"

HOT = "hot"
WARM = "warm"
COLD = "cold"


@dataclass
class TierState:
    """Residency of one model on one node, per tier (modelmgr.py:26-36)."""

    node: int
    model_id: str
    gpu_blocks: set = field(default_factory=set)
    mem_blocks: set = field(default_factory=set)
    ssd: bool = False
    last_use_s: float = 0.0
    pinned: bool = False


@dataclass
class StartupPlan:
    classes: dict
    sources: list
    bootstrap_node: int | None = None


class TierMap:
    """Every (node, model) residency record of a cluster (modelmgr.py:59-106)."""

    def __init__(self):
        self._by_key: dict = {}

    def get(self, node: int, model_id: str):
        return self._by_key.get((node, model_id))

    def ensure(self, node: int, model_id: str) -> TierState:
        key = (node, model_id)
        if key not in self._by_key:
            self._by_key[key] = TierState(node, model_id)
        return self._by_key[key]

    def states(self) -> list:
        return [self._by_key[key] for key in sorted(self._by_key)]

    def full_nodes(self, model_id: str, tier: str, block_count: int) -> list:
        """Nodes whose ``tier`` copy holds at least ``block_count`` blocks."""
        picked = []
        for (node, mid) in sorted(self._by_key):
            if mid != model_id:
                continue
            st = self._by_key[(node, mid)]
            if tier == GPU:
                ok = len(st.gpu_blocks) >= block_count
            elif tier == MEMORY:
                ok = len(st.mem_blocks) >= block_count
            elif tier == SSD:
                ok = st.ssd
            else:
                ok = False
            if ok:
                picked.append(node)
        return picked

    def to_lines(self) -> list:
        """``node,model,tier,blocks_resident,last_use_s`` per resident tier."""
        lines = []
        for st in self.states():
            for tier, count, present in ((GPU, len(st.gpu_blocks), bool(st.gpu_blocks)),
                                         (MEMORY, len(st.mem_blocks), bool(st.mem_blocks)),
                                         (SSD, -1, st.ssd)):
                if present:
                    lines.append(f"{st.node},{st.model_id},{tier},{count},{st.last_use_s:.6f}")
        return lines


def startup_plan(model_id: str, block_count: int, demand_nodes: list,
                 tiers: TierMap, k_max: int = 1) -> StartupPlan:
    """Classify demand nodes hot/warm/cold and choose up to ``k_max`` sources."""
    if k_max < 1:
        raise InvalidArgumentError("k_max must be >= 1")
    classes = {}
    for node in demand_nodes:
        st = tiers.get(node, model_id)
        if st is not None and len(st.gpu_blocks) >= block_count:
            classes[node] = HOT
        elif st is not None and len(st.mem_blocks) >= block_count:
            classes[node] = WARM
        else:
            classes[node] = COLD
    on_gpu = tiers.full_nodes(model_id, GPU, block_count)
    in_mem = [n for n in tiers.full_nodes(model_id, MEMORY, block_count) if n not in on_gpu]
    chosen = (on_gpu + in_mem)[:k_max]
    boot = None
    if not chosen:
        on_ssd = tiers.full_nodes(model_id, SSD, block_count)
        if not on_ssd:
            raise UnsatisfiableScalingError(
                f"no copy of model {model_id} exists on any node in any tier")
        boot = on_ssd[0]
        chosen = [boot]
    return StartupPlan(classes, chosen, boot)


@dataclass(frozen=True)
class Region:
    block_id: int
    offset: int
    length: int


@dataclass
class MemoryLayout:
    regions: tuple
    activation_buffer_bytes: int
    staging_buffer_bytes: int
    total_bytes: int


def pack_layout(plan: BlockPlan, working_set_bytes: int,
                capacity_bytes: int | None = None) -> MemoryLayout:
    """Blocks back to back in block order + working set + max-block staging."""
    if working_set_bytes < 0:
        raise InvalidArgumentError("working_set_bytes must be >= 0")
    regions = []
    cursor = 0
    for blk in plan.blocks:
        regions.append(Region(blk.block_id, cursor, blk.size_bytes))
        cursor += blk.size_bytes
    staging = max(blk.size_bytes for blk in plan.blocks)
    total = cursor + working_set_bytes + staging
    if capacity_bytes is not None and total > capacity_bytes:
        raise CapacityError(f"layout needs {total} bytes, device offers {capacity_bytes} "
                            f"(deficit {total - capacity_bytes})")
    return MemoryLayout(tuple(regions), working_set_bytes, staging, total)
