"""``scale_out``: the reference's λScale launch sequence on real GPUs.

Mirrors ``_Engine._launch_lambda_scale`` (simengine.py:564-602): startup
classes and sources (modelmgr.startup_plan), ``k_eff = min(|sources|, |cold|,
k)``, sub-groups + k-way orders, ``compose_schedule``, completion-ordered
groups, execution pipelines with activation steps — then, instead of pushing
modelled ``transfer_step_done`` events, it executes the schedule with the
CUDA multicast engine and reports measured times.

Two entry points:

* :func:`plan_scale_out` — the reference CLI's numbering (cli.py:308-309):
  ``nodes[:k]`` are the sources; on one box a node is a GPU (rank) and a
  HOST node (pinned memory) is node 0 when the source tier is host memory
  (config C3).
* :func:`plan_from_tiers` / :func:`scale_out` — the simulator's tier-driven
  sequence (simengine.py:442-467 ``_scale_out`` -> ``startup_plan`` ->
  ``_warm_and_hot`` -> ``_launch_lambda_scale``): demand nodes are classified
  hot / warm / cold from a ``TierMap`` (modelmgr.py:109-141), sources are the
  GPU-resident copies first and then host-memory copies (the box's pinned
  host copy is one more node, the HOST node), ``k_eff = min(|sources|,
  |cold|, k)``, and the λPipe plan covers ``sources + cold`` in that order.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

from . import engine as E
from .cluster import ClusterSpec, b200_box, transfer_step_time
from .image import CONFIGS, ImageLayout, LlamaConfig, build_layout, model_spec
from .modelmgr import COLD, GPU, HOT, MEMORY, WARM, StartupPlan, TierMap, startup_plan
from .multicast import (MulticastSchedule, SubGroup, Transfer, attach_orders, compose_schedule,
                        k_way_orders, partition_subgroups, schedule_to_lines, select_block_count)
from .pipeline import assign_blocks_to_stages, completion_ordered_groups, generate_pipelines


@dataclass
class ScaleOutPlan:
    config: LlamaConfig
    layout: ImageLayout
    nodes: list
    sources: list
    groups: list
    schedule: MulticastSchedule
    ordered: list
    pipelines: list
    step_s_model: float
    host_source: bool = False
    strategy: str = "lambda"
    host_nodes: tuple = ()        # positions that are the HOST node (pinned host copy)

    @property
    def block_count(self) -> int:
        return self.layout.plan.block_count

    @property
    def receivers(self) -> list:
        return [n for n in self.nodes if n not in self.sources]

    def lines(self) -> list:
        return schedule_to_lines(self.schedule)


def sharded_host_schedule(n_nodes: int, plan) -> MulticastSchedule:
    """Host-sourced load for GPUs that SHARE the host copy (one box).

    The reference gives every node holding a host-memory copy ("warm") its
    own local h2d load (simengine.py:508-521) and multicasts from a memory
    source only to nodes without one.  On a B200 box all GPUs read the same
    pinned host memory, each over its own PCIe link, so here every GPU loads a
    disjoint shard over its link and the shards are exchanged over NVLink:
    block j is owned by GPU ``1 + j % G`` (G = n_nodes - 1 GPUs, node 0 =
    HOST), arrives from the host at step ``G * (j // G)`` and is forwarded by its
    owner to the other GPUs in a rotation over the next G - 1 steps (one send
    and one receive per GPU per step; only the host sends G per step, one per
    PCIe link).  The engine runs the PCIe and NVLink legs concurrently (steps
    only order each node's ops).  Host egress is spread
    over G PCIe links instead of the binomial tree's ``ceil(log2 n)`` host
    partners (measured 215 GB/s for 4 concurrent links vs 55.6 for one,
    tools/h2d_concurrency.py).  ``max_send_degree = G`` (the host), no step
    bound; validate_schedule accepts it.
    """
    G = n_nodes - 1
    if G < 1:
        raise ValueError("sharded host load needs the HOST node and at least one GPU")
    order = tuple(bl.block_id for bl in plan.blocks)
    rounds = (len(order) + G - 1) // G
    steps = [[] for _ in range(rounds * G)]
    for r in range(rounds):
        blocks = order[r * G:(r + 1) * G]          # block r*G + q is owned by GPU 1 + q
        for q, blk in enumerate(blocks):
            steps[r * G].append(Transfer(r * G, 0, 1 + q, blk))
        for i in range(1, G):                      # rotation: one send and one receive per GPU per step
            for q, blk in enumerate(blocks):
                peer = 1 + (q + i) % G
                steps[r * G + i].append(Transfer(r * G + i, 1 + q, peer, blk))
    while steps and not steps[-1]:
        steps.pop()
    return MulticastSchedule((SubGroup(0, tuple(range(n_nodes)), order),), steps, max_send_degree=G,
                             enforce_step_bound=False, label="sharded_host")


def plan_scale_out(config, n_nodes: int, k: int = 1, block_count="auto",
                   cluster: ClusterSpec | None = None, host_source: bool = False,
                   strategy: str = "lambda", host_nodes: tuple | None = None) -> ScaleOutPlan:
    """Planning half of ``_launch_lambda_scale`` (simengine.py:579-590).

    ``host_nodes``: positions that are the HOST node (default: node 0 when
    ``host_source``); a HOST node must be one of the k sources.
    ``strategy="sharded_host"`` (host sources only) replaces the binomial
    schedule by :func:`sharded_host_schedule`; it has no λPipe pipelines
    (every GPU completes at about the same time)."""
    if host_nodes is None:
        host_nodes = (0,) if host_source else ()
    host_nodes = tuple(host_nodes)
    host_source = bool(host_nodes)
    if strategy not in ("lambda", "sharded_host"):
        raise ValueError("strategy is 'lambda' or 'sharded_host'")
    if strategy == "sharded_host" and not host_source:
        raise ValueError("sharded_host needs host_source=True")
    cfg = CONFIGS[config] if isinstance(config, str) else config
    cluster = cluster or b200_box(node_count=n_nodes)
    spec = model_spec(cfg)
    if block_count == "auto":
        block_count = select_block_count(spec, n_nodes, cluster.step_fixed_overhead_s, cluster.nic_Bps)
    layout = build_layout(cfg, int(block_count))
    nodes = list(range(n_nodes))
    k_eff = max(1, min(k, n_nodes - 1)) if n_nodes > 1 else 1
    sources = nodes[:k_eff]
    if any(h not in sources for h in host_nodes):
        raise ValueError("a HOST node must be one of the sources (positions < k)")
    groups = attach_orders(partition_subgroups(nodes, sources), k_way_orders(layout.plan.block_count, k_eff))
    sched = compose_schedule(groups, layout.plan, cluster.step_fixed_overhead_s, cluster.nic_Bps)
    ordered = completion_ordered_groups(groups, sched)
    orders = [g.transfer_order for g in ordered]
    pipes = generate_pipelines(ordered) if any(g.receivers for g in ordered) else []
    eps = [assign_blocks_to_stages(pn, orders, layout.plan.block_count, sched, i) for i, pn in enumerate(pipes)]
    step_s = transfer_step_time(sched, layout.plan, cluster)
    if strategy == "sharded_host":
        sched = sharded_host_schedule(n_nodes, layout.plan)
        if host_nodes != (0,):
            raise ValueError("sharded_host needs the HOST node at position 0")
        return ScaleOutPlan(cfg, layout, nodes, [0], list(sched.groups), sched, list(sched.groups), [], step_s,
                            host_source, strategy, host_nodes)
    return ScaleOutPlan(cfg, layout, nodes, sources, groups, sched, ordered, eps, step_s, host_source,
                        host_nodes=host_nodes)


@dataclass
class TieredPlan:
    """A tier-driven scale-out (simengine.py:442-467, :507-521, :564-602).

    ``plan`` is the λPipe multicast to the cold nodes over positions
    0..n-1 (``None`` when nothing is cold); ``ref_nodes[i]`` is the
    reference node id at position i (the HOST node's id is ``host_id``).
    Warm demand nodes load locally from host memory (the reference's h2d
    path, ``warm_loads`` rows (block, node) in block order); hot ones serve
    at once."""
    startup: StartupPlan
    hot: list
    warm: list
    cold: list
    sources: list                 # reference ids, after k_eff
    plan: ScaleOutPlan | None
    ref_nodes: list
    host_id: int | None
    # what the engine executes: the λPipe plan plus, when warm nodes load
    # from host memory, their k-way-ordered loads and warm pipeline
    # (warm_pipeline_plan); exec_ref_nodes[i] = reference id of position i
    exec_plan: ScaleOutPlan | None = None
    exec_ref_nodes: list = field(default_factory=list)

    def position(self, ref_node: int) -> int:
        return self.ref_nodes.index(ref_node)

    def ref_lines(self) -> list:
        """The multicast schedule in reference node ids (schedule_to_lines format)."""
        if self.plan is None:
            return []
        rows = sorted((t.step, self.ref_nodes[t.sender], self.ref_nodes[t.receiver], t.block_id)
                      for row in self.plan.schedule.steps for t in row)
        return [f"{a},{b},{c},{d}" for a, b, c, d in rows]


def box_tiers(model_id: str, block_count: int, gpu_resident=(), host_copy: bool = True, host_id: int = 8,
              warm=()) -> TierMap:
    """The residency of one model on a B200 box in the reference's terms: GPU
    node g holds a GPU-tier copy for g in ``gpu_resident``; the box's pinned
    host copy is node ``host_id`` with a MEMORY-tier copy; nodes in ``warm``
    hold a node-local MEMORY copy (they load over their own PCIe link)."""
    tm = TierMap()
    blocks = set(range(block_count))
    for g in gpu_resident:
        tm.ensure(g, model_id).gpu_blocks = set(blocks)
    if host_copy:
        tm.ensure(host_id, model_id).mem_blocks = set(blocks)
    for w in warm:
        tm.ensure(w, model_id).mem_blocks = set(blocks)
    return tm


def plan_from_tiers(config, demand: list, tiers: TierMap, k: int = 1, block_count: int = 16,
                    host_id: int | None = None, cluster: ClusterSpec | None = None) -> TieredPlan:
    """``startup_plan`` -> ``_warm_and_hot`` -> ``_launch_lambda_scale``'s
    planning on reference node ids (simengine.py:450-452, :507-521, :564-590):
    classify ``demand``; sources = GPU copies then MEMORY copies (<= k);
    if every source is itself cold, the first one seeds the rest; ``k_eff =
    min(|sources|, |cold|, k)``; λPipe over ``sources + cold``.  ``host_id``
    names the box's pinned host copy when it is a node of its own; every
    source whose copy is in host memory (that node, or a warm demand node that
    also loads itself, as in the reference) becomes a HOST position of the
    plan — on one box they all read the same pinned host copy."""
    cfg = CONFIGS[config] if isinstance(config, str) else config
    if not isinstance(block_count, int):
        raise ValueError("plan_from_tiers needs an explicit block_count")
    sp = startup_plan(cfg.name, block_count, list(demand), tiers, k_max=k)
    hot = [n for n in demand if sp.classes[n] == HOT]
    warm = [n for n in demand if sp.classes[n] == WARM]
    cold = [n for n in demand if sp.classes[n] == COLD]
    if not cold:
        return TieredPlan(sp, hot, warm, cold, [], None, [], host_id)
    sources = [s for s in sp.sources if s not in cold]
    if not sources:
        sources = sp.sources[:1]
        cold = [n for n in cold if n not in sources]
        if not cold:
            return TieredPlan(sp, hot, warm, cold, sources, None, [], host_id)
    k_eff = min(len(sources), len(cold), k)
    sources = sources[:k_eff]
    ref_nodes = sources + cold
    def tier_of(n):
        st = tiers.get(n, cfg.name)
        if st is not None and len(st.gpu_blocks) >= block_count:
            return GPU
        if st is not None and len(st.mem_blocks) >= block_count:
            return MEMORY
        return None                        # the SSD bootstrap: seeded before the multicast
    # a source whose copy is in host memory sends from it: on one box every
    # such source reads the box's one pinned host copy (the HOST node)
    hosts = tuple(i for i, n in enumerate(sources) if tier_of(n) == MEMORY)
    plan = plan_scale_out(cfg, len(ref_nodes), k_eff, block_count, cluster=cluster, host_nodes=hosts)
    return TieredPlan(sp, hot, warm, cold, sources, plan, ref_nodes, host_id)


def warm_pipeline_plan(tp: TieredPlan, config, block_count: int, cluster: ClusterSpec | None = None) -> TieredPlan:
    """Execution plan with warm-node pipelines (the
    reference simulator specifies but does not implement them, loading warm
    nodes in block order and serving only after the full load,
    simengine.py:507-521).

    The W warm demand nodes load from the host copy in k-way order — warm node
    i first loads chunk i of ``k_way_orders(b, W)`` (multicast.py:246-265),
    each over its own PCIe link — and form one execution pipeline among
    themselves (stage i = chunk i), planned with the reference's own
    ``completion_ordered_groups`` / ``generate_pipelines`` /
    ``assign_blocks_to_stages`` over the warm loads as W one-receiver groups,
    so it activates after about 1/W of the load.  The rows run on the same
    engine as the λPipe multicast (same counters, same activation logic).
    Sets ``tp.exec_plan`` / ``tp.exec_ref_nodes`` and returns ``tp``."""
    cfg = CONFIGS[config] if isinstance(config, str) else config
    base = tp.plan
    if not tp.warm:
        tp.exec_plan, tp.exec_ref_nodes = base, list(tp.ref_nodes)
        return tp
    layout = base.layout if base is not None else build_layout(cfg, block_count)
    b = layout.plan.block_count
    refs = list(tp.ref_nodes) if base is not None else []
    steps = [list(row) for row in base.schedule.steps] if base is not None else []
    groups = list(base.groups) if base is not None else []
    sources = list(base.sources) if base is not None else []
    hosts = list(base.host_nodes) if base is not None else []
    pipes = list(base.pipelines) if base is not None else []
    ordered = list(base.ordered) if base is not None else []
    # warm node i reads its "own host memory" — a HOST position over the one
    # pinned copy per warm node — so every load is a one-receiver sub-group
    # and the λPipe groups stay disjoint
    W = len(tp.warm)
    orders = k_way_orders(b, W)
    hpos = list(range(len(refs), len(refs) + W))
    refs += [tp.host_id if tp.host_id is not None else -1] * W
    sources += hpos
    hosts += hpos
    wpos = list(range(len(refs), len(refs) + W))
    refs += list(tp.warm)
    wsteps = [[Transfer(st, hpos[i], wpos[i], orders[i][st]) for i in range(W)] for st in range(b)]
    # the warm pipeline, planned on its own (group ids 0..W-1, as the
    # reference's pipeline functions index the k-way orders by group id)
    local = [SubGroup(i, (hpos[i], wpos[i]), tuple(orders[i])) for i in range(W)]
    wsched = MulticastSchedule(tuple(local), wsteps, max_send_degree=1, enforce_step_bound=False, label="warm")
    wordered = completion_ordered_groups(local, wsched)
    for pn in generate_pipelines(wordered):
        ep = assign_blocks_to_stages(pn, [g.transfer_order for g in wordered], b, wsched, len(pipes))
        pipes.append(ep)
    wgroups = [SubGroup(len(groups) + i, g.member_nodes, g.transfer_order) for i, g in enumerate(local)]
    for st, row in enumerate(wsteps):
        while len(steps) <= st:
            steps.append([])
        steps[st] = steps[st] + row
    deg = base.schedule.max_send_degree if base is not None else 1
    sched = MulticastSchedule(tuple(groups + wgroups), steps, max_send_degree=deg, enforce_step_bound=False,
                              label="lambda+warm")
    step_s = base.step_s_model if base is not None else transfer_step_time(wsched, layout.plan,
                                                                             cluster or b200_box(node_count=len(refs)))
    tp.exec_plan = ScaleOutPlan(cfg, layout, list(range(len(refs))), sources, groups + wgroups, sched,
                                ordered + wgroups, pipes, step_s, True, "lambda+warm", tuple(hosts))
    tp.exec_ref_nodes = refs
    return tp


def node_ops(plan: ScaleOutPlan, node: int, direction: int = 1) -> list:
    """Transfers executed by ``node`` — the host-side mirror of the engine's
    op assignment (lp_multicast.cu compile()): the receiver executes when
    direction == 1 (pull) or the sender is the HOST node, else the sender.
    Rows (step, sender, receiver, block, wait) in (step, sender, receiver)
    order; ``wait`` = the sender is not a source (it must first receive)."""
    hosts = set(plan.host_nodes)
    srcs = set(plan.sources)
    rows = sorted((t.step, t.sender, t.receiver, t.block_id) for row in plan.schedule.steps for t in row)
    out = []
    for step, snd, rcv, blk in rows:
        pulled = direction == 1 or snd in hosts
        if (pulled and rcv == node) or (not pulled and snd == node):
            out.append((step, snd, rcv, blk, int(snd not in srcs)))
    return out


KERNEL_TILE = 2 << 20    # in-kernel executor (a tile is one CTA's unit): measured best on 8B / 13B images
CE_TILE = 256 << 20
HYBRID_TILE = 64 << 20   # DMA tile of the PCIe hop = relay granule of the kernel
SPLIT_CE_TILE = 64 << 20  # copy-engine blocks of the split executor


def split_tiles(n_blocks: int, kernel_tile: int, ce_split: int = 2) -> list:
    """Per-block tile sizes of the split executor (lp_mc_create_tiled): the
    copy-engine blocks (b % ce_split == 0, the engine's option) in
    SPLIT_CE_TILE tiles (few stream ops), the in-kernel ones in kernel_tile
    (a tile is one CTA's unit)."""
    return [SPLIT_CE_TILE if b % ce_split == 0 else kernel_tile for b in range(n_blocks)]


def choose_strategy(host_source: bool, n_gpus: int) -> str:
    """Full-replica scale-out from the box's shared host copy with >= 2 GPUs:
    sharded PCIe loads + NVLink exchange (2.0x the binomial tree's host
    egress at 4 GPUs); otherwise the reference's λPipe schedule.  Serving
    (execute-while-load) always plans λPipe: its pipelines need the
    binomial arrival order."""
    return "sharded_host" if host_source and n_gpus >= 2 else "lambda"


def choose_executor(plan: ScaleOutPlan, tile_bytes: int = KERNEL_TILE):
    """Measured policy (profiles/mc_sweeps_r01.md, p2p_micro_r01.txt):
    host-sourced schedules run hybrid — the PCIe hop as pinned DMA on the
    copy engines (55.3 GB/s vs 51.4 GB/s for SM-issued PCIe reads), NVLink
    relays in the kernel; GPU-sourced schedules with relays (>= 3 nodes) run
    on the copy engines with 256 MiB tiles — DMA keeps ~778 GB/s per
    direction while a relay sends and receives, SM-issued NVLink traffic
    drops to ~673 GB/s — everything else (1 -> 1) runs in-kernel."""
    if plan.host_source:
        return "hybrid", HYBRID_TILE
    if len(plan.nodes) >= 3 and plan.block_count <= 32:
        return "ce", CE_TILE
    # long schedules (e.g. Llama-3-70B, b = 80: 81 serial ops per relay) lose
    # more to tile-granular waits on the copy engines than they gain: measured
    # 295 ms (CE) vs 218-248 ms (kernel) for GPU0 -> 3 peers
    return "kernel", tile_bytes


@dataclass
class ScaleOutResult:
    epoch: int
    kernel_ms: float                 # device time of this rank's multicast kernel
    wall_ms: float                   # host wall time launch -> complete
    arrivals_ms: dict = field(default_factory=dict)   # node -> [per-block arrival, ms from start]
    checksums: dict = field(default_factory=dict)     # node -> per-block checksums (verify=True)
    launches: int = 0                                  # our kernels launched by this run (this process)


class ScaleOut:
    """Owns a cluster + compiled schedule; ``run()`` performs one scale-out."""

    def __init__(self, plan: ScaleOutPlan, distributed: bool = False, tile_bytes: int = E.DEFAULT_TILE,
                 push_ctas: int = 0, pull_ctas: int = 64, seed: int = 0, device: int = 0, direction: int = 1,
                 copy_mode: int = 1, chunk_bytes: int = 16384, executor: str = "kernel", ce_streams: int = 1,
                 verify: bool = False, verify_ctas: int | None = None, window: int = 3):
        self.plan = plan
        self.distributed = distributed
        self.push_ctas, self.pull_ctas = push_ctas, pull_ctas
        if executor == "auto":
            executor, tile_bytes = choose_executor(plan, tile_bytes)
        lay = plan.layout
        if executor == "split" and not isinstance(tile_bytes, (list, tuple)):
            tile_bytes = split_tiles(len(lay.block_offsets), tile_bytes)
        if distributed:
            self.cluster = E.Cluster.distributed(lay.block_offsets, lay.block_lengths, lay.weights_bytes,
                                                 host_node=plan.host_source, tile_bytes=tile_bytes)
        else:
            n_gpu = len(plan.nodes) - (1 if plan.host_source else 0)
            self.cluster = E.Cluster.local(n_gpu, lay.block_offsets, lay.block_lengths, lay.weights_bytes,
                                           device=device, host_node=plan.host_source, tile_bytes=tile_bytes)
        if executor not in ("kernel", "ce", "hybrid", "split"):
            raise ValueError("executor is 'kernel' (in-kernel NVLink/PCIe copies), 'ce' (copy engines), "
                             "'hybrid' (host DMA + in-kernel relay), 'split' (hybrid + every other block's "
                             "GPU->GPU transfers on the copy engines) or 'auto'")
        self.split = executor == "split"
        if self.split:
            executor = "hybrid"
        self.executor = executor
        self.ce_streams = ce_streams
        self.cluster.engine.configure(direction, copy_mode, copy_mode, chunk_bytes, window)
        self.cluster.engine.set_option("host_dma", int(executor == "hybrid"))
        self.cluster.engine.set_option("ce_split", 2 if self.split else 0)
        self.kernel_launches = 0      # multicast kernels of the last run (this process)
        # verify-as-it-lands (lp_mc_verify): receivers checksum every block
        # once its counter completes (one checksum launch per block, grid
        # capped at verify_ctas); run() returns the sums (a d2h of 8 B per block)
        self.verify = verify
        self.verify_ctas = verify_ctas or (96 if executor == "ce" else 48)
        self._vbuf = {}
        self.seed = seed
        self.device = device
        self._loaded = False

    def load_sources(self):
        """Materialise the model on every source (GPU fill / host copy)."""
        import torch.distributed as dist
        for s in self.plan.sources:
            nb = self.cluster.node(s)
            mine = (nb.kind == E.LP_NODE_HOST and self.cluster.rank == 0) or \
                (nb.kind == E.LP_NODE_GPU and s in self.cluster.exec_nodes)
            if mine:
                E.load_source_image(self.cluster, s, self.plan.layout, self.seed, self.device)
        if self.distributed:
            dist.barrier()
        self.cluster.set_schedule(self.plan.schedule, self.plan.sources)
        self._loaded = True

    def launch(self, stream: int = 0) -> int:
        if not self._loaded:
            self.load_sources()
        return self.cluster.launch(self.push_ctas, self.pull_ctas, stream)

    def run(self, stream=None) -> ScaleOutResult:
        """One scale-out epoch.  The producers (kernel / copy engines) are
        enqueued first; verify-as-it-lands goes after them on side streams,
        each parked in stream-ordered waits on its node's block counters (no
        SM spins on work queued elsewhere, so the run also completes under
        ncu's serialisation or a sanitizer)."""
        import torch
        s = stream or torch.cuda.current_stream()
        sp = E.N.stream_ptr(s)
        t0 = time.perf_counter()
        vnodes = [n for n in self.cluster.exec_nodes if n not in self.plan.sources] if self.verify else []
        for node in vnodes:     # allocated before ev0: nothing of this run may follow on s and touch them
            if node not in self._vbuf:
                self._vbuf[node] = (torch.empty(self.plan.block_count, dtype=torch.int64, device=s.device),
                                    torch.empty(self.plan.block_count, dtype=torch.int64, pin_memory=True),
                                    torch.cuda.Stream(device=s.device))
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(s)
        if not self._loaded:
            self.load_sources()
        epoch_next = self.cluster.epoch + 1
        if self.executor == "ce":
            epoch = self.cluster.launch_ce(self.ce_streams, after=ev0)
            self.cluster.join_ce(s)
            self.kernel_launches = 0
        elif self.executor == "hybrid":
            epoch, self.kernel_launches = self.cluster.launch_hybrid(s, self.push_ctas, self.pull_ctas)
        else:
            epoch = self.launch(sp)
            self.kernel_launches = 1 + int(self.pull_ctas > 0)    # count reset + multicast kernel
        assert epoch == epoch_next
        vstreams = []
        for node in vnodes:
            vs = self._vbuf[node][2]
            vs.wait_event(ev0)
            self.cluster.engine.verify(node, epoch, self._vbuf[node][0].data_ptr(), vs.cuda_stream,
                                       self.verify_ctas)
            vstreams.append((node, vs))
        for node, vs in vstreams:
            ev = torch.cuda.Event()
            ev.record(vs)
            s.wait_event(ev)
        self._readback(vstreams, s)
        ev1.record(s)
        if self.executor == "ce":
            s.synchronize()
        else:
            self.cluster.wait(sp)
        sums = {}
        for node, _ in vstreams:
            sums[node] = [int(x) & 0xFFFFFFFFFFFFFFFF for x in self._vbuf[node][1].tolist()]
        verify_launches = sum(len(self.cluster.engine.received_blocks(n)) for n, _ in vstreams)
        wall = (time.perf_counter() - t0) * 1e3
        return ScaleOutResult(epoch, ev0.elapsed_time(ev1), wall, checksums=sums,
                              launches=self.kernel_launches + verify_launches)

    def poison(self, value: int = 0xA5, stream=None) -> None:
        """Overwrite every receiver image this process executes with a byte
        pattern (outside any timed region), so the next run's checksums prove
        that run delivered every byte rather than an earlier one."""
        import torch
        s = stream or torch.cuda.current_stream()
        for node in self.cluster.exec_nodes:
            if node in self.plan.sources:
                continue
            nb = self.cluster.node(node)
            with E.on_device(nb.device):
                E.N.call("lp_memset", E.C.c_void_p(nb.image), int(value) & 0xFF, self.plan.layout.weights_bytes,
                         E.C.c_void_p(s.cuda_stream))
        s.synchronize()

    def _readback(self, vstreams, s):
        import torch
        with torch.cuda.stream(s):
            for node, _ in vstreams:
                self._vbuf[node][1].copy_(self._vbuf[node][0], non_blocking=True)

    def arrivals(self, node: int) -> list:
        return self.cluster.engine.arrivals_ns(node)

    def checksums(self, node: int) -> list:
        nb = self.cluster.node(node)
        return E.block_checksums(nb.image, self.plan.layout.block_offsets, self.plan.layout.block_lengths)

    def close(self):
        self.cluster.close()


class TieredScaleOut:
    """Executes a :class:`TieredPlan` on this process's GPUs (one process,
    ``engine.Cluster.devices``) through its execution plan
    (:func:`warm_pipeline_plan`): the λPipe multicast to the cold nodes plus
    the warm nodes' k-way-ordered loads from the pinned host copy, all rows on
    one engine (position i on device ``node_devices[exec_ref_nodes[i]]``,
    HOST positions in pinned memory); hot nodes keep their copy.  The
    multicast runs in-kernel in the pull direction (receivers read peers over
    NVLink and the host over PCIe).  ``plan`` is what ``serving.Server``
    takes: its pipelines include the warm pipeline."""

    def __init__(self, tp: TieredPlan, node_devices: dict | None = None, seed: int = 0,
                 tile_bytes: int = KERNEL_TILE, config=None, block_count: int | None = None):
        self.tp = tp
        self.seed = seed
        self.dev_of = dict(node_devices or {})
        self.cluster = None
        if tp.exec_plan is None:
            cfg = config or (tp.plan.config if tp.plan is not None else None)
            warm_pipeline_plan(tp, cfg, block_count or (tp.plan.block_count if tp.plan is not None else 16))
        plan = tp.exec_plan
        self.layout = plan.layout if plan is not None else None
        if plan is not None:
            lay = plan.layout
            devs = [-1 if i in plan.host_nodes else self.dev_of.get(n, n) for i, n in enumerate(tp.exec_ref_nodes)]
            self.cluster = E.Cluster.devices(devs, lay.block_offsets, lay.block_lengths, lay.weights_bytes,
                                             tile_bytes=tile_bytes)

    @property
    def plan(self):
        return self.tp.exec_plan

    def _any_device(self) -> int:
        devs = [nb.device for nb in self.cluster.nodes if nb.device >= 0] if self.cluster else [0]
        return min(devs)

    def load_sources(self):
        if self.cluster is None:
            return
        plan = self.tp.exec_plan
        filled_host = False
        for i in plan.sources:
            nb = self.cluster.node(i)
            if nb.kind == E.LP_NODE_HOST:
                if filled_host:
                    continue
                filled_host = True
            E.load_source_image(self.cluster, i, plan.layout, self.seed, device=self._any_device())
        self.cluster.set_schedule_all(plan.schedule, plan.sources)

    def launch(self, streams: dict, pull_ctas: int = 32) -> int | None:
        """Start the multicast + warm loads (one kernel per device on
        ``streams[device]``); returns the epoch."""
        if self.cluster is None:
            return None
        return self.cluster.launch_devices(streams, 0, pull_ctas)

    def wait(self, streams: dict):
        if self.cluster is not None:
            self.cluster.wait_devices()
        for st in streams.values():
            st.synchronize()

    def checksums(self) -> dict:
        """reference node id -> per-block checksums of every demand node's copy."""
        out = {}
        if self.cluster is None:
            return out
        plan = self.tp.exec_plan
        lay = plan.layout
        for i, n in enumerate(self.tp.exec_ref_nodes):
            if i in plan.sources:
                continue
            nb = self.cluster.node(i)
            with E.on_device(nb.device):
                out[n] = E.block_checksums(nb.image, lay.block_offsets, lay.block_lengths)
        return out

    def close(self):
        if self.cluster is not None:
            self.cluster.close()
            self.cluster = None


def scale_out(model, demand: list, tiers: TierMap, k: int = 1, block_count: int = 16, host_id: int | None = None,
              node_devices: dict | None = None, seed: int = 0, pull_ctas: int = 32):
    """Drop-in entry for the simulator's scale-out of
    ``demand`` nodes (simengine.py:442-467 then :564-602) on real GPUs:
    ``startup_plan`` over ``tiers`` (GPU copies first, then the box's host
    copy ``host_id``), hot nodes kept, warm nodes loaded from host memory in
    k-way order (with their pipeline, :func:`warm_pipeline_plan`), the λPipe
    multicast to the cold ones — executed and waited for.  Returns
    ``(TieredScaleOut, epoch)``; the caller closes it."""
    import torch
    cfg = CONFIGS[model] if isinstance(model, str) else model
    tp = warm_pipeline_plan(plan_from_tiers(cfg, demand, tiers, k, block_count, host_id), cfg, block_count)
    so = TieredScaleOut(tp, node_devices, seed)
    so.load_sources()
    if so.cluster is None:
        return so, None
    devs = sorted({nb.device for nb in so.cluster.nodes if nb.device >= 0})
    streams = {d: torch.cuda.Stream(device=d) for d in devs}
    epoch = so.launch(streams, pull_ctas)
    so.wait(streams)
    return so, epoch
