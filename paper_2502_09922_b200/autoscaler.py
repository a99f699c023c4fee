"""Reactive autoscaling over real GPUs: the reference's scale-out trigger and
scale-in loop (simengine.py:397-467 ``_eval_scaling``/``_scale_out``,
:418-438 ``_on_scale_in_check``) driving repeated λPipe scale-outs.

One process drives the box's GPUs; each GPU is a reference *node* with one
persistent packed image + multicast signal area.  A node is

* **hot**   — holds the model and serves as a local replica,
* **loading** — the target of an in-flight scale-out (serves through the
  op's execution pipelines while blocks land, then switches to local),
* **idle**  — no model (released after ``keep_alive_s`` without work).

Every ``eval_interval_s`` the reference rule ``autoscale(policy, queue,
active + pending)`` (cluster.py, simengine.py:78-92) decides how many
replicas to add; that many idle GPUs are claimed and a scale-out op is
planned exactly as ``_scale_out`` / ``_launch_lambda_scale`` do
(simengine.py:442-467, :564-590): ``startup_plan`` over the box's tiers — hot
GPUs hold a GPU copy, the optional pinned host copy (``host_copy``, node id
``len(devices)``) a MEMORY copy, released GPUs lose theirs (the eviction of
simengine.py:404-416) — picks GPU sources first, then the host copy, up to
``k``; ``scaleout.plan_from_tiers`` builds the λPipe plan, executed by the
multicast engine (copy engines: no SM time is taken from serving; host rows
are PCIe DMA), with pipelines activating on landed blocks and a mode switch
at completion (``serving.Server`` machinery).
Events use the reference's kinds so ``workload.aggregate`` yields TTFT
percentiles, the tokens/s timeline and GPU-seconds.
"""

from __future__ import annotations

import math
import time
from collections import deque

from . import engine as E
from .cluster import AutoscalePolicy, autoscale
from .image import CONFIGS, build_layout, model_spec
from .pipeline import plan_mode_switch
from .errors import UnsatisfiableScalingError
from .modelmgr import TierMap
from .scaleout import CE_TILE, plan_from_tiers
from .serving import Request, Server, Stage
from .workload import SimEvent


class _Nodes:
    """Global node table (node id = device index)."""

    def __init__(self, buffers):
        self.buffers = buffers

    def node(self, i):
        return self.buffers[i]

    def node_device(self, i):
        return self.buffers[i].device


class _ScaleOp:
    def __init__(self, op_id, sources, targets, plan, cluster, stream_of, pipelines):
        self.op_id = op_id
        self.sources = sources          # global node ids
        self.targets = targets
        self.plan = plan                # op-local numbering (sources first)
        self.cluster = cluster
        self.stream_of = stream_of
        self.pipelines = pipelines      # pipeline Units (global node ids)
        self.epoch = None
        self.done = False
        self.t_start = None


class AutoscaleServer(Server):
    """Serves a trace on ``devices`` with reactive λPipe scale-out/scale-in."""

    def __init__(self, model, devices: list, block_count: int = 16, k: int = 1, hot: tuple = (0,),
                 policy: AutoscalePolicy | None = None, local_slots: int = 16, max_len: int = 192,
                 use_graphs: bool = True, seed: int = 20250815, max_replicas: int | None = None,
                 host_copy: bool = False):
        import torch
        self.torch = torch
        self.cfg = CONFIGS[model] if isinstance(model, str) else model
        self.lay = build_layout(self.cfg, block_count)
        self.local_slots, self.max_len, self.use_graphs = local_slots, max_len, use_graphs
        self.pipeline_batch = 1                                    # the reference's pipeline capacity
        self.pipeline_prefill_tokens = self.prefill_budget(self.lay)
        self.prefill_ms_per_token = model_spec(self.cfg).prefill_ms_per_token
        self.policy = policy or AutoscalePolicy()
        self.k = k
        self.max_replicas = max_replicas or len(devices)
        self.events, self.profile, self.units = [], [], {}
        self._next_uid = 0
        self.switched = True
        lay = self.lay
        for a in devices:                 # stream waits / copies on peer memory need peer access
            for b in devices:
                if a != b:
                    E.N.call("lp_enable_peer", a, b)
        # one persistent image + signal area per GPU
        probe = E.MulticastEngine(2, lay.block_offsets, lay.block_lengths, CE_TILE)
        sig_bytes = probe.signal_bytes
        probe.close()
        self.buffers = []
        for d in devices:
            img = E.dev_malloc(d, lay.weights_bytes)
            sig = E.dev_malloc(d, sig_bytes)
            self.buffers.append(E.NodeBuffer(d, E.LP_NODE_GPU, d, img, sig, [("dev", img), ("dev", sig)]))
        self.cluster = _Nodes(self.buffers)
        for n in hot:
            E.load_source_image(self.cluster, n, lay, seed)
        self.host_id = len(devices)          # reference node id of the box's pinned host copy
        self.host = None
        if host_copy:
            with E.on_device(devices[0]):
                self.host = E.HostImage(lay.weights_bytes)
            scratch = E.dev_malloc(devices[0], lay.weights_bytes)
            with E.on_device(devices[0]):
                E.fill_image(scratch, lay, seed)
                E.N.call("lp_memcpy", E.C.c_void_p(self.host.host_ptr), E.C.c_void_p(scratch), lay.weights_bytes,
                         None)
            E.N.call("lp_sync_device", devices[0])
            E.dev_free(devices[0], scratch)
        for d in devices:
            torch.cuda.synchronize(d)
        self.state = {n: ("hot" if n in hot else "idle") for n in range(len(devices))}
        self.last_busy = {n: 0.0 for n in range(len(devices))}
        # one local replica (executor + captured graphs) per GPU, reused across scale-outs
        self.replica = {n: self._local_unit(n, active=(self.state[n] == "hot")) for n in range(len(devices))}
        for n, u in self.replica.items():
            u.cold = n not in hot
        self.streams = {d: torch.cuda.Stream(device=d) for d in devices}
        self.ops = []
        self._op_id = 0
        self.decisions = []     # (t, queue, active, pending, scale_out, room) per evaluation

    # -- scale-out --------------------------------------------------------------
    def tiers(self) -> TierMap:
        """The box's residency in the reference's terms: serving (hot) GPUs hold
        a GPU copy, the pinned host copy (node ``host_id``) a MEMORY copy;
        loading and released GPUs hold nothing usable as a source."""
        tm = TierMap()
        blocks = set(range(self.lay.plan.block_count))
        for n, st in self.state.items():
            tm.ensure(n, self.cfg.name).gpu_blocks = set(blocks) if st == "hot" else set()
        if self.host is not None:
            tm.ensure(self.host_id, self.cfg.name).mem_blocks = set(blocks)
        return tm

    def _scale_out(self, now, want):
        idle = [n for n, st in self.state.items() if st == "idle"]
        targets = idle[:want]
        if not targets:
            return
        try:
            tp = plan_from_tiers(self.cfg, targets, self.tiers(), k=self.k, block_count=self.lay.plan.block_count,
                                 host_id=self.host_id)
        except UnsatisfiableScalingError:     # no copy of the model anywhere: nothing to scale from
            return
        if tp.plan is None:
            return
        sources, targets = tp.sources, tp.cold
        g = tp.ref_nodes                                               # op-local -> global
        sched, srcs, eps = tp.plan.schedule, tp.plan.sources, tp.plan.pipelines
        host_nb = (E.NodeBuffer(self.host_id, E.LP_NODE_HOST, -1, self.host.device_ptr)
                   if self.host is not None else None)
        bufs = [host_nb if i in tp.plan.host_nodes else self.buffers[x] for i, x in enumerate(g)]
        for x in targets:
            with E.on_device(self.buffers[x].device):
                E.N.call("lp_memset", E.C.c_void_p(self.buffers[x].signals), 0, self._sig_bytes(), None)
            self.torch.cuda.synchronize(self.buffers[x].device)
        cl = E.Cluster.over_buffers(bufs, self.lay.block_offsets, self.lay.block_lengths, CE_TILE)
        cl.set_schedule_all(sched, srcs)
        for eng in cl.per_device.values():
            eng.configure(1, 0, 0, 16384, 3)
        units = []
        for ep in eps:
            stages, covered = [], -1
            for st in ep.stages:
                if st.block_lo > st.block_hi:
                    continue
                lo = max(self.lay.plan.blocks[st.block_lo].layer_lo, covered + 1)
                hi = self.lay.plan.blocks[st.block_hi].layer_hi
                covered = max(covered, hi)
                node = g[st.node]
                stages.append(Stage(node, self.buffers[node].device, st.block_lo, st.block_hi, lo, hi,
                                    st.block_lo == 0))
            units.append(self._add_unit("pipeline", stages, max(1, len(ep.stages)), True, ep))
        op = _ScaleOp(self._op_id, sources, targets, None, cl, None, units)
        op.local_of = {i: x for i, x in enumerate(g)}
        self._op_id += 1
        for x in targets:
            self.state[x] = "loading"
        op.t_start = now
        streams = {d: self.streams[d] for d in cl.per_device}
        op.epoch = cl.launch_devices_ce(streams)
        self.ops.append(op)
        self.log(now, "scale_out", model=self.cfg.name, nodes=targets, sources=sources, strategy="lambda_scale",
                 classes={n: tp.startup.classes[n] for n in targets})
        self._sample_alloc(now)

    def _sig_bytes(self):
        if not hasattr(self, "_sb"):
            probe = E.MulticastEngine(2, self.lay.block_offsets, self.lay.block_lengths, CE_TILE)
            self._sb = probe.signal_bytes
            probe.close()
        return self._sb

    def _warm_units(self, units):
        for u in units:
            scratch = u.stages[0].executor.scratch_seq
            self._forward(u, [0] * 8, list(range(8)), [scratch] * 8, [7])

    def _poll_ops(self, now):
        for op in self.ops:
            if op.done:
                continue
            done = op.cluster.complete_nodes(op.epoch)          # op-local ids
            for u in op.pipelines:
                if not u.active and not u.retired:
                    inv = {v: k for k, v in op.local_of.items()}
                    if all(all(done[inv[st.node]][b] for b in range(st.block_lo, st.block_hi + 1)) for st in u.stages):
                        u.active = True
            if all(all(done[i]) for i in done if op.local_of[i] in op.targets):
                self._switch(op, now)

    def _switch(self, op, now):
        for u in op.pipelines:
            u.retired = True
            inflight = [u.busy[s] for s in sorted(u.busy)]
            plan = plan_mode_switch(u.pipeline, [(r.rid, len(r.out)) for r in inflight], self.prefill_ms_per_token)
            by_id = {r.rid: r for r in inflight}
            for row in plan.assignments:
                tgt = self.replica[op.local_of[row.node]]
                r = by_id[row.request_id]
                s = tgt.free_slot()
                r.unit, r.slot, r.kv_len, r.needs_prefill = tgt.uid, s, 0, True
                tgt.busy[s] = r
        for u in op.pipelines:                      # free the pipeline stages' KV caches
            for st in u.stages:
                st.executor = None
        for x in op.targets:
            self.state[x] = "hot"
            self.replica[x].active = True
            self.last_busy[x] = now
        self.log(now, "mode_switch", model=self.cfg.name, nodes=sorted(op.targets), mode="local")
        op.done = True
        for st in self.streams.values():
            st.synchronize()
        op.cluster.close()

    # -- scale-in -------------------------------------------------------------
    def _scale_in(self, now, queue_empty):
        hot = [n for n, st in self.state.items() if st == "hot"]
        for n in hot:
            u = self.replica[n]
            if u.busy:
                self.last_busy[n] = now
                continue
            busy_src = any(not op.done and n in op.sources for op in self.ops)
            if (queue_empty and now - self.last_busy[n] >= self.policy.keep_alive_s and not busy_src
                    and sum(1 for s in self.state.values() if s == "hot") > max(1, self.policy.min_replicas)):
                self.state[n] = "idle"
                u.active = False
                self.log(now, "scale_in", node=n, model=self.cfg.name)
                self._sample_alloc(now)

    def _sample_alloc(self, now):
        self.log(now, "allocation", allocated_gpus=sum(1 for s in self.state.values() if s != "idle"))

    # -- main loop ---------------------------------------------------------------
    def run(self, trace, prompts: dict, timeout_s: float = 600.0):
        torch = self.torch
        if self.use_graphs:
            for u in self.replica.values():
                if u.graph is None:
                    from .llama import DecodeGraph
                    u.graph = DecodeGraph(u.stages[0].executor, u.slots)
                    u.graph.capture()
                for cap in self.PREFILL_BUCKETS:
                    if cap <= self.max_len * u.slots:
                        self._prefill_graph(u, cap)
        for d in self.streams:
            torch.cuda.synchronize(d)
        self.t0 = time.perf_counter()
        self._sample_alloc(0.0)
        pending = deque(sorted(trace, key=lambda r: (r.arrival_s, r.request_id)))
        queue, live = deque(), {}
        next_eval = None
        while True:
            now = time.perf_counter() - self.t0
            if now > timeout_s:
                raise TimeoutError("autoscaling serve loop exceeded its timeout")
            while pending and pending[0].arrival_s <= now:
                rec = pending.popleft()
                r = Request(rec, list(prompts[rec.request_id]))
                live[rec.request_id] = r
                queue.append(r)
                self.log(rec.arrival_s, "request_arrival", request=rec.request_id, model=rec.model_id)
                if next_eval is None:
                    next_eval = now + self.policy.eval_interval_s
            if next_eval is not None and now >= next_eval:
                active = sum(1 for s in self.state.values() if s == "hot")
                pending_r = sum(1 for s in self.state.values() if s == "loading")
                dec = autoscale(self.policy, len(queue), active + pending_r)
                room = self.max_replicas - active - pending_r
                self.decisions.append((now, len(queue), active, pending_r, dec.scale_out, room))
                if dec.scale_out > 0 and room > 0:
                    self._scale_out(now, min(dec.scale_out, room))
                next_eval = now + self.policy.eval_interval_s if queue else None
            self._poll_ops(now)
            self._admit(queue)
            work = []
            for u in sorted(self.units.values(), key=lambda x: x.uid):
                if u.active and not u.retired and u.busy:
                    for w in self._step_unit(u) or []:
                        work.append((u, w))
            if not work:
                self._scale_in(now, not queue)
                if not pending and not queue and all(r.done for r in live.values()) and all(o.done for o in self.ops):
                    break
                time.sleep(0.0005)
                continue
            for d in {st.device for u, _ in work for st in u.stages}:
                # the compute stream only: a device-wide sync would also wait for the
                # multicast still landing blocks on its own stream
                torch.cuda.current_stream(d).synchronize()
            now = time.perf_counter() - self.t0
            for u, (reqs, tok) in work:
                for r, t in zip(reqs, tok.cpu().tolist()):
                    if r.needs_prefill:
                        r.kv_len = len(r.prompt) + len(r.out)
                        r.needs_prefill = False
                    else:
                        r.kv_len += 1
                    r.out.append(int(t))
                    if r.first_token_s is None:
                        r.first_token_s = now
                    self.log(now, "token_emitted", request=r.rid, node=u.emit_node, cold_capacity=u.cold)
                    if r.done:
                        r.done_s = now
                        del u.busy[r.slot]
                        self.log(now, "request_done", request=r.rid, node=u.emit_node)
                for st in u.stages:
                    self.last_busy[st.node] = now
        self.requests = live
        return self.events

    def close(self):
        if self.host is not None:
            self.host.close()
            self.host = None
        for nb in self.buffers:
            for kind, ptr in nb.owned:
                E.dev_free(nb.device, ptr)
            nb.owned = []
