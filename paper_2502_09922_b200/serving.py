"""Execute-while-load serving on real GPUs — the reference's serving units,
activation and mode switch (simengine.py:320-389, 646-712, 736-741) with
real tokens instead of modelled periods.

While the λPipe multicast runs (``engine.Cluster.devices``, one kernel per
GPU), receivers that hold only their pipeline stage's blocks already serve:

* every :class:`~.pipeline.ExecutionPipeline` of the plan becomes a
  pipeline unit whose stages run their resident layers (``llama.
  LlamaExecutor``); the hidden state moves stage to stage over NVLink
  (``lp_handoff``) and returns to the vocab stage (block 0: embedding, final
  norm, LM head) for the next token.  A unit activates when every block its
  stages need has *landed* (the engine's per-block tile counters) — the
  measured counterpart of ``activation_step`` (pipeline.py:175-185);
* capacity = stage count (pipeline.py:43-46; × ``pipeline_batch`` requests
  per slot when local replicas batch too); requests are admitted FIFO into
  free slots of active units in unit order (``_admit``, simengine.py:356-368)
  and batched per iteration (prefill and decode tokens in one ragged batch);
* when every receiver holds the whole model the pipelines retire and
  ``plan_mode_switch`` (pipeline.py:252-270) spreads their in-flight requests
  round-robin over the pipeline's nodes, whose local units rebuild the KV
  cache by prefilling prompt + generated tokens (the reference's recompute
  cost), then continue decoding.

Events follow the reference's ``SimEvent`` kinds/payloads (workload.py:28-32)
with wall-clock times from the start of the scale-out, so
``workload.aggregate`` yields TTFT percentiles and the 100 ms tokens/s
timeline unchanged.
"""

from __future__ import annotations

import os
import time
from collections import deque
from dataclasses import dataclass, field

from . import _native as N
from .pipeline import plan_mode_switch
from .workload import SimEvent, TraceRecord


@dataclass
class Request:
    rec: TraceRecord
    prompt: list
    out: list = field(default_factory=list)
    unit: int | None = None
    slot: int = -1
    kv_len: int = 0
    needs_prefill: bool = True
    first_token_s: float | None = None
    done_s: float | None = None

    @property
    def rid(self) -> str:
        return self.rec.request_id

    @property
    def done(self) -> bool:
        return len(self.out) >= self.rec.output_tokens


@dataclass
class Stage:
    node: int
    device: int
    block_lo: int
    block_hi: int
    layer_lo: int
    layer_hi: int
    vocab: bool
    executor: object = None


@dataclass
class Unit:
    uid: int
    kind: str                     # pipeline | local
    stages: list
    slots: int
    cold: bool
    pipeline: object = None
    active: bool = False
    retired: bool = False
    busy: dict = field(default_factory=dict)   # slot -> Request
    graph: object = None                        # DecodeGraph (local units)
    prefill: dict = field(default_factory=dict)  # token bucket -> PrefillGraph

    @property
    def nodes(self) -> tuple:
        return tuple(st.node for st in self.stages)

    @property
    def emit_node(self) -> int:
        return self.stages[-1].node

    def free_slot(self) -> int:
        for s in range(self.slots):
            if s not in self.busy:
                return s
        return -1


class Server:
    """Serves a request trace while ``plan`` is being multicast."""

    PREFILL_PASS_FLOP = 8.2e12     # pipeline prefill budget per pass (see __init__)

    @classmethod
    def prefill_budget(cls, layout, tokens=None) -> int:
        """Prompt tokens one pipeline pass prefills: ``tokens``, else
        PREFILL_PASS_FLOP of prompt (2 FLOP per parameter per token)."""
        if tokens is None:
            tokens = cls.PREFILL_PASS_FLOP / (2.0 * layout.weights_bytes / 2)
        return max(1, int(tokens))

    def __init__(self, plan, cluster, local_slots: int = 8, max_len: int = 512, switch_hold_tokens: int = 0,
                 prefill_ms_per_token: float = 0.5, use_graphs: bool = True, pipeline_batch: int = 1,
                 pipeline_prefill_tokens: int | None = None):
        """``pipeline_batch``: requests per pipeline slot.  The reference's
        capacity is one request per stage (pipeline.py:43-46) — with its
        one-request local units (``batch_slots = 1``, simengine.py:236).
        Local replicas here batch ``local_slots`` requests; passing
        ``pipeline_batch = local_slots`` scales the pipelines the same way
        (capacity = stages x pipeline_batch), keeping the reference's ratio of
        pipeline to local capacity.

        ``pipeline_prefill_tokens``: prompt tokens a pipeline pass prefills
        (at least one request; the rest keep waiting in their slots, decodes
        always run).  Default: ~8 TFLOP of prompt per pass (PREFILL_PASS_FLOP),
        512 tokens for Llama-3-8B and one request for 70B.  Without a budget
        a burst admitted into a wide pipeline is one long prefill that pushes
        every first token past the first full replica."""
        import torch
        self.plan = plan
        self.cluster = cluster
        self.lay = plan.layout
        self.cfg = plan.config
        self.local_slots = local_slots
        self.max_len = max_len
        self.switch_hold_tokens = switch_hold_tokens
        self.use_graphs = use_graphs
        self.prefill_ms_per_token = prefill_ms_per_token
        self.pipeline_batch = max(1, int(pipeline_batch))
        self.pipeline_prefill_tokens = self.prefill_budget(plan.layout, pipeline_prefill_tokens)
        self.events = []
        self.profile = []          # per iteration: (start, enqueue s, device s, tokens, unit batches)
        self.profile_detail = [] if os.environ.get("LP_SERVE_PROFILE") else None
        self.units = {}
        self._next_uid = 0
        self.switched = False
        self.t0 = None
        self.torch = torch
        self.receivers = [n for n in plan.receivers if cluster.node(n).kind == 0]
        self.block_complete_s = {}      # node -> time it held every block
        self.activation_s = {}          # pipeline unit -> time its stages' blocks had all landed
        # pipeline units from the plan (one per ExecutionPipeline)
        for ep in plan.pipelines:
            stages = []
            covered = -1
            for st in ep.stages:
                if st.block_lo > st.block_hi:
                    continue                  # empty stage (reference quirk): pass-through
                l_lo = self.lay.plan.blocks[st.block_lo].layer_lo
                l_hi = self.lay.plan.blocks[st.block_hi].layer_hi
                l_lo = max(l_lo, covered + 1)  # overlapped chunks (k > b) run once
                covered = max(covered, l_hi)
                stages.append(Stage(st.node, cluster.node_device(st.node), st.block_lo, st.block_hi, l_lo, l_hi,
                                    st.block_lo == 0))
            self._add_unit("pipeline", stages, max(1, len(stages)) * self.pipeline_batch, True, ep)
        # post-switch local replicas, built (and their decode graphs captured)
        # before the scale-out starts; activated at mode switch
        self.local_units = {n: self._local_unit(n, active=False) for n in self.receivers}

    # -- units -------------------------------------------------------------------
    def _add_unit(self, kind, stages, slots, cold, pipeline=None):
        from .llama import LlamaExecutor
        for st in stages:
            st.executor = LlamaExecutor(self.lay, self.cluster.node(st.node).image, st.device,
                                        st.layer_lo, st.layer_hi, max_seqs=slots, max_len=self.max_len,
                                        vocab_ops=st.vocab)
        u = Unit(self._next_uid, kind, stages, slots, cold, pipeline)
        self.units[u.uid] = u
        self._next_uid += 1
        return u

    def _local_unit(self, node, active: bool = True):
        dev = self.cluster.node_device(node)
        st = Stage(node, dev, 0, self.lay.plan.block_count - 1, 0, self.cfg.n_layers - 1, True)
        u = self._add_unit("local", [st], self.local_slots, True)
        u.active = active
        return u

    def log(self, t, kind, **payload):
        self.events.append(SimEvent(t, kind, payload))

    # -- forward through a unit --------------------------------------------------
    def _dev_tensor(self, vals, device):
        return self.torch.as_tensor(vals, dtype=self.torch.int32, device=f"cuda:{device}")

    def _move(self, x, src_dev, dst_dev):
        """Hidden-state hand-off stage -> stage (NVLink stores, lp_handoff)."""
        torch = self.torch
        if src_dev == dst_dev:
            return x
        dst = torch.empty(x.shape, dtype=x.dtype, device=f"cuda:{dst_dev}")
        # dst comes from the destination stream's allocator pool: a block freed
        # there may still be read by queued destination kernels, so the
        # source-stream stores must wait for that stream first
        free_ev = torch.cuda.Event()
        free_ev.record(torch.cuda.current_stream(dst_dev))
        torch.cuda.current_stream(src_dev).wait_event(free_ev)
        with torch.cuda.device(src_dev):
            N.check(N.lib().lp_handoff(N.C.c_void_p(x.data_ptr()), N.C.c_void_p(dst.data_ptr()),
                                       x.numel() * x.element_size(), None, 0, None,
                                       N.C.c_void_p(torch.cuda.current_stream(src_dev).cuda_stream)),
                    "lp_handoff")
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(src_dev))
        torch.cuda.current_stream(dst_dev).wait_event(ev)
        return dst

    def _forward(self, unit, tokens, pos, seq, last_idx):
        """Run one ragged batch through the unit's stages; returns next tokens
        (int32, on the vocab device) for rows ``last_idx``."""
        torch = self.torch
        vocab = next(st for st in unit.stages if st.vocab)
        vdev = vocab.device
        with torch.cuda.device(vdev):
            x = vocab.executor.embed(self._dev_tensor(tokens, vdev))
        cur = vdev
        for st in unit.stages:
            if st.layer_lo > st.layer_hi:
                continue
            x = self._move(x, cur, st.device)
            cur = st.device
            with torch.cuda.device(cur):
                p, s = self._dev_tensor(pos, cur), self._dev_tensor(seq, cur)
                ex = st.executor
                for layer in range(st.layer_lo, st.layer_hi + 1):
                    x = ex.layer(layer, x, p, s)
        x = self._move(x, cur, vdev)
        with torch.cuda.device(vdev):
            xl = x[self._dev_tensor(last_idx, vdev).long()].contiguous()
            logits = vocab.executor.head(xl)
            tok, _ = vocab.executor.greedy(logits)
        return tok

    # -- scheduling --------------------------------------------------------------
    def _admit(self, queue):
        """FIFO admission (simengine.py:356-368).  Each request goes to the
        active unit with the most free slots, ties to the lowest unit id: with
        the reference's one slot per local unit (``batch_slots = 1``) that is
        exactly its unit-order fill; with 16-slot continuous-batching replicas
        it spreads a burst over the replicas instead of stacking every prefill
        on the first one."""
        live = [u for u in sorted(self.units.values(), key=lambda x: x.uid) if u.active and not u.retired]
        while queue and live:
            u = max(live, key=lambda x: (x.slots - len(x.busy), -x.uid))
            s = u.free_slot()
            if s < 0:
                break
            r = queue.popleft()
            r.unit, r.slot, r.kv_len, r.needs_prefill = u.uid, s, 0, True
            u.busy[s] = r

    def _pipeline_pass(self, reqs: list) -> list:
        """The requests one pipeline pass runs: every decode, and prefills in
        slot order while they fit ``pipeline_prefill_tokens`` (always at
        least one, so a long prompt still makes progress)."""
        keep, n_pf = [], 0
        for r in reqs:
            if r.needs_prefill:
                n = len(r.prompt) + len(r.out)
                if n_pf and n_pf + n > self.pipeline_prefill_tokens:
                    continue
                n_pf += n
            keep.append(r)
        return keep

    def _mode_switch(self, now):
        switched_nodes = []
        for u in sorted(self.units.values(), key=lambda x: x.uid):
            if u.kind != "pipeline" or u.retired:
                continue
            u.retired = True
            inflight = [u.busy[s] for s in sorted(u.busy)]
            plan = plan_mode_switch(u.pipeline, [(r.rid, len(r.out)) for r in inflight],
                                    self.prefill_ms_per_token)
            # every node of the plan's pipeline (an empty stage's node too:
            # plan_mode_switch deals requests over all of them)
            locals_by_node = {st.node: self.local_units[st.node] for st in u.pipeline.stages}
            for lu in locals_by_node.values():
                lu.active = True
            by_id = {r.rid: r for r in inflight}
            for row in plan.assignments:
                r = by_id[row.request_id]
                tgt = locals_by_node[row.node]
                s = tgt.free_slot()
                r.unit, r.slot, r.kv_len, r.needs_prefill = tgt.uid, s, 0, True   # KV recompute
                tgt.busy[s] = r
            switched_nodes.extend(u.nodes)
        if switched_nodes:
            self.log(now, "mode_switch", model=self.cfg.name, nodes=sorted(switched_nodes), mode="local")
        self.switched = True

    PREFILL_BUCKETS = (128, 256, 384, 512, 768, 1024, 1536, 2048)

    def _prefill_graph(self, u, n_tokens):
        """Smallest captured prefill graph that fits (captured on demand)."""
        if not self.use_graphs:
            return None
        for cap in self.PREFILL_BUCKETS:
            if n_tokens <= cap and cap <= self.max_len * u.slots:
                if cap not in u.prefill:
                    from .llama import PrefillGraph
                    u.prefill[cap] = PrefillGraph(u.stages[0].executor, cap, u.slots)
                    u.prefill[cap].capture()
                return u.prefill[cap]
        return None

    def _pipeline_graph(self, u, n_tokens):
        """Captured ring for a pipeline unit: decode width = slots, prefill
        buckets like local replicas (captured on demand, or before the clock)."""
        if not self.use_graphs:
            return None
        from .llama import PipelineGraph
        vocab = next(st for st in u.stages if st.vocab).executor
        execs = [st.executor for st in u.stages]
        caps = [u.slots] + [c for c in self.PREFILL_BUCKETS if c <= self.max_len * u.slots]
        for cap in caps:
            if n_tokens <= cap:
                if cap not in u.prefill:
                    u.prefill[cap] = PipelineGraph(execs, vocab, cap, u.slots)
                    u.prefill[cap].capture()
                return u.prefill[cap]
        return None

    def _step_unit(self, u):
        """Enqueue one iteration for unit u; returns [(requests, token tensor)].

        Local replicas decode through a captured CUDA graph (one replay per
        step); prefills and pipeline units run eagerly."""
        reqs = [u.busy[s] for s in sorted(u.busy)]
        if not reqs:
            return None
        out = []
        if u.kind == "local" and self.use_graphs:
            dec = [r for r in reqs if not r.needs_prefill]
            reqs = [r for r in reqs if r.needs_prefill]
            if dec:
                if u.graph is None:
                    from .llama import DecodeGraph
                    u.graph = DecodeGraph(u.stages[0].executor, u.slots)
                with self.torch.cuda.device(u.stages[0].device):
                    tok = u.graph.step([r.out[-1] for r in dec], [r.kv_len for r in dec], [r.slot for r in dec])
                out.append((dec, tok))
            if reqs:
                # one graph replay per iteration: requests beyond the largest
                # bucket keep needs_prefill and go in the next iteration
                # (an eager 32-layer forward would cost ~50 ms of launches)
                cap_max = max(c for c in self.PREFILL_BUCKETS if c <= self.max_len * u.slots)
                take, n_tok = [], 0
                for r in reqs:
                    n = len(r.prompt) + len(r.out)
                    if take and n_tok + n > cap_max:
                        break
                    take.append(r)
                    n_tok += n
                reqs = take
                pf = self._prefill_graph(u, n_tok)
                if pf is not None:
                    tokens, pos, seq, last = [], [], [], []
                    for r in reqs:
                        ctx = r.prompt + r.out
                        tokens += ctx
                        pos += list(range(len(ctx)))
                        seq += [r.slot] * len(ctx)
                        last.append(len(tokens) - 1)
                    t_pf = time.perf_counter()
                    with self.torch.cuda.device(u.stages[0].device):
                        out.append((reqs, pf.step(tokens, pos, seq, last)))
                    if getattr(self, "profile_detail", None) is not None:
                        self.profile_detail.append(("prefill_enqueue", u.uid, pf.cap, time.perf_counter() - t_pf))
                        self.profile_detail.append(("prefill_parts " + " ".join("%.4f" % v for v in pf.last_timing),
                                                    u.uid, pf.cap, 0.0))
                    reqs = []
            if not reqs:
                return out
        if u.kind == "pipeline":
            reqs = self._pipeline_pass(reqs)
        tokens, pos, seq, last = [], [], [], []
        for r in reqs:
            if r.needs_prefill:
                ctx = r.prompt + r.out
                tokens += ctx
                pos += list(range(len(ctx)))
                seq += [r.slot] * len(ctx)
            else:
                tokens.append(r.out[-1])
                pos.append(r.kv_len)
                seq.append(r.slot)
            last.append(len(tokens) - 1)
        pg = self._pipeline_graph(u, len(tokens)) if u.kind == "pipeline" else None
        if pg is not None:
            out.append((reqs, pg.step(tokens, pos, seq, last)))
            return out
        tok = self._forward(u, tokens, pos, seq, last)
        out.append((reqs, tok))
        return out

    def _warm_up(self, tokens: int = 16):
        """One dummy ragged forward per unit on its scratch sequence slot
        before the clock starts: loads every kernel module on every device and
        sets the per-device smem attributes, so the first real request does
        not pay them.  Receiver weights are still garbage here — harmless, only
        the scratch KV slot is written."""
        torch = self.torch
        for u in self.units.values():
            scratch = u.stages[0].executor.scratch_seq
            n = min(tokens, self.max_len)
            self._forward(u, [0] * n, list(range(n)), [scratch] * n, [n - 1])
        for d in {st.device for u in self.units.values() for st in u.stages}:
            torch.cuda.synchronize(d)

    def run(self, trace, prompts: dict, mc_streams: dict, push_ctas: int = 0, pull_ctas: int = 64,
            timeout_s: float = 120.0, executor: str = "kernel"):
        """Launch the multicast, then serve ``trace`` (TraceRecords whose
        arrival_s is relative to the launch).  Returns the event list."""
        torch = self.torch
        devs = sorted(set(st.device for u in self.units.values() for st in u.stages) |
                      set(self.cluster.node_device(n) for n in self.receivers))
        self._warm_up()
        if self.use_graphs:
            from .llama import DecodeGraph
            for u in self.local_units.values():
                if u.graph is None:
                    u.graph = DecodeGraph(u.stages[0].executor, u.slots)
                    u.graph.capture()
                for cap in self.PREFILL_BUCKETS:     # prefill graphs too, before the clock
                    if cap <= self.max_len * u.slots:
                        self._prefill_graph(u, cap)
            for u in self.units.values():
                if u.kind == "pipeline":
                    for cap in [u.slots] + list(self.PREFILL_BUCKETS):
                        if cap <= self.max_len * u.slots:
                            self._pipeline_graph(u, cap)
        for d in devs:
            torch.cuda.synchronize(d)
        self.t0 = time.perf_counter()
        if executor == "ce":
            epoch = self.cluster.launch_devices_ce(mc_streams)
        else:
            epoch = self.cluster.launch_devices(mc_streams, push_ctas, pull_ctas)
        self.log(0.0, "scale_out", model=self.cfg.name, nodes=list(self.plan.nodes),
                 sources=list(self.plan.sources), strategy="lambda_scale")
        self.log(0.0, "allocation", allocated_gpus=len(self.receivers))
        pending = deque(sorted(trace, key=lambda r: (r.arrival_s, r.request_id)))
        queue = deque()
        live = {}
        tokens_emitted = 0
        while True:
            now = time.perf_counter() - self.t0
            if now > timeout_s:
                raise TimeoutError("serving loop exceeded its timeout")
            while pending and pending[0].arrival_s <= now:
                rec = pending.popleft()
                r = Request(rec, list(prompts[rec.request_id]))
                live[rec.request_id] = r
                queue.append(r)
                self.log(rec.arrival_s, "request_arrival", request=rec.request_id, model=rec.model_id)
            if not self.switched:
                t_cn = time.perf_counter()
                done = self.cluster.complete_nodes(epoch)
                if getattr(self, "profile_detail", None) is not None:
                    self.profile_detail.append(("complete_nodes", -1, 0, time.perf_counter() - t_cn))
                now = time.perf_counter() - self.t0
                for n in self.receivers:
                    if n not in self.block_complete_s and all(done[n]):
                        self.block_complete_s[n] = now
                for u in self.units.values():
                    if u.kind == "pipeline" and not u.active and not u.retired:
                        if all(all(done[st.node][b] for b in range(st.block_lo, st.block_hi + 1))
                               for st in u.stages):
                            u.active = True
                            self.activation_s[u.uid] = now
                all_done = all(all(done[n]) for n in self.receivers)
                if all_done and tokens_emitted >= self.switch_hold_tokens:
                    t_ms = time.perf_counter()
                    self._mode_switch(now)
                    if getattr(self, "profile_detail", None) is not None:
                        self.profile_detail.append(("mode_switch", -1, 0, time.perf_counter() - t_ms))
            self._admit(queue)
            t_enq = time.perf_counter()
            work = []
            for u in sorted(self.units.values(), key=lambda x: x.uid):
                if u.active and not u.retired and u.busy:
                    for w in self._step_unit(u) or []:
                        work.append((u, w))
            if not work:
                if not pending and not queue and all(r.done for r in live.values()) and self.switched:
                    break
                time.sleep(0.0002)
                continue
            t_sync = time.perf_counter()
            for d in {u.stages[0].device for u, _ in work} | {st.device for u, _ in work for st in u.stages}:
                # the compute stream only: a device-wide sync would also wait for the
                # multicast still landing blocks on its own stream
                torch.cuda.current_stream(d).synchronize()
            t_done = time.perf_counter()
            self.profile.append((t_enq - self.t0, t_sync - t_enq, t_done - t_sync,
                                 sum(len(w[0]) for _, w in work), sum(1 for _, w in work)))
            host = [(u, reqs, tok.cpu()) for u, (reqs, tok) in work]
            now = time.perf_counter() - self.t0
            for u, reqs, tok in host:
                for r, t in zip(reqs, tok.tolist()):
                    if r.needs_prefill:
                        r.kv_len = len(r.prompt) + len(r.out)
                        r.needs_prefill = False
                    else:
                        r.kv_len += 1
                    r.out.append(int(t))
                    tokens_emitted += 1
                    if r.first_token_s is None:
                        r.first_token_s = now
                    self.log(now, "token_emitted", request=r.rid, node=u.emit_node, cold_capacity=u.cold)
                    if r.done:
                        r.done_s = now
                        del u.busy[r.slot]
                        self.log(now, "request_done", request=r.rid, node=u.emit_node)
        if executor == "ce":
            for st in mc_streams.values():
                st.synchronize()
        else:
            self.cluster.wait_devices()
        for d in devs:
            torch.cuda.synchronize(d)
        self.requests = live
        return self.events


def generate(executor, prompts: list, max_new_tokens: int, use_graph: bool = True) -> list:
    """Greedy generation on one local replica — the reference has no
    ``generate()``; its per-request token loop (simengine.py:370-378,
    690-712) is the analogue.  ``executor`` is a full-model
    ``llama.LlamaExecutor``; ``prompts`` lists token-id lists (at most the
    executor's sequence slots).  Prefill is one ragged batch, decode steps
    replay a captured graph.  Returns the generated token lists."""
    import torch
    from .llama import DecodeGraph
    n = len(prompts)
    if n > executor.scratch_seq:
        raise ValueError("more prompts than the executor's sequence slots")
    dev = executor.torch_device
    toks, pos, seq, last = [], [], [], []
    for i, p in enumerate(prompts):
        toks += list(p)
        pos += list(range(len(p)))
        seq += [i] * len(p)
        last.append(len(toks) - 1)
    with torch.cuda.device(executor.device):
        t = torch.as_tensor(toks, dtype=torch.int32, device=dev)
        x, _ = executor.forward(tokens=t, pos=torch.as_tensor(pos, dtype=torch.int32, device=dev),
                                seq=torch.as_tensor(seq, dtype=torch.int32, device=dev), want_logits=False)
        logits = executor.head(x[torch.as_tensor(last, device=dev)].contiguous())
        nxt, _ = executor.greedy(logits)
        out = [[v] for v in nxt.cpu().tolist()]
        kv = [len(p) for p in prompts]
        graph = DecodeGraph(executor, n) if use_graph else None
        for _ in range(max_new_tokens - 1):
            cur = [o[-1] for o in out]
            if graph is not None:
                res = graph.step(cur, kv, list(range(n)))
                torch.cuda.current_stream().synchronize()
                vals = res.tolist()
            else:
                _, lg = executor.forward(tokens=torch.as_tensor(cur, dtype=torch.int32, device=dev),
                                         pos=torch.as_tensor(kv, dtype=torch.int32, device=dev),
                                         seq=torch.arange(n, dtype=torch.int32, device=dev))
                vals = executor.greedy(lg)[0].cpu().tolist()
            for o, v in zip(out, vals):
                o.append(int(v))
            kv = [k + 1 for k in kv]
    return out
