"""Benchmark of the λScale scaling hot path on B200 (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N ...)

Workload (BASELINE.json configs[2], the largest config that fits one GPU):
Llama-2-13B bf16 (26.03 GB packed image, b = 40 one-layer blocks) scaled out
from pinned host memory (schedule node 0, the reference's MEMORY tier) to N
GPUs with the reference's binomial λPipe schedule (n = N + 1 nodes, k = 1).
One step = one complete scale-out: every receiver ends holding the whole
model byte-exactly, checked EVERY step: receivers checksum each block while
it lands (lp_mc_verify) and the sums are compared with the source manifest.
Executor: scaleout.choose_executor — hybrid for host sources (PCIe hop as
pinned DMA on the copy engines, NVLink relays in the multicast kernel).

metric/value: aggregate delivered GB/s = N x model bytes / max-over-ranks
device time of one scale-out (CUDA events around it on its stream), with the
reference's λPipe binomial schedule at EVERY N.  Receivers are overwritten
with a byte pattern before every step (untimed), so each step's checksums
prove that step delivered the model.  At N >= 2 the line also carries
"sharded_host" (our non-reference host-load plan, labelled as such) and the
GPU-sourced multicast (Llama-3-8B, GPU0 -> N-1 peers, b = 16; BASELINE
configs[1] at N = 8) as "gpu_source"; at N >= 3 "execute_while_load"
(Llama-3-8B, 2 GPU sources, λPipe pipelines serving a burst while the rest
receive; tokens/s + TTFT), at N >= 4 "execute_while_load_70b" (BASELINE
configs[3] shape) and "bursty_trace" (configs[4]: the reference's synthetic
spike trace with repeated scale-outs).

cpu_baseline (rank 0, N = 1): the oracle's CPU restatement of the same
scale-out over host buffers (full image), plus BASELINE.md §3's other CPU
items: the unmodified reference planner's ms per plan and its simulator's
wall time on the C5 trace (from baseline/_ref), and the CPU logits oracle's
tokens/s.

--impl reference: the reference has no data plane (pure-Python planner +
cost-model simulator); its CPU path for this workload is the
oracle's restatement of the schedule's byte movement (oracle/dataplane.c,
all host cores) over the same full config (config.same_config; a
memory-bounded block prefix only if N + 1 images do not fit in host RAM).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scale-out time & aggregate GB/s (1→N GPUs); tokens/s + TTFT during load"
C3_MODEL, C3_BLOCKS = "llama2-13b", 40
C2_MODEL, C2_BLOCKS = "llama3-8b", 16     # serving (execute-while-load) plan
C2_MC_BLOCKS = 16                          # GPU-sourced multicast: measured best at N = 4 (0.675 vs 0.642 at
                                           # b = 32, profiles/r02/mc_gpu_source_n4_blocks.txt); the reference
                                           # planner's elbow is 10 (N = 4) / 14 (N = 8); round 1's copy
                                           # engines preferred 32 on one box (23.67 vs 24.04 ms)
SEED = 20250815
NCU_TRAFFIC_RATIO = (3.153332e9 + 10.150656e6) / 3193006080   # profiles/mc_kernel_host_pull_full_r01.csv


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# CPU path (oracle restatement) — reference arm and cpu_baseline


def mem_available() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


class CpuPort:
    """The oracle's CPU restatement of the C3 scale-out (oracle/dataplane.c
    lp_ref_execute: every transfer of the reference's λPipe schedule lines a
    memcpy, transfers of a step on all host threads, one barrier per step)
    over host buffers: node 0 = the host copy, nodes 1..N = receivers.  Runs
    the FULL image whenever (N + 1) images fit in 80 % of MemAvailable, else
    the longest block prefix that does (``same_config`` says which)."""

    def __init__(self, n_gpus: int, threads: int):
        import numpy as np
        from paper_2502_09922_b200 import scaleout as SO
        self.np = np
        self.threads = threads
        self.plan = SO.plan_scale_out(C3_MODEL, n_gpus + 1, 1, C3_BLOCKS, host_source=True)
        lay = self.plan.layout
        n = len(self.plan.nodes)
        budget = 0.8 * mem_available()
        nb = lay.plan.block_count
        span = lambda k: lay.block_offsets[k - 1] + lay.block_lengths[k - 1]   # noqa: E731
        while nb > 1 and n * span(nb) > budget:
            nb -= 1
        self.blocks = nb
        self.same_config = nb == lay.plan.block_count
        self.span = span(nb)
        keep = set(range(nb))
        self.lines = [ln for ln in self.plan.lines() if int(ln.split(",")[3]) in keep]
        self.offs, self.lens = lay.block_offsets[:nb], lay.block_lengths[:nb]
        self.delivered = sum(self.lens) * (n - 1)
        seed = np.random.default_rng(0).integers(0, 255, 64 << 20, dtype=np.uint8)
        self.src = np.empty(self.span, np.uint8)
        for o in range(0, self.span, seed.size):
            m = min(seed.size, self.span - o)
            self.src[o:o + m] = seed[:m]
        self.imgs = [self.src] + [np.empty(self.span, np.uint8) for _ in range(n - 1)]

    def step(self) -> float:
        from oracle import dataplane as D
        t0 = time.perf_counter()
        D.execute(self.imgs, self.offs, self.lens, self.lines, [0], threads=self.threads)
        return time.perf_counter() - t0

    def check(self) -> bool:
        """Wipe a sample of blocks on every receiver, run one more scale-out,
        and compare them with the source (a full compare of N x 26 GB would
        take longer than the runs)."""
        np = self.np
        sample = sorted({0, self.blocks // 2, self.blocks - 1})
        for im in self.imgs[1:]:
            for b in sample:
                im[self.offs[b]:self.offs[b] + self.lens[b]] = 0
        self.step()
        return all(np.array_equal(im[self.offs[b]:self.offs[b] + self.lens[b]],
                                  self.src[self.offs[b]:self.offs[b] + self.lens[b]])
                   for im in self.imgs[1:] for b in sample)

    def sample(self) -> str:
        what = "full image" if self.same_config else f"blocks 0..{self.blocks - 1} (memory-bounded prefix)"
        return (f"C3 λPipe schedule (n={len(self.plan.nodes)}, b={C3_BLOCKS}) executed host->host, {what}: "
                f"{sum(self.lens) / 1e9:.2f} GB per receiver, {self.threads} threads")


def reference_cpu_items(n_gpus: int, threads: int) -> dict:
    """BASELINE.md §3 CPU items beside the byte-movement port:
    (1) the real reference planner's wall time per plan, (2) the real
    reference simulator's run over the C5 burst trace — both from the
    unmodified reference installed in baseline/_ref (absent: reported as
    such) — and (4) the CPU logits oracle's tokens/s on the tiny model."""
    out = {}
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "blockcast")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        try:
            from blockcast import multicast as RM
            from blockcast import pipeline as RP

            def plan(model, size, layers, n, k, b):
                p = RM.partition_blocks(RM.ModelSpec(model, size, layers), b)
                nodes = list(range(n))
                g = RM.attach_orders(RM.partition_subgroups(nodes, nodes[:k]), RM.k_way_orders(b, k))
                sch = RM.compose_schedule(g, p)
                o = RP.completion_ordered_groups(g, sch)
                return [RP.assign_blocks_to_stages(x, [q.transfer_order for q in o], b, sch, i)
                        for i, x in enumerate(RP.generate_pipelines(o))]
            rows = {}
            for label, args in (("c3_host_to_%d_b40" % n_gpus, ("llama2-13b", 26031728640, 40, n_gpus + 1, 1, 40)),
                                ("c2_gpu0_to_7_b16", ("llama3-8b", 16060522496, 32, 8, 1, 16)),
                                ("c4_70b_1_to_8_b80_k2", ("llama3-70b", 141107412992, 80, 8, 2, 80))):
                reps, t0 = 0, time.perf_counter()
                while reps < 3 or time.perf_counter() - t0 < 1.0:
                    plan(*args)
                    reps += 1
                rows[label] = round((time.perf_counter() - t0) / reps * 1e3, 3)
            out["reference_planner_ms_per_plan"] = rows
            from blockcast import simengine as RS
            from blockcast import workload as RW
            trace = RW.synth_burst(0.05, 6.0, [120.0, 800.0, 1500.0], 1800.0, seed=4, spike_duration_s=60.0,
                                   output_tokens=(16, 32))
            t0 = time.perf_counter()
            res = RS.run(RS.ClusterSpec(), [RM.ModelSpec("m0", 13476831232, 32)], "lambda_scale", trace,
                         RS.AutoscalePolicy(), block_count=16)
            out["reference_simulator"] = {"s": round(time.perf_counter() - t0, 3), "requests": len(trace),
                                          "completed": res.report.requests_completed,
                                          "workload": "C5 synth_burst (1800 s, seed 4), Llama-2-7B size, lambda_scale, b=16"}
            out["reference_install"] = "baseline/_ref (pip --target from the unmodified reference)"
        except Exception as e:  # noqa: BLE001
            out["reference_error"] = f"{type(e).__name__}: {e}"
    else:
        out["reference_install"] = "absent (baseline/_ref not installed): planner/simulator items skipped"
    try:
        import torch
        from oracle import dataplane as D
        from oracle import llama as OL
        from paper_2502_09922_b200 import image as I
        torch.set_num_threads(threads)
        cfg = I.CONFIGS["tiny"]
        lay = I.build_layout(cfg, 4)
        W = OL.weights(lay, D.fill_image(lay, 7))
        prompt = list(range(1, 129))
        t0 = time.perf_counter()
        for _ in range(3):
            OL.forward(cfg, W, prompt, bf16=True)
        pre = 3 * 128 / (time.perf_counter() - t0)
        t0 = time.perf_counter()
        OL.greedy(cfg, W, prompt[:32], 8, bf16=True)
        dec = 8 / (time.perf_counter() - t0)
        out["oracle_tokens_per_s"] = {"prefill": round(pre, 1), "decode_recompute": round(dec, 2),
                                      "model": "tiny (4 layers, d=256)", "threads": threads,
                                      "note": "oracle/llama.py bf16 mode; decode re-runs the causal forward "
                                              "per token (no KV cache)"}
    except Exception as e:  # noqa: BLE001
        out["oracle_error"] = f"{type(e).__name__}: {e}"
    return out


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    port = CpuPort(args.gpus, threads)
    times = []
    for i in range(args.warmup + args.steps):
        dt = port.step()
        if i >= args.warmup:
            times.append(dt)
    T = statistics.median(times)
    ok = port.check()
    v = port.delivered / T / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(T * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{C3_MODEL} bf16 scale-out from the host copy to {args.gpus} receiver(s), "
                                   f"b={C3_BLOCKS}, k=1, λPipe schedule",
                       "same_config": port.same_config,
                       "executor": "oracle/dataplane.c lp_ref_execute (CPU memcpy per transfer, barrier per step)"},
            "byte_exact": ok,
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": port.sample()},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


POISON = True


def quiesce(distributed: bool) -> None:
    """Host-side fence across ranks: every rank's previous scale-out (whose
    relays may still be reading this rank's image) has finished."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
        torch.cuda.synchronize()


def timed_steps(so, steps, warmup, distributed, stream, want=None):
    """Device time per step (max over ranks).  With ``want`` (the source's
    per-block checksums) every step's verify-as-it-lands sums are checked;
    returns (times, all steps byte-exact, our kernel launches in timed steps
    summed over ranks)."""
    import torch
    import torch.distributed as dist
    times, ok, launches = [], True, 0
    for i in range(warmup + steps):
        if POISON:
            quiesce(distributed)         # every rank is done with the previous step (relays read peers)
            so.poison(0x5A ^ i, stream)  # receivers start every step without the model (untimed)
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()
        r = so.run(stream)
        t = torch.tensor([r.kernel_ms], device="cuda")
        if distributed:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if want is not None:
            ok = ok and all(v == want for v in r.checksums.values())   # sources hold no sums
        if i >= warmup:
            times.append(t.item())
            launches += r.launches
    if distributed:
        x = torch.tensor([launches, int(not ok)], device="cuda")
        dist.all_reduce(x)
        launches, ok = int(x[0].item()), x[1].item() == 0
    return times, ok, launches


def source_sums(so, rank, distributed, node=0):
    """Per-block checksums of the source image (node 0), on every rank."""
    import torch.distributed as dist
    sums = so.checksums(node) if rank == 0 else None
    if distributed:
        box = [sums]
        dist.broadcast_object_list(box, src=0)
        sums = box[0]
    return sums


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pull-ctas", type=int, default=64)
    ap.add_argument("--no-verify", action="store_true",
                    help="skip verify-as-it-lands (for ncu launch lists: ncu serialises kernels, so a kernel "
                         "waiting on copy-engine flags can never finish under it); bytes are then checked once "
                         "after the timed region")
    ap.add_argument("--strategy", default="lambda", choices=["lambda", "sharded_host"],
                    help="host-sourced scale-out plan of the headline value (default: the reference's λPipe "
                         "binomial schedule; sharded_host is always measured beside it at N >= 2)")
    ap.add_argument("--executor", default="auto", choices=["auto", "hybrid", "kernel", "ce"],
                    help="host-sourced scale-out executor (auto = scaleout.choose_executor)")
    ap.add_argument("--no-poison", action="store_true", help="A/B only: skip overwriting receivers between steps")
    ap.add_argument("--no-gpu-source", action="store_true")
    ap.add_argument("--no-serving", action="store_true")
    ap.add_argument("--requests", type=int, default=32)
    ap.add_argument("--no-burst", action="store_true")
    ap.add_argument("--no-serving-70b", action="store_true")
    ap.add_argument("--burst-compress", type=float, default=60.0)
    args = ap.parse_args()
    t_start = time.perf_counter()
    global POISON
    POISON = not args.no_poison
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2502_09922_b200 import _native
    from paper_2502_09922_b200 import scaleout as SO

    rank, world, local = env_rank()
    distributed = world > 1
    if distributed:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    _native.lib()
    dev = torch.cuda.current_device()
    stream = torch.cuda.Stream()
    N = world
    peaks = measured_peaks()

    # --- main workload: C3 host -> N GPUs -----------------------------------
    strategy = args.strategy
    plans = {st: SO.plan_scale_out(C3_MODEL, N + 1, 1, C3_BLOCKS, host_source=True, strategy=st)
             for st in ({strategy, "lambda", "sharded_host"} if N >= 2 else {strategy})}
    plan = plans[strategy]
    M = plan.layout.weights_bytes
    tiles = {"hybrid": SO.HYBRID_TILE, "kernel": 2 << 20, "ce": SO.CE_TILE}
    executor = SO.choose_executor(plan)[0] if args.executor == "auto" else args.executor
    # the policy's (strategy, executor) first and timed in full; the others
    # briefly, for the comparison table in config.host_executors
    arms = [(strategy, executor)] + [a for a in (("sharded_host", "hybrid"), ("lambda", "hybrid"),
                                                 ("lambda", "kernel"))
                                     if a != (strategy, executor) and a[0] in plans]
    host_exec = {}
    main_res = None
    for st, ex in arms:
        so = SO.ScaleOut(plans[st], distributed=distributed, tile_bytes=tiles[ex], push_ctas=0,
                         pull_ctas=args.pull_ctas, seed=SEED, device=dev, direction=1, copy_mode=0,
                         executor=ex, verify=not args.no_verify)
        so.load_sources()
        want = source_sums(so, rank, distributed)
        main = (st, ex) == (strategy, executor)
        if main:
            clocks = ClockSampler(dev)
            clocks.start()
        times, ok, launches = timed_steps(so, args.steps if main else 3, args.warmup, distributed,
                                          stream, want)
        if args.no_verify:   # one check after the timed region instead
            mine = [n for n in so.cluster.exec_nodes if n not in so.plan.sources]
            ok = all(so.checksums(n) == want for n in mine)
        T = statistics.median(times)
        host_exec[f"{st}/{ex}"] = {"ms": round(T, 3), "agg_GBps": round(N * M / (T * 1e-3) / 1e9, 3),
                                   "byte_exact": ok}
        if not main:
            so.close()
            continue
        clk = clocks.stop()
        main_res = (T, ok, launches)

        # --- e2e through the public API: plan + compile + launch + wait + read back
        # (the verified per-block checksums of every receiver: 8 B per block)
        my_nodes = so.cluster.exec_nodes
        e2e_times = []
        for i in range(args.warmup + args.steps):
            quiesce(distributed)
            so.poison(0xC3 ^ i, stream)
            if distributed:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p2 = SO.plan_scale_out(C3_MODEL, N + 1, 1, C3_BLOCKS, host_source=True, strategy=strategy)
            so.cluster.set_schedule(p2.schedule, p2.sources)
            r = so.run(stream)
            assert all(v == want for v in r.checksums.values()), "e2e step delivered wrong bytes"
            assert r.checksums or args.no_verify
            done = so.cluster.engine.complete(my_nodes[0], r.epoch)
            assert all(done)
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            if distributed:
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            if i >= args.warmup:
                e2e_times.append(dt.item())
        e2e = N * M / statistics.median(e2e_times) / 1e9
        so.close()
    T, ok, launches = main_res
    value = N * M / (T * 1e-3) / 1e9
    h2d = sum(plan.layout.block_lengths[int(ln.split(",")[3])] for ln in plan.lines()
              if int(ln.split(",")[1]) == 0)

    # --- GPU-sourced multicast (C2 shape): GPU0 -> N-1 peers -----------------
    gpu_source = None
    if distributed and N >= 2 and not args.no_gpu_source:
        plan2 = SO.plan_scale_out(C2_MODEL, N, 1, C2_MC_BLOCKS)
        M2 = plan2.layout.weights_bytes
        src_egress = sum(plan2.layout.block_lengths[int(ln.split(",")[3])] for ln in plan2.lines()
                         if int(ln.split(",")[1]) == 0)
        gpu_source = {"workload": f"{C2_MODEL} bf16 GPU0->{N - 1} peers, b={C2_MC_BLOCKS}, k=1",
                      "schedule_ceiling": round(M2 / src_egress, 4), "executors": {}}
        # in-kernel: 64 pull CTAs per receiver (96 CTAs / window 6 measured
        # 0.698 vs 0.673 without verify, but no better beside the verify
        # kernels: profiles/r02/mc_gpu_source_n4_ctas.txt)
        for name, kw in (("kernel", dict(executor="kernel", tile_bytes=2 << 20, pull_ctas=64, copy_mode=0)),
                         ("copy_engine", dict(executor="ce", tile_bytes=SO.CE_TILE))):
            so2 = SO.ScaleOut(plan2, distributed=True, push_ctas=0, seed=SEED, device=dev, direction=1,
                              verify=not args.no_verify, **kw)
            so2.load_sources()
            t2, exact, _ = timed_steps(so2, args.steps, args.warmup, True, stream, source_sums(so2, rank, True))
            T2 = statistics.median(t2)
            gpu_source["executors"][name] = {
                "ms": round(T2, 3), "agg_GBps": round((N - 1) * M2 / (T2 * 1e-3) / 1e9, 1),
                "nvlink_roofline_frac": round(M2 / (900e9 * T2 * 1e-3), 4), "byte_exact": exact,
                "detail": ("in-kernel NVLink pulls (LDG.128, 64 CTAs/rank, 2 MiB tiles)" if name == "kernel" else
                           "copy engines: cuStreamWaitValue32 -> cudaMemcpyAsync -> cuStreamWriteValue32, "
                           "256 MiB tiles, no SMs")}
            so2.close()
        best = min(gpu_source["executors"].items(), key=lambda kv: kv[1]["ms"])
        gpu_source.update({"best_executor": best[0], "ms": best[1]["ms"], "agg_GBps": best[1]["agg_GBps"],
                           "nvlink_roofline_frac": best[1]["nvlink_roofline_frac"]})

    # --- execute-while-load serving (tokens/s + TTFT during load) ------------
    serving = None
    serving_host = None
    serving70 = None
    burst = None
    if distributed and N >= 3 and not args.no_serving:
        torch.cuda.synchronize()
        # CPU (gloo) barrier: an NCCL barrier would leave a spinning kernel on
        # every idle rank's GPU and time-slice against rank 0's serving work
        cpu_group = dist.new_group(backend="gloo")
        dist.barrier(group=cpu_group)       # every rank has freed its images
        if rank == 0:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from serve_bench import run_serving
            try:
                serving = run_serving(N, model=C2_MODEL, k=2, blocks=C2_BLOCKS, requests=args.requests)
                serving["note"] = ("rank 0 drives all N GPUs from one process for this sub-measurement "
                                   "(cross-device pipelines); other ranks idle at a barrier")
            except Exception as e:  # noqa: BLE001
                serving = {"error": f"{type(e).__name__}: {e}"}
            try:   # tier-driven plan: GPU 0 + the pinned host copy as the k = 2 sources
                serving_host = run_serving(N, model=C2_MODEL, k=2, blocks=C2_BLOCKS, requests=args.requests,
                                           host_source=True)
                serving_host["note"] = ("startup_plan sources: GPU 0 (GPU tier) then the pinned host copy "
                                        "(MEMORY tier); one sub-group and its pipeline stages are fed over PCIe")
            except Exception as e:  # noqa: BLE001
                serving_host = {"error": f"{type(e).__name__}: {e}"}
            if N >= 4 and not args.no_serving_70b:
                # BASELINE configs[3]: Llama-3-70B (141 GB per replica) with λPipe
                # pipelines over partial replicas while the multicast runs
                import gc
                gc.collect()
                for d in range(N):
                    with torch.cuda.device(d):
                        torch.cuda.empty_cache()
                try:
                    serving70 = run_serving(N, model="llama3-70b", k=2, blocks=16, requests=16, executor="kernel",
                                            pull_ctas=64)
                    serving70["note"] = ("in-kernel multicast (64 CTAs per receiver) beside serving; rank 0 drives "
                                         "all N GPUs")
                except Exception as e:  # noqa: BLE001
                    serving70 = {"error": f"{type(e).__name__}: {e}"}
                gc.collect()
                for d in range(N):
                    with torch.cuda.device(d):
                        torch.cuda.empty_cache()
            if not args.no_burst:
                from burst_bench import run_burst
                try:
                    burst = run_burst(N, compress=args.burst_compress)
                except Exception as e:  # noqa: BLE001
                    burst = {"error": f"{type(e).__name__}: {e}"}
        dist.barrier(group=cpu_group)

    if rank == 0:
        threads = os.cpu_count() or 1
        cpu = None
        if N == 1:
            try:
                port = CpuPort(1, threads)
                port.step()                                   # page faults
                dt = statistics.median([port.step() for _ in range(2)])
                cpu = {"value": round(port.delivered / dt / 1e9, 3), "unit": "GB/s", "cores": threads,
                       "kind": "port", "sample": port.sample() + ", median of 2 steps after 1 warm-up",
                       "same_config": port.same_config}
                del port
            except Exception as e:  # noqa: BLE001
                cpu = {"value": None, "unit": "GB/s", "cores": threads, "kind": "port", "sample": f"failed: {e}"}
            cpu.update(reference_cpu_items(N, threads))
        host_rows = [ln.split(",") for ln in plan.lines() if ln.split(",")[1] == "0"]
        n_links = len({r[2] for r in host_rows})  # GPUs the host feeds = PCIe links in use
        achieved = h2d / (T * 1e-3) / 1e9       # host->GPU bytes per step / step time
        exec_desc = {
            "hybrid": f"hybrid: PCIe hop as pinned DMA on the copy engines ({SO.HYBRID_TILE >> 20} MiB tiles, "
                      f"per-tile flags), NVLink relays in the multicast kernel ({args.pull_ctas} CTAs/rank, "
                      "LDG.128 pulls)",
            "kernel": f"in-kernel PCIe/NVLink pulls (LDG.128, {args.pull_ctas} CTAs/rank, 2 MiB tiles)",
            "ce": "copy engines only (256 MiB tiles)"}[executor]
        if executor == "kernel":
            traffic, tnote = int(NCU_TRAFFIC_RATIO * M), (
                "dram read+write per launch from ncu --set full of the same kernel "
                "(profiles/mc_kernel_host_pull_full_r01.csv: 3.163 GB for a 3.193 GB image, ratio 0.991) "
                "scaled to this image")
        else:
            traffic, tnote = None, (
                "the PCIe hop is copy-engine DMA, not an SM kernel; the in-kernel PCIe pull executor's ncu "
                "traffic is 0.991 x image bytes (profiles/mc_kernel_host_pull_full_r01.csv)")
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(T, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{C3_MODEL} bf16 ({M / 1e9:.2f} GB) scale-out from pinned host memory "
                                   f"to {N} GPU(s), b={C3_BLOCKS}, k=1",
                       "strategy": {"lambda": f"reference λPipe binomial schedule ({plan.schedule.step_count} "
                                              "steps, host = node 0)",
                                    "sharded_host": "sharded host load: every GPU DMAs a disjoint block shard "
                                                    "over its own PCIe link, shards exchanged over NVLink "
                                                    f"(scaleout.sharded_host_schedule, {plan.schedule.step_count}"
                                                    " steps)"}[strategy],
                       "executor": exec_desc,
                       "host_executors": host_exec,
                       "verify": "every step: receivers checksum each block while it lands (lp_mc_verify, "
                                 "48-96 CTAs on a side stream) and the sums are read back and compared with the "
                                 "source manifest",
                       "l2": "inputs larger than L2 (26 GB image per step)",
                       "parallelism": f"{N} GPU ranks, one process per GPU"},
            "scale_out_ms": round(T, 3), "byte_exact": ok,
            "roofline": {"bound": "pcie", "achieved": round(achieved, 2),
                         "peak": 64.0 * n_links, "unit": "GB/s", "frac": round(achieved / (64.0 * n_links), 4),
                         "achieved_note": f"host bytes per step / step time over the {n_links} PCIe link(s) the "
                                          "plan drives (one per GPU the host sends to)",
                         "peak_note": "PCIe Gen5 x16 nominal per link (the reference's h2d_Bps) x links; measured DMA H2D on "
                                      "this pool 55.6 GB/s per link, 215 GB/s for 4 concurrent links (profiles/probe_r01.json, tools/h2d_concurrency.py)",
                         "traffic": traffic, "traffic_note": tnote},
            "e2e": {"value": round(e2e, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(12 * plan.block_count * N),
                    "path": "paper_2502_09922_b200.scaleout: plan_scale_out + set_schedule + run (verified "
                            "checksums read back) + completion readback"},
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
            "peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "bf16_tflops": peaks.get("bf16_tflops")},
        }
        if N >= 2 and "sharded_host/hybrid" in host_exec:
            line["sharded_host"] = dict(host_exec["sharded_host/hybrid"], note=(
                "NOT the reference schedule: every GPU DMAs a disjoint block shard over its own PCIe link and the "
                "shards rotate over NVLink (scaleout.sharded_host_schedule); reported beside the λPipe headline"))
        if gpu_source:
            line["gpu_source"] = gpu_source
        if serving:
            line["execute_while_load"] = serving
        if serving_host:
            line["execute_while_load_host_source"] = serving_host
        if serving70:
            line["execute_while_load_70b"] = serving70
        if burst:
            line["bursty_trace"] = burst
        line["bench_wall_s"] = round(time.perf_counter() - t_start, 1)
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
