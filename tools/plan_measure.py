"""``blockcast plan`` / ``sweep b=`` on real GPUs.

  python tools/plan_measure.py --gpus 4 --model llama3-8b --k 1 --b 16 --outdir DIR
  python tools/plan_measure.py --gpus 4 --model llama3-8b --k 1 --sweep-b 4,8,16,32 --outdir DIR

Writes what the reference's ``cmd_plan`` writes (cli.py:288-339) —
``schedule.txt``, ``pipelines.txt`` (byte-identical to the reference planner),
``summary.txt`` with the reference's modelled lines (cluster = one 8×B200
box: NVLink 900 GB/s as the fabric, ``cluster.b200_box``) — and appends the
MEASURED counterparts: the schedule executed on the copy engines of N GPUs
(one process, ``engine.Cluster.devices``, push direction), a CUDA event
recorded on each receiver's side stream as each block lands
(``lp_mc_landing_events``: waits on the receiver's own block counters):
transfer time, per-node completion, per-step time and the first pipeline's
activation (its stages' blocks landed).  ``--sweep-b`` adds ``sweep.csv``
in the reference's sweep layout (cli.py:372-410) with the measured columns
beside the modelled ``predicted_transfer_s`` — the real-hardware elbow
instead of the modelled one.  Every run is checked byte-exact.
"""
import argparse
import ctypes as C
import os
import statistics
import sys
from pathlib import Path

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _fmt(x):
    from paper_2502_09922_b200.workload import fmt
    return fmt(x)


def measure(model: str, n: int, k: int, b: int, reps: int = 3, seed: int = 5, ce_streams: int = 1):
    import torch

    from paper_2502_09922_b200 import _native as N
    from paper_2502_09922_b200 import engine as E
    from paper_2502_09922_b200 import scaleout as SO

    plan = SO.plan_scale_out(model, n, k, b)
    lay = plan.layout
    cl = E.Cluster.devices(list(range(n)), lay.block_offsets, lay.block_lengths, lay.weights_bytes,
                           tile_bytes=SO.CE_TILE)
    try:
        for s in plan.sources:
            E.load_source_image(cl, s, lay, seed)
        cl.set_schedule_all(plan.schedule, plan.sources)
        streams = {d: [torch.cuda.Stream(device=d) for _ in range(ce_streams)] for d in range(n)}  # CE ops
        ev_streams = {d: torch.cuda.Stream(device=d) for d in range(n)}    # landing events

        def event(dev):
            N.call("lp_set_device", dev)
            h = C.c_void_p()
            N.call("lp_event_create", C.byref(h))
            return h.value

        recv = plan.receivers
        dev_of = {node: cl.node_device(node) for node in plan.nodes}
        start = {node: event(dev_of[node]) for node in recv}
        blk_ev = {node: [event(dev_of[node]) for _ in range(b)] for node in recv}
        runs = []
        for rep in range(reps + 1):
            for d in range(n):
                torch.cuda.synchronize(d)
            for node in recv:
                d = dev_of[node]
                N.call("lp_set_device", d)
                N.call("lp_event_record", C.c_void_p(start[node]), C.c_void_p(ev_streams[d].cuda_stream))
            epoch = cl.launch_devices_ce(streams)          # push direction (see launch_devices_ce)
            for node in recv:
                d = dev_of[node]
                N.call("lp_set_device", d)
                cl.per_device[d].landing_events(node, epoch, ev_streams[d].cuda_stream, blk_ev[node])
            arr = {}
            for node in recv:
                ms = C.c_float()
                row = []
                for e in blk_ev[node]:
                    N.call("lp_event_elapsed_ms", C.c_void_p(start[node]), C.c_void_p(e), C.byref(ms))
                    row.append(ms.value / 1e3)
                arr[node] = row
            if rep > 0:
                runs.append(arr)
        want = E.block_checksums(cl.node(plan.sources[0]).image, lay.block_offsets, lay.block_lengths)
        for node in recv:
            N.call("lp_set_device", dev_of[node])
            assert E.block_checksums(cl.node(node).image, lay.block_offsets, lay.block_lengths) == want, node
    finally:
        cl.close()

    def act(arr):
        acts = [max(max(arr[st.node][x] for x in range(st.block_lo, st.block_hi + 1))
                    for st in ep.stages if st.block_lo <= st.block_hi) for ep in plan.pipelines]
        return min(acts) if acts else None

    med = lambda xs: statistics.median(xs)  # noqa: E731
    total = med([max(max(r[n_]) for n_ in recv) for r in runs])
    return {
        "plan": plan,
        "transfer_s": total,
        "completion_s": {node: med([max(r[node]) for r in runs]) for node in recv},
        "first_activation_s": med([act(r) for r in runs]) if plan.pipelines else None,
        "nvlink_frac": lay.weights_bytes / (900e9 * total),
    }


def write_plan(outdir: Path, model: str, k: int, m: dict):
    from paper_2502_09922_b200.cluster import b200_box, transfer_step_time
    from paper_2502_09922_b200.multicast import predicted_transfer_s, schedule_summary
    from paper_2502_09922_b200.pipeline import pipelines_to_lines

    plan = m["plan"]
    n, b = len(plan.nodes), plan.block_count
    cluster = b200_box(node_count=n)
    sched = plan.schedule
    step_s = transfer_step_time(sched, plan.layout.plan, cluster)
    eps = plan.pipelines
    first_act = min(ep.activation_step for ep in eps) if eps else -1
    outdir.mkdir(parents=True, exist_ok=True)
    (outdir / "schedule.txt").write_text("\n".join(plan.lines()) + "\n")
    lines = pipelines_to_lines(eps)
    (outdir / "pipelines.txt").write_text("\n".join(lines) + ("\n" if lines else ""))
    size = plan.layout.weights_bytes
    out = [
        f"model: {model}", f"model_bytes: {size}", f"nodes: {n}", f"sources_k: {k}", f"block_count: {b}",
        f"step_count: {sched.step_count}", f"step_time_s: {_fmt(step_s)}",
        f"predicted_transfer_s: {_fmt(predicted_transfer_s(size, b, n, cluster.step_fixed_overhead_s, cluster.nic_Bps))}",
        f"first_pipeline_activation_step: {first_act}",
        f"first_pipeline_activation_s: {_fmt((first_act + 1) * step_s)}",
        f"pipeline_count: {len(eps)}",
    ]
    for node, step in schedule_summary(sched)["completion_step"].items():
        out.append(f"completion_step node {node}: {step}")
    out += [
        "measured_executor: copy engines, push direction (256 MiB tiles), one process driving the GPUs, byte-exact",
        f"measured_transfer_s: {_fmt(m['transfer_s'])}",
        f"measured_step_time_s: {_fmt(m['transfer_s'] / sched.step_count)}",
        f"measured_first_pipeline_activation_s: {_fmt(m['first_activation_s'])}",
        f"measured_nvlink_roofline_frac: {_fmt(m['nvlink_frac'])}",
    ]
    for node, t in sorted(m["completion_s"].items()):
        out.append(f"measured_completion_s node {node}: {_fmt(t)}")
    (outdir / "summary.txt").write_text("\n".join(out) + "\n")
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--b", type=int, default=16)
    ap.add_argument("--sweep-b", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ce-streams", type=int, default=1, help="copy-engine streams per GPU (ops round-robin)")
    ap.add_argument("--outdir", default="gpurun_out/plan_measure")
    a = ap.parse_args()
    out = Path(a.outdir)
    if not a.sweep_b:
        print("\n".join(write_plan(out, a.model, a.k, measure(a.model, a.gpus, a.k, a.b, a.reps, ce_streams=a.ce_streams))))
    else:
        from paper_2502_09922_b200.cluster import b200_box
        from paper_2502_09922_b200.image import CONFIGS, model_spec
        from paper_2502_09922_b200.multicast import predicted_transfer_s, select_block_count
        cl = b200_box(node_count=a.gpus)
        spec = model_spec(CONFIGS[a.model])
        elbow = select_block_count(spec, a.gpus, cl.step_fixed_overhead_s, cl.nic_Bps)
        rows = ["axis,value,elbow_b,predicted_transfer_s,measured_transfer_s,"
                "measured_first_pipeline_activation_s,measured_nvlink_roofline_frac"]
        for raw in a.sweep_b.split(","):
            b = int(raw)
            m = measure(a.model, a.gpus, a.k, b, a.reps, ce_streams=a.ce_streams)
            write_plan(out / f"b_{b}", a.model, a.k, m)
            size = m["plan"].layout.weights_bytes
            rows.append(f"b,{b},{elbow},{_fmt(predicted_transfer_s(size, b, a.gpus, cl.step_fixed_overhead_s, cl.nic_Bps))},"
                        f"{_fmt(m['transfer_s'])},{_fmt(m['first_activation_s'])},{_fmt(m['nvlink_frac'])}")
            print(rows[-1], flush=True)
        out.mkdir(parents=True, exist_ok=True)
        (out / "sweep.csv").write_text("\n".join(rows) + "\n")
