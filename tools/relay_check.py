"""Single-process multi-GPU relay check (dev tool).

  python tools/relay_check.py N K B EXECUTOR    (EXECUTOR: ce | kernel)

One process drives N GPUs (engine.Cluster.devices, as serving does) through
the reference's schedule for (n = N, k = K, b = B) — with K < N/2 the groups
have relays, so receivers wait on OTHER receivers' flags across devices.
Prints the time and checks every receiver byte-exact."""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import _native as N  # noqa: E402
from paper_2502_09922_b200 import engine as E  # noqa: E402
from paper_2502_09922_b200 import image as I  # noqa: E402
from paper_2502_09922_b200 import scaleout as SO  # noqa: E402

n, k, b = (int(x) for x in sys.argv[1:4])
executor = sys.argv[4] if len(sys.argv) > 4 else "ce"
cfg = I.LlamaConfig("llama3-8b-8L", 8, 4096, 32, 8, 14336, 128256)
plan = SO.plan_scale_out(cfg, n, k, b)
lay = plan.layout
tile = SO.CE_TILE if executor == "ce" else 2 << 20
cl = E.Cluster.devices(list(range(n)), lay.block_offsets, lay.block_lengths, lay.weights_bytes, tile_bytes=tile)
for s in plan.sources:
    E.load_source_image(cl, s, lay, 3)
cl.set_schedule_all(plan.schedule, plan.sources)
for d in range(n):
    N.call("lp_set_device", d)
    cl.per_device[d].configure(int(os.environ.get("LP_RELAY_DIR", "1")), 0, 0, 16384, 3)   # 1 pull, 0 push
streams = {d: torch.cuda.Stream(device=d) for d in range(n)}
print("schedule:", plan.lines(), flush=True)
for rep in range(3):
    for d in range(n):
        torch.cuda.synchronize(d)
    t0 = time.perf_counter()
    if executor == "ce":
        if os.environ.get("LP_RELAY_REVERSE"):      # experiment: enqueue receivers last-to-first
            cl.epoch += 1
            for nb in reversed(cl.nodes):
                if nb.kind == E.LP_NODE_GPU:
                    N.call("lp_set_device", nb.device)
                    cl.per_device[nb.device].run_ce(nb.node, cl.epoch, [streams[nb.device].cuda_stream])
        else:
            cl.launch_devices_ce(streams)
        print(f"rep {rep}: enqueued in {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
        for st in streams.values():
            st.synchronize()
    else:
        cl.launch_devices(streams, 0, 64)
        cl.wait_devices()
    print(f"rep {rep}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
want = E.block_checksums(cl.node(plan.sources[0]).image, lay.block_offsets, lay.block_lengths)
for node in plan.receivers:
    N.call("lp_set_device", cl.node_device(node))
    assert E.block_checksums(cl.node(node).image, lay.block_offsets, lay.block_lengths) == want, node
print("byte-exact", flush=True)
cl.close()
