"""Single-process NVLink target for `ncu --set full` (needs >= 2 GPUs).

  python tools/ncu_nvlink_target.py [n_gpus] [iters] [layers]

GPU0 holds a Llama-3-8B-shaped image (``layers`` decoder layers, one block
per layer, vocab tensors in block 0); the reference's binomial schedule
(n = n_gpus, k = 1) moves it to the other GPUs with the in-kernel executor
(pull direction, LDG.128, 64 CTAs, 2 MiB tiles), one kernel per device from
this one process (engine.Cluster.devices).  With n_gpus = 2 the receiver's
kernel reads GPU0 over NVLink and writes local HBM; ncu serialises the two
launches, which is safe for the pull direction: the source's flags are set at
load time, so the receiver never waits on a kernel that has not run.
(n_gpus > 2 relays would wait on a relay's kernel: run those without ncu.)

Prints per-iteration kernel time and payload GB/s (not a bench number when
run under ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import engine as E  # noqa: E402
from paper_2502_09922_b200 import image as I  # noqa: E402
from paper_2502_09922_b200 import scaleout as SO  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
layers = int(sys.argv[3]) if len(sys.argv) > 3 else 8
cfg = I.LlamaConfig(f"llama3-8b-{layers}L", layers, 4096, 32, 8, 14336, 128256)
plan = SO.plan_scale_out(cfg, n, 1, layers)
lay = plan.layout
cl = E.Cluster.devices(list(range(n)), lay.block_offsets, lay.block_lengths, lay.weights_bytes)
cl.engine.configure(1, 0, 0, 16384, 3)
for eng in cl.per_device.values():
    eng.configure(1, 0, 0, 16384, 3)
E.load_source_image(cl, 0, lay, 7)
cl.set_schedule_all(plan.schedule, plan.sources)
streams = {d: torch.cuda.Stream(device=d) for d in range(n)}
want = E.block_checksums(cl.node(0).image, lay.block_offsets, lay.block_lengths)
for _ in range(iters):
    for d in range(n):
        torch.cuda.synchronize(d)
    evs = {}
    for d in range(1, n):
        with torch.cuda.device(d):
            evs[d] = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            evs[d][0].record(streams[d])
    cl.launch_devices(streams, 0, 64)
    for d in range(1, n):
        with torch.cuda.device(d):
            evs[d][1].record(streams[d])
    for d in range(n):
        torch.cuda.synchronize(d)
    ms = max(a.elapsed_time(b) for a, b in evs.values())
    print(f"n={n} image={lay.weights_bytes / 1e9:.3f} GB kernel_ms={ms:.3f} "
          f"GB/s per receiver={lay.weights_bytes / ms / 1e6:.1f}", flush=True)
for node in range(1, n):
    with torch.cuda.device(node):
        got = E.block_checksums(cl.node(node).image, lay.block_offsets, lay.block_lengths)
    assert got == want, f"node {node} bytes differ"
print("byte-exact on every receiver")
cl.close()
