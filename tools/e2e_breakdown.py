"""Where the N = 1 e2e step's time goes beyond the device-timed run (dev
tool): plan_scale_out, set_schedule (engine compile), run() wall vs its
CUDA-event time, the completion query — C3 host -> 1 GPU, hybrid executor."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_09922_b200 import scaleout as SO  # noqa: E402

torch.cuda.set_device(0)
plan = SO.plan_scale_out(bench.C3_MODEL, 2, 1, bench.C3_BLOCKS, host_source=True, strategy="lambda")
so = SO.ScaleOut(plan, distributed=False, tile_bytes=SO.HYBRID_TILE, push_ctas=0, pull_ctas=64, seed=bench.SEED,
                 device=0, direction=1, copy_mode=0, executor="hybrid", verify=True)
so.load_sources()
stream = torch.cuda.Stream()
rows = []
for i in range(6):
    so.poison(0x5A ^ i, stream)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p2 = SO.plan_scale_out(bench.C3_MODEL, 2, 1, bench.C3_BLOCKS, host_source=True, strategy="lambda")
    t1 = time.perf_counter()
    so.cluster.set_schedule(p2.schedule, p2.sources)
    t2 = time.perf_counter()
    r = so.run(stream)
    t3 = time.perf_counter()
    done = so.cluster.engine.complete(so.cluster.exec_nodes[0], r.epoch)
    t4 = time.perf_counter()
    rows.append((t1 - t0, t2 - t1, t3 - t2, r.kernel_ms / 1e3, t4 - t3, t4 - t0))
for row in rows[1:]:
    print("plan %.2f ms  set_schedule %.2f ms  run wall %.2f ms (events %.2f ms)  complete %.2f ms  total %.2f ms"
          % tuple(x * 1e3 for x in row))
so.close()
