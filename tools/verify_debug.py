"""Debug: verify-as-it-lands sums on the hybrid / kernel executors (tiny)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dataplane as D  # noqa: E402
from paper_2502_09922_b200 import scaleout as SO  # noqa: E402

for n, k, b, host, ex, tile in [(2, 1, 4, True, "hybrid", 1 << 20), (4, 2, 3, False, "kernel", 65536),
                                (3, 1, 4, True, "ce", 1 << 20)]:
    plan = SO.plan_scale_out("tiny", n, k=k, block_count=b, host_source=host)
    so = SO.ScaleOut(plan, executor=ex, tile_bytes=tile, pull_ctas=8, push_ctas=0, direction=1, copy_mode=0,
                     verify=True, verify_ctas=8)
    so.load_sources()
    lay = plan.layout
    want = D.block_checksums(D.fill_image(lay, 0), lay.block_offsets, lay.block_lengths)
    for it in range(2):
        r = so.run()
        torch.cuda.synchronize()
        for node in plan.receivers:
            got = r.checksums[node]
            print(n, k, b, ex, "run", it, "node", node, "ok" if got == want else
                  f"BAD {[int(g == w) for g, w in zip(got, want)]}", "complete", so.cluster.engine.complete(node, r.epoch),
                  "after-run sums ok", so.checksums(node) == want, flush=True)
            buf = so._vbuf[node][0]
            print("   device sums now ok:", [int(x) & 0xFFFFFFFFFFFFFFFF for x in buf.cpu().tolist()] == want)
    so.close()
