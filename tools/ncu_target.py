"""Small, single-process target for `ncu --set full` of the multicast kernel
(the bench's dominant kernel): Llama-2-13B layer shapes, 4 layers / 4 blocks
(~3.9 GB image), host -> 1 GPU, same engine settings as bench.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import image as I  # noqa: E402
from paper_2502_09922_b200 import scaleout as SO  # noqa: E402

cfg = I.LlamaConfig("llama2-13b-4L", 4, 5120, 40, 40, 13824, 32000)
plan = SO.plan_scale_out(cfg, 2, 1, 4, host_source=True)
so = SO.ScaleOut(plan, tile_bytes=2 << 20, push_ctas=0, pull_ctas=64, seed=1, direction=1, copy_mode=0)
so.load_sources()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    r = so.run()
    print(f"kernel_ms={r.kernel_ms:.3f} GB/s={plan.layout.weights_bytes / r.kernel_ms / 1e6:.2f}")
so.close()
