"""Small, single-process targets for `ncu --set full`: Llama-2-13B layer
shapes, 4 layers / 4 blocks (~3.9 GB image), host -> 1 GPU.

  python tools/ncu_target.py [iters]          in-kernel PCIe pull executor
  python tools/ncu_target.py [iters] verify   verify-as-it-lands kernel over a
                                              landed image (hybrid executor
                                              first; ncu serialises kernels, so
                                              the kernel is launched after the
                                              copy-engine flags are set)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import image as I  # noqa: E402
from paper_2502_09922_b200 import scaleout as SO  # noqa: E402

cfg = I.LlamaConfig("llama2-13b-4L", 4, 5120, 40, 40, 13824, 32000)
plan = SO.plan_scale_out(cfg, 2, 1, 4, host_source=True)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
if len(sys.argv) > 2 and sys.argv[2] == "verify":
    so = SO.ScaleOut(plan, tile_bytes=SO.HYBRID_TILE, executor="hybrid", seed=1, direction=1, copy_mode=0)
    so.load_sources()
    r = so.run()
    sums = torch.zeros(plan.block_count, dtype=torch.int64, device="cuda")
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        so.cluster.engine.verify(1, r.epoch, sums.data_ptr(), torch.cuda.current_stream().cuda_stream, 48)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"verify_ms={ms:.3f} GB/s={plan.layout.weights_bytes / ms / 1e6:.1f}")
    assert [int(x) & (2**64 - 1) for x in sums.tolist()] == so.checksums(1)
else:
    so = SO.ScaleOut(plan, tile_bytes=2 << 20, push_ctas=0, pull_ctas=64, seed=1, direction=1, copy_mode=0)
    so.load_sources()
    for _ in range(iters):
        r = so.run()
        print(f"kernel_ms={r.kernel_ms:.3f} GB/s={plan.layout.weights_bytes / r.kernel_ms / 1e6:.2f}")
so.close()
