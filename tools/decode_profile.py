"""One captured decode step of the 8B local replica, replayed a few times
(ncu target for the per-kernel launch list of a decode step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import engine as E  # noqa: E402
from paper_2502_09922_b200 import image as I  # noqa: E402
from paper_2502_09922_b200.llama import DecodeGraph, LlamaExecutor  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = I.CONFIGS["llama3-8b"]
lay = I.build_layout(cfg, 16)
ptr = E.dev_malloc(0, lay.weights_bytes)
E.fill_image(ptr, lay, 1)
ex = LlamaExecutor(lay, ptr, 0, max_seqs=B, max_len=256)
g = DecodeGraph(ex, B)
g.capture()
for _ in range(3):
    g.step([1] * B, [128] * B, list(range(B)))
torch.cuda.synchronize()
print("done")
