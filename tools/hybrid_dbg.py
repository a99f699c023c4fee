"""Debug: hybrid executor + verify on one GPU (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_09922_b200 import scaleout as SO, engine as E

def case(model, n, b, tile, verify, own_stream, ex="hybrid", vctas=8, pull=8):
    plan = SO.plan_scale_out(model, n, 1, b, host_source=True)
    so = SO.ScaleOut(plan, executor=ex, tile_bytes=tile, pull_ctas=pull, push_ctas=0, direction=1, copy_mode=0,
                     verify=verify, verify_ctas=vctas)
    so.cluster.engine.set_option("timeout_ms", 4000)
    so.load_sources()
    st = torch.cuda.Stream() if own_stream else None
    try:
        for i in range(2):
            r = so.run(st)
            print(model, n, b, tile, verify, own_stream, ex, "ok", round(r.kernel_ms, 2), r.launches,
                  {k: v[:2] for k, v in r.checksums.items()}, flush=True)
    except Exception as e:
        print(model, n, b, tile, verify, own_stream, ex, "FAIL", e, flush=True)
        torch.cuda.synchronize()
        lay = plan.layout
        nt = [(x + tile - 1) // tile for x in lay.block_lengths]
        T = sum(nt)
        for node in plan.receivers:
            nb = so.cluster.node(node)
            fl = E.device_view(nb.signals, T * 4, 0, torch.int32).cpu().tolist()
            off = (T * 4 + 255) // 256 * 256
            cnt = E.device_view(nb.signals + off, len(nt) * 4, 0, torch.int32).cpu().tolist()
            print(" node", node, "ntiles", nt, "counts", cnt, "flags", fl, flush=True)
        print(" lines", plan.lines(), flush=True)
    so.close()

for args in [("tiny", 3, 4, 512 << 10, True, False),
             ("llama2-13b", 2, 40, 16 << 20, True, True, "hybrid", 8, 64),
             ("llama2-13b", 2, 40, 64 << 20, True, True, "hybrid", 32, 64),
             ("llama2-13b", 3, 40, 16 << 20, True, True, "hybrid", 32, 64),
             ("llama2-13b", 3, 40, 16 << 20, False, True, "hybrid", 32, 64),
             ("llama2-13b", 3, 40, 2 << 20, False, True, "kernel", 32, 64)]:
    case(*args)
