"""Concurrent pinned-host -> GPU DMA on every rank (PCIe topology probe).

  torchrun --nproc-per-node 4 tools/h2d_concurrency.py --gib 4 [--shared]
Each rank copies its own pinned buffer (cudaHostAlloc via torch) or, with
--shared, a disjoint slice of ONE /dev/shm image registered in every rank
(engine.HostImage, as the HOST node of a scale-out) to its GPU; prints
per-rank and aggregate GB/s for 1, 2, ... N ranks active at once."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist

ap = argparse.ArgumentParser()
ap.add_argument("--gib", type=float, default=4)
ap.add_argument("--shared", action="store_true")
ap.add_argument("--chunk-mib", type=int, default=0)
a = ap.parse_args()
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(r)
n = int(a.gib * (1 << 30))
d = torch.empty(n, dtype=torch.uint8, device="cuda")
if a.shared:
    from paper_2502_09922_b200 import engine as E
    if r == 0:
        img = E.HostImage(n * w, "h2d_probe", create=True)
        img.array[:: 1 << 20] = 1
    dist.barrier()
    if r != 0:
        img = E.HostImage(n * w, "h2d_probe", create=False)
    src_ptr = img.device_ptr + r * n
else:
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h[:: 1 << 20] = 1
    src_ptr = h.data_ptr()
cudart = torch.cuda.cudart()
chunk = (a.chunk_mib << 20) or n


def copy():
    s = torch.cuda.current_stream().cuda_stream
    from paper_2502_09922_b200 import _native as N
    import ctypes as C
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        N.call("lp_memcpy", C.c_void_p(d.data_ptr() + off), C.c_void_p(src_ptr + off), m, C.c_void_p(s))


res = {}
for active in sorted({1, 2, w} | ({4} if w >= 4 else set())):
    dist.barrier()
    ms = None
    if r < active:
        for it in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            copy()
            e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1)
            ms = t if ms is None else min(ms, t)
    dist.barrier()
    out = [None] * w
    dist.all_gather_object(out, ms)
    if r == 0:
        per = [n / (x * 1e-3) / 1e9 for x in out if x]
        res[active] = {"per_rank_GBps": [round(x, 1) for x in per], "aggregate_GBps": round(sum(per), 1)}
        print("shared" if a.shared else "private", a.chunk_mib, active, json.dumps(res[active]), flush=True)
dist.barrier()
if a.shared:
    img.close(unlink=r == 0)
dist.destroy_process_group()
