"""One-off hardware probe: topology, host cores, peer-copy and H2D bandwidth."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
try:
    out["lscpu"] = subprocess.run(["bash", "-c", "lscpu | egrep 'Model name|Socket|Thread|Core|NUMA'"], capture_output=True, text=True).stdout
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
    out["smi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout
except Exception as e:
    out["err"] = str(e)
n = torch.cuda.device_count()
out["ndev"] = n
def bw_copy(dst, src, iters=10):
    s = torch.cuda.current_stream()
    for _ in range(2): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(iters): dst.copy_(src, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    return src.numel() * src.element_size() * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9
sz = 1 << 30
h = torch.empty(sz, dtype=torch.uint8).pin_memory()
for d in range(n):
    with torch.cuda.device(d):
        g = torch.empty(sz, dtype=torch.uint8, device=f"cuda:{d}")
        out[f"h2d_GBps_dev{d}"] = bw_copy(g, h, 5)
        out[f"d2h_GBps_dev{d}"] = bw_copy(h, g, 5)
if n > 1:
    a = torch.empty(sz, dtype=torch.uint8, device="cuda:0")
    for d in range(1, n):
        b = torch.empty(sz, dtype=torch.uint8, device=f"cuda:{d}")
        with torch.cuda.device(0):
            out[f"p2p_0to{d}_GBps"] = bw_copy(b, a, 10)
    # concurrent H2D to all GPUs
    gs = [torch.empty(sz, dtype=torch.uint8, device=f"cuda:{d}") for d in range(n)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        for d in range(n):
            with torch.cuda.device(d):
                gs[d].copy_(h, non_blocking=True)
    for d in range(n): torch.cuda.synchronize(d)
    out["h2d_concurrent_all_GBps"] = 3 * n * sz / (time.perf_counter() - t0) / 1e9
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
