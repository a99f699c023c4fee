"""Stage-to-stage activation hand-off over NVLink (dev tool, >= 2 GPUs).

  python tools/handoff_perf.py

Times ``lp_handoff`` (SM stores into the next stage's buffer, optional
sys-scope release of a flag the consumer waits on) GPU0 -> GPU1 for the
hidden-state sizes a λPipe pipeline moves — one decode row of Llama-3-8B
(d = 4096 fp32 = 16 KB), a 16-row decode batch, 1024- and 2048-token
prefills — against a copy-engine peer copy (torch ``copy_``), CUDA events on
the producer's stream, 200 repetitions each."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_09922_b200 import _native as N  # noqa: E402

lib = N.lib()
N.check(lib.lp_enable_peer(0, 1), "peer")
N.check(lib.lp_enable_peer(1, 0), "peer")
d = 4096
for rows in (1, 16, 256, 1024, 2048):
    src = torch.randn(rows, d, device="cuda:0")
    dst = torch.zeros(rows, d, device="cuda:1")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda:1")
    scratch = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    nbytes = src.numel() * 4
    s = torch.cuda.current_stream(0)
    res = {}
    for name in ("lp_handoff", "lp_handoff+flag", "peer copy_"):
        def go(i, name=name):
            if name == "peer copy_":
                dst.copy_(src, non_blocking=True)
            else:
                fl = C.c_void_p(flag.data_ptr()) if name.endswith("flag") else None
                N.check(lib.lp_handoff(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), nbytes, fl,
                                       i + 1, C.c_void_p(scratch.data_ptr()), C.c_void_p(s.cuda_stream)),
                        "lp_handoff")
        with torch.cuda.device(0):
            for i in range(10):
                go(i)
            torch.cuda.synchronize(0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for i in range(200):
                go(i)
            e1.record(s)
            torch.cuda.synchronize(0)
            us = e0.elapsed_time(e1) / 200 * 1e3
        torch.cuda.synchronize(1)
        assert torch.equal(dst.cpu(), src.cpu()), name
        res[name] = us
    print(f"rows={rows:5d} bytes={nbytes:>9d}  " + "  ".join(
        f"{k}: {v:7.2f} us ({nbytes / v / 1e3:6.1f} GB/s)" for k, v in res.items()), flush=True)
