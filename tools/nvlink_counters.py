"""NVLink data counters around a command (copy-engine evidence, no ncu):

  python tools/nvlink_counters.py -- <command ...>

Reads NVML's per-link NVLink byte counters (falling back to ``nvidia-smi
nvlink -gt d``) for every GPU before and after the command and prints one JSON line with the
per-GPU byte deltas, so a copy-engine multicast (which ncu's kernel counters
cannot see) is measured the same way the in-kernel one is: bytes that crossed
NVLink per GPU vs the schedule's delivered bytes.
"""
import json
import re
import subprocess
import sys
import time


def snapshot_smi() -> dict:
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d"], capture_output=True, text=True).stdout
    gpu, res = None, {}
    for line in out.splitlines():
        m = re.match(r"GPU (\d+):", line.strip())
        if m:
            gpu = int(m.group(1))
            res[gpu] = {"tx": 0, "rx": 0}
            continue
        m = re.search(r"Data Tx:\s*(\d+)\s*KiB", line)
        if m and gpu is not None:
            res[gpu]["tx"] += int(m.group(1)) * 1024
        m = re.search(r"Data Rx:\s*(\d+)\s*KiB", line)
        if m and gpu is not None:
            res[gpu]["rx"] += int(m.group(1)) * 1024
    return res


def snapshot_nvml() -> dict:
    """Per-GPU sums over links of NVML's NVLink byte counters (field values
    NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES, scope = link)."""
    import pynvml as nv
    nv.nvmlInit()
    res = {}
    for g in range(nv.nvmlDeviceGetCount()):
        h = nv.nvmlDeviceGetHandleByIndex(g)
        tx = rx = 0
        for link in range(18):
            try:
                vals = nv.nvmlDeviceGetFieldValues(h, [(nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, link),
                                                       (nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, link)])
            except Exception:  # noqa: BLE001
                continue
            if vals[0].nvmlReturn == 0:
                tx += vals[0].value.ullVal
            if vals[1].nvmlReturn == 0:
                rx += vals[1].value.ullVal
        res[g] = {"tx": tx, "rx": rx}
    return res


def snapshot() -> dict:
    try:
        n = snapshot_nvml()
        if any(v["tx"] or v["rx"] for v in n.values()):
            return {"nvml": n}
    except Exception:  # noqa: BLE001
        n = None
    return {"smi": snapshot_smi(), "nvml": n}


def main():
    cmd = sys.argv[sys.argv.index("--") + 1:] if "--" in sys.argv else sys.argv[1:]
    a = snapshot()
    t0 = time.time()
    rc = subprocess.run(cmd).returncode
    dt = time.time() - t0
    b = snapshot()
    src = "nvml" if "nvml" in b and b["nvml"] else "smi"
    A, B = a.get(src) or {}, b.get(src) or {}
    delta = {g: {"tx_bytes": B[g]["tx"] - A[g]["tx"], "rx_bytes": B[g]["rx"] - A[g]["rx"]} for g in B if g in A}
    print(json.dumps({"nvlink_counters": delta, "command": " ".join(cmd), "rc": rc, "wall_s": round(dt, 2),
                      "source": {"nvml": "NVML field values NVLINK_COUNT_XMIT/RCV_BYTES summed over links",
                                 "smi": "nvidia-smi nvlink -gt d (Data Tx/Rx KiB per link)"}[src]}), flush=True)
    return rc


if __name__ == "__main__":
    sys.exit(main())
