"""NVLink data counters around a command (copy-engine evidence, no ncu):

  python tools/nvlink_counters.py -- <command ...>

Reads ``nvidia-smi nvlink -gt d`` (per-link Data Tx / Rx counters, KiB) for
every GPU before and after the command and prints one JSON line with the
per-GPU byte deltas, so a copy-engine multicast (which ncu's kernel counters
cannot see) is measured the same way the in-kernel one is: bytes that crossed
NVLink per GPU vs the schedule's delivered bytes.
"""
import json
import re
import subprocess
import sys
import time


def snapshot() -> dict:
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


def main():
    cmd = sys.argv[sys.argv.index("--") + 1:] if "--" in sys.argv else sys.argv[1:]
    a = snapshot()
    t0 = time.time()
    rc = subprocess.run(cmd).returncode
    dt = time.time() - t0
    b = snapshot()
    delta = {g: {"tx_bytes": b[g]["tx"] - a[g]["tx"], "rx_bytes": b[g]["rx"] - a[g]["rx"]} for g in b if g in a}
    print(json.dumps({"nvlink_counters": delta, "command": " ".join(cmd), "rc": rc, "wall_s": round(dt, 2),
                      "source": "nvidia-smi nvlink -gt d (Data Tx/Rx KiB per link, summed per GPU)"}), flush=True)
    return rc


if __name__ == "__main__":
    sys.exit(main())
