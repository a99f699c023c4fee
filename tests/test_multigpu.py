"""Multi-GPU parity of the multicast engine, one process per GPU (torchrun,
NCCL rendezvous on 127.0.0.1): every executor and source tier delivers the
source's bytes to every rank.  Skipped on boxes with fewer than 2 GPUs."""
import json
import os
import subprocess
import sys

import pytest

from conftest import gpu_count

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(gpu_count() < 2, reason="needs >= 2 GPUs")
def test_distributed_multicast_all_executors():
    n = min(gpu_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + os.getpid() % 200),
           os.path.join(ROOT, "tools", "mc_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=280, cwd=ROOT)
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert res.returncode == 0 and line, res.stdout[-2000:] + res.stderr[-2000:]
    out = json.loads(line[-1])
    assert out["ok"] and len(out["results"]) == 5, out


@pytest.mark.skipif(gpu_count() < 3, reason="needs >= 3 GPUs for cross-device relays")
@pytest.mark.parametrize("executor", ["ce", "kernel"])
def test_single_process_relays(executor):
    """One process driving several GPUs (as serving and the autoscaler do)
    through a schedule whose relays wait on each other across devices: the
    copy-engine executor must not deadlock (it runs in the push direction in
    this mode) and every receiver ends byte-exact.  Run in a subprocess with
    a timeout, since a stream-level deadlock has no watchdog."""
    n = min(gpu_count(), 4)
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "relay_check.py"), str(n), "1", "4", executor],
                         capture_output=True, text=True, timeout=150, cwd=ROOT, env=env)
    assert res.returncode == 0 and "byte-exact" in res.stdout, res.stdout[-2000:] + res.stderr[-2000:]
