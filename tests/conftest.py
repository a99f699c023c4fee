import os
import sys

# The copy-engine executor parks stream-ordered waits (cuStreamWaitValue32) on
# its streams; emulating many nodes on one GPU needs at least one hardware
# connection per stream, or a parked wait on a shared connection stalls
# unrelated streams (the driver default is 8).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / round-end GPU tier)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


def load_golden(name):
    import json
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]
    return get


def gpu_count():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0
