import json
import os
import sys

import pytest

# Several ODC ranks in ONE process (OdcEngine.local_group, config0) wait on one
# another's device flags from different streams. CUDA maps streams onto
# CUDA_DEVICE_MAX_CONNECTIONS hardware work queues (default 8); two ranks'
# streams sharing a queue serialise, so rank a's spinning barrier kernel would
# block rank b's kernels queued behind it. 32 queues give every stream these
# tests create its own. Must be set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# (the engine also force-loads its protocol kernels at context creation: a lazily loaded
# kernel's first launch can wait for running work, i.e. for a peer's spinning barrier)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) — run with -m gpu on the GPU box")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def have_gpus(n=1):
    try:
        import torch

        return torch.cuda.is_available() and torch.cuda.device_count() >= n
    except Exception:
        return False
