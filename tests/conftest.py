import json
import os
import sys

import pytest

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
