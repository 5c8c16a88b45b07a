"""Host-side multi-rank plumbing of the ODC path (torch.distributed, any
backend): the one-time IPC blob exchange and the max-over-ranks timing
reduction of the bench. Testable on CPU with gloo (tests/test_dist_gloo.py)."""
from __future__ import annotations

from typing import List, Sequence


def exchange_blobs(blob: bytes, group=None) -> List[bytes]:
    """All-gather one opaque byte blob per rank (the 64-byte odc_ctx_export
    payloads); returns them in rank order."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return [bytes(b) for b in out]


def rank_timings(ms: float, busy_ms: float, launches: int, device=None, group=None):
    """Gathers (ms, busy, launches) from every rank. Returns (max ms over
    ranks, idle fraction 1 - sum(busy)/(N * max ms) [src/runtime.cpp:43],
    total launches, per-rank rows)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([ms, busy_ms, float(launches)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        rows = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(rows, t, group=group)
        rows = torch.stack(rows).cpu()
    else:
        rows = t[None].cpu()
    mx = rows[:, 0].max().item()
    idle = 1.0 - rows[:, 1].sum().item() / (rows.shape[0] * mx) if mx > 0 else 0.0
    return mx, idle, int(rows[:, 2].sum().item()), rows.tolist()


def plan_digest(plan: Sequence) -> str:
    import hashlib
    import json

    return hashlib.sha256(json.dumps(plan, separators=(",", ":")).encode()).hexdigest()
