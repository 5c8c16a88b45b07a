"""Standalone timing of the worker's fused glue kernels at one microbatch size
(CUDA events), with achieved HBM GB/s for each."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200 import fused as F  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 19000
d, ffn = 1536, 8960


def bench(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def bf(*s):
    return torch.randn(*s, device="cuda").to(torch.bfloat16)


x, w, dy, res = bf(T, d), bf(d), bf(T, d), bf(T, d)
y, rstd = F.rmsnorm_fwd(x, w)
dw = torch.zeros(d, device="cuda")
gu, dm = bf(T, 2 * ffn), bf(T, ffn)
rows = [
    ("rmsnorm_fwd", lambda: F.rmsnorm_fwd(x, w), 2 * T * d * 2),
    ("rmsnorm_bwd", lambda: F.rmsnorm_bwd(dy, x, w, rstd, dw, resid=res), 4 * T * d * 2),
    ("swiglu_fwd", lambda: F.swiglu_fwd(gu, ffn), 3 * T * ffn * 2),
    ("swiglu_bwd", lambda: F.swiglu_bwd(dm, gu, ffn), 5 * T * ffn * 2),
]
for name, fn, nbytes in rows:
    ms = bench(fn)
    print(json.dumps({"kernel": name, "T": T, "us": round(ms * 1e3, 1), "GBps": round(nbytes / ms / 1e6, 1)}))
