"""TFLOP/s of the tcgen05 GEMM vs torch.matmul (cuBLAS) on the Qwen2.5-1.5B
layer shapes at T tokens (fwd / dgrad / wgrad)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200 import gemm as G  # noqa: E402


def bench(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
for name, inn, out in [("qkv", 1536, 2048), ("o", 1536, 1536), ("gate_up", 1536, 17920), ("down", 8960, 1536)]:
    x = torch.randn(T, inn, device="cuda").to(torch.bfloat16)
    w = torch.randn(out, inn, device="cuda").to(torch.bfloat16)
    dy = torch.randn(T, out, device="cuda").to(torch.bfloat16)
    fl = 2 * T * inn * out
    r = {"shape": name, "T": T, "in": inn, "out": out}
    for k, ours, ref in [("fwd", lambda: G.linear_fwd(x, w), lambda: x @ w.t()),
                         ("dgrad", lambda: G.linear_dgrad(dy, w), lambda: dy @ w),
                         ("wgrad", lambda: G.linear_wgrad(dy, x), lambda: dy.t().float() @ x.float() if False else torch.matmul(dy.t(), x))]:
        r[k] = round(fl / bench(ours) / 1e9, 1)
        r[k + "_cublas"] = round(fl / bench(ref) / 1e9, 1)
    print(json.dumps(r), flush=True)
