"""Calibrates the load balancer's cost model on B200: times one SFT microbatch
(forward + backward, ODC engine at N=1, CUDA events) for several sequence-length
mixes and least-squares fits   t = alpha * sum(s^2) + beta * sum(s) + c
(the reference's per-sample cost alpha*s^2 + beta*s, src/cost_model.cpp:14-18,
plus a per-microbatch constant). Prints beta/alpha, the one knob that shapes
LB-Mini / LB-Micro plans (shapes.Shape.beta_over_alpha_b200).

usage: python tools/calibrate_cost.py [model]   (default qwen2.5-1.5b)
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200 import shapes  # noqa: E402
from paper_2601_19362_b200 import worker as W  # noqa: E402
from paper_2601_19362_b200.engine import OdcEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-1.5b"
S = shapes.SHAPES[name]
dev = torch.device("cuda", 0)
sizes = W.unit_sizes(S)
eng = OdcEngine(sizes)
gen = torch.Generator(device=dev).manual_seed(0)
for u in range(len(sizes)):
    eng.set_params(u, W.init_unit(S, u, gen, dev))
wk = W.Worker(S, W.OdcComm(eng), dev, cache_params=True)

mixes = [[512] * 32, [1024] * 16, [2048] * 8, [4096] * 4, [8192] * 2, [16384], [32768],
         [512] * 8, [2048] * 2, [4096], [8192], [16384, 512, 512], [6000, 3000, 1500, 700],
         [24000, 2000], [12000, 12000]]
rows = []
for lens in mixes:
    b = W.make_batch(lens, list(range(len(lens))), S.vocab, dev, heads=S.heads, kv_heads=S.kv_heads)
    wk.microbatch(b, 1.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        wk.microbatch(b, 1.0)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = float(np.median(ts))
    rows.append((sum(s * s for s in lens), sum(lens), t))
    print(json.dumps({"lens": lens[:4], "n": len(lens), "tokens": sum(lens), "ms": round(t, 3)}), flush=True)
A = np.array([[q, s, 1.0] for q, s, _ in rows])
y = np.array([t for _, _, t in rows])
(alpha, beta, c), *_ = np.linalg.lstsq(A, y, rcond=None)
pred = A @ np.array([alpha, beta, c])
print(json.dumps({"model": name, "alpha_ms_per_s2": alpha, "beta_ms_per_token": beta, "c_ms": c,
                  "beta_over_alpha": beta / alpha, "max_rel_residual": float(np.max(np.abs(pred - y) / y)),
                  "flop_beta_over_alpha": S.beta_over_alpha()}))
