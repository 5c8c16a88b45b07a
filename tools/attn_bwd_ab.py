"""tcgen05 attention backward timing (CUDA events, 5 reps after a warm-up) on
the verdict's shapes: one 32K sequence and 16 x 2K at H/KV 12/2, one 64K at
40/8. One JSON line per case (A/B of kernel variants: build them with
`python -m paper_2601_19362_b200.build --variant NAME DEFINE` and select with
ODC_LIB_PATH; the label comes from ODC_ATTN_BWD).

usage: python tools/attn_bwd_ab.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_19362_b200 import fused as F  # noqa: E402

for lens, H, KV in (([32768], 12, 2), ([2048] * 16, 12, 2), ([8192, 6000, 4000, 3000, 2000, 1024, 512, 512], 12, 2),
                    ([65536], 40, 8)):
    T = sum(lens)
    q = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
    k = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
    do = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
    sc = 128 ** -0.5
    o, lse = F.attn_fwd(q, k, v, F.attn_items(lens, H, "cuda"), sc)
    bi = F.attn_bwd_items(lens, H, KV, "cuda")
    fl = sum(2 * 2 * s * s / 2 * 128 * H for s in lens) * 2.5  # 5 causal matmuls of the backward
    res = {"lens": lens[:3] + (["..."] if len(lens) > 3 else []), "n_seq": len(lens), "T": T, "H": H, "KV": KV,
           "variant": os.environ.get("ODC_ATTN_BWD", "shipped")}
    for name, fn in (("bwd", lambda: F.attn_bwd(q, k, v, o, do, lse, bi, sc)),
                     ("fwd", lambda: F.attn_fwd(q, k, v, F.attn_items(lens, H, "cuda"), sc))):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        res[name + "_ms"] = round(ms, 3)
        res[name + "_tflops"] = round((fl if name == "bwd" else fl / 2.5) / ms / 1e9, 1)
    print(json.dumps(res), flush=True)
    del q, k, v, do, o, lse
    torch.cuda.empty_cache()
