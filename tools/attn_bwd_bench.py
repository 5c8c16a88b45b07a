"""tcgen05 attention backward vs flash-attn 2.8 backward: time and TFLOP/s."""
import json
import sys

import torch

sys.path.insert(0, ".")
from flash_attn.flash_attn_interface import _flash_attn_varlen_backward  # noqa: E402

from paper_2601_19362_b200 import fused as F  # noqa: E402

H, KV = 12, 2
for lens in ([32768], [8192, 6000, 4000, 3000, 2000, 1024, 512, 512], [2048] * 16):
    T = sum(lens)
    q = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
    k = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
    do = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device="cuda")
    sc = 128 ** -0.5
    o, lse = F.attn_fwd(q, k, v, F.attn_items(lens, H, "cuda"), sc)
    bi = F.attn_bwd_items(lens, H, KV, "cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    res = {"lens": lens[:3], "T": T}
    fl = sum(2 * 2 * s * s / 2 * 128 * H for s in lens) * 2.5
    for name, fn in (("ours", lambda: F.attn_bwd(q, k, v, o, do, lse, bi, sc)),
                     ("fa2", lambda: _flash_attn_varlen_backward(do, q, k, v, o, lse, dq, dk, dv, cu, cu, max(lens),
                                                                 max(lens), 0.0, sc, True, -1, -1, 0.0, None, False))):
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
        res[name + "_tflops"] = round(fl / ms / 1e9, 1)
    print(json.dumps(res), flush=True)
