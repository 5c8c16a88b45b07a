"""flash-attn 2.8 varlen vs cuDNN (torch aten._cudnn_attention_*) varlen on
B200: fwd+bwd time and agreement, causal, GQA 12/2, hd 128."""
import json
import sys

import torch

sys.path.insert(0, ".")
from flash_attn.flash_attn_interface import _flash_attn_varlen_backward, _flash_attn_varlen_forward  # noqa

torch.manual_seed(0)
dev = "cuda"
H, KV, hd = 12, 2, 128
for lens in ([32768], [8192, 6000, 4000, 3000, 2000, 1024, 512, 512], [2048] * 16):
    T = sum(lens)
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device=dev)
    mx = max(lens)
    q = torch.randn(T, H, hd, device=dev, dtype=torch.bfloat16)
    k = torch.randn(T, KV, hd, device=dev, dtype=torch.bfloat16)
    v = torch.randn(T, KV, hd, device=dev, dtype=torch.bfloat16)
    do = torch.randn(T, H, hd, device=dev, dtype=torch.bfloat16)
    sc = hd ** -0.5

    def fa2():
        o, lse, _, _ = _flash_attn_varlen_forward(q, k, v, cu, cu, mx, mx, 0.0, sc, True)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        _flash_attn_varlen_backward(do, q, k, v, o, lse, dq, dk, dv, cu, cu, mx, mx, 0.0, sc, True, -1, -1, 0.0,
                                    None, False)
        return o, dq, dk, dv

    def cudnn():
        r = torch.ops.aten._cudnn_attention_forward(q, k, v, None, cu, cu, mx, mx, True, 0.0, True, False, scale=sc)
        o, lse = r[0], r[1]
        dq, dk, dv = torch.ops.aten._cudnn_attention_backward(do, q, k, v, o, lse, r[6], r[7], None,
                                                              cu, cu, mx, mx, 0.0, True, scale=sc)
        return o, dq, dk, dv

    res = {"lens": lens[:4], "T": T}
    outs = {}
    for name, fn in (("fa2", fa2), ("cudnn", cudnn)):
        try:
            outs[name] = fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                fn()
            b.record()
            torch.cuda.synchronize()
            res[name + "_ms"] = round(a.elapsed_time(b) / 5, 3)
        except Exception as e:
            res[name + "_err"] = str(e)[:200]
    if "fa2" in outs and "cudnn" in outs:
        res["max_abs_diff"] = [round((x.float() - y.float()).abs().max().item(), 4) for x, y in zip(outs["fa2"], outs["cudnn"])]
    fl = sum(4 * s * s / 2 * hd * H for s in lens) * 3.5  # fwd (2 matmuls, causal) + bwd (2.5x)
    for n in ("fa2", "cudnn"):
        if n + "_ms" in res:
            res[n + "_tflops"] = round(fl / res[n + "_ms"] / 1e9, 1)
    print(json.dumps(res), flush=True)
