"""Times the bench's large GEMM shapes (Qwen2.5-1.5B layer at T = 32,768 and
the LM-head chunk) with CUDA events, one JSON line per shape: the A/B tool
for the tile raster (ODC_GEMM_GROUP=8 = the round-1 fixed group; unset = the
L2-budget raster of csrc/gemm.cu raster_group). Run under ncu with
--metrics dram__bytes_read.sum,dram__bytes_write.sum for the traffic side.

usage: python tools/gemm_raster_ab.py [reps]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_19362_b200 import gemm as G  # noqa: E402

dev = torch.device("cuda", 0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
T = 32768
SHAPES = [("qkv", T, 1536, 2048), ("o", T, 1536, 1536), ("gate_up", T, 1536, 17920), ("down", T, 8960, 1536),
          ("lm_head", 8192, 1536, 151936)]


def r(*s):
    return (torch.randn(*s, device=dev) * 0.1).to(torch.bfloat16)


for name, rows, inn, out in SHAPES:
    x, w, dy = r(rows, inn), r(out, inn), r(rows, out)
    y = torch.empty(rows, out, dtype=torch.bfloat16, device=dev)
    dx = torch.empty(rows, inn, dtype=torch.bfloat16, device=dev)
    dw = torch.empty(out, inn, dtype=torch.float32, device=dev)
    ops = {"fwd": lambda: G.linear_fwd(x, w, out=y), "dgrad": lambda: G.linear_dgrad(dy, w, out=dx),
           "wgrad": lambda: G.linear_wgrad(dy, x, out=dw)}
    for op, fn in ops.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        fl = 2.0 * rows * inn * out
        print(json.dumps({"shape": name, "op": op, "M_N_K": {"fwd": [rows, out, inn], "dgrad": [rows, inn, out],
                                                             "wgrad": [out, inn, rows]}[op],
                          "group_env": os.environ.get("ODC_GEMM_GROUP", "auto"), "ms": round(ms, 4),
                          "tflops": round(fl / ms / 1e9, 1)}), flush=True)
    del x, w, dy, y, dx, dw
    torch.cuda.empty_cache()
