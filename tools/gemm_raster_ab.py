"""Interleaved A/B of the GEMM tile raster on the bench's large GEMM shapes
(Qwen2.5-1.5B layer at T = 32,768 and the LM-head chunk): for every shape and
op, the variants are timed in turn (CUDA events) for several rounds inside ONE
process, so clock / power drift hits every variant alike; the median per
variant is printed as one JSON line per (shape, op).

Variants: group8 (the round-1 fixed raster), auto40 / auto80 (csrc/gemm.cu
raster_group with a 40 / 80 MB L2 budget), rowmajor (group 1: B reused from L2).

usage: python tools/gemm_raster_ab.py [rounds] [reps]
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_19362_b200 import gemm as G  # noqa: E402
from paper_2601_19362_b200._lib import check, lib  # noqa: E402

dev = torch.device("cuda", 0)
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
T = 32768
SHAPES = [("qkv", T, 1536, 2048), ("o", T, 1536, 1536), ("gate_up", T, 1536, 17920), ("down", T, 8960, 1536),
          ("lm_head", 8192, 1536, 151936)]
VARIANTS = {"group8": (8, 40), "auto40": (0, 40), "auto80": (0, 80), "rowmajor": (1, 40)}


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
        times = {v: [] for v in VARIANTS}
        for _ in range(rounds):
            for v, (grp, mb) in VARIANTS.items():
                check(lib().odc_gemm_set_raster(grp, mb))
                fn()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    fn()
                b.record()
                torch.cuda.synchronize()
                times[v].append(a.elapsed_time(b) / reps)
        fl = 2.0 * rows * inn * out
        row = {"shape": name, "op": op}
        for v, ts in times.items():
            ms = statistics.median(ts)
            row[v] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)}
        print(json.dumps(row), flush=True)
    del x, w, dy, y, dx, dw
    torch.cuda.empty_cache()
check(lib().odc_gemm_set_raster(0, 40))
