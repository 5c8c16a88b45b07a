"""One RED push and one FIXED push (+ its finalize) of a Qwen2.5-1.5B layer
unit at N=1 (for ncu captures of push_red_kernel / push_fixed_kernel /
fixed_finalize_kernel); with --time, CUDA-event times of 20 pushes per mode."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200.engine import OdcEngine  # noqa: E402

M = 46_797_824
g = torch.randn(M, device="cuda") * 1e-3
for mode in ("red", "fixed"):
    eng = OdcEngine([M], push_mode=mode)
    eng.set_params(0, torch.zeros(M, device="cuda"))
    for _ in range(2):
        eng.push(0, g, 0.5)
    if "--time" in sys.argv:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            eng.push(0, g, 0.5)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        wire = 8 if mode == "fixed" else 4
        print(f"{mode}: {us:.1f} us per push, {M * (4 + 2 * wire) / us / 1e3:.0f} GB/s (read g + RMW shard)")
    eng.minibatch_end()
    eng.check()
    eng.close()
torch.cuda.synchronize()
print("ok")
