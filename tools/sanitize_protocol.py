"""Small driver of every ODC protocol kernel for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

  compute-sanitizer --tool memcheck python tools/sanitize_protocol.py

world = 1 engines in RED / SLOT / FIXED mode over ragged units (a tail shard,
a unit smaller than a vector, a bulk-path unit): set_params, fetch (TMA and
LDG engines), push (fp32 and bf16 gradients), push_slice, the minibatch
barrier, AdamW, and the reference-semantics fabric (stage / consume /
finalize). The sanitizer serialises kernels, so ranks that wait on each other
cannot run under it; with one rank every gate is already open and every
kernel's memory accesses are still checked.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_19362_b200.engine import OdcEngine  # noqa: E402
from paper_2601_19362_b200.primitives import ShardFabric  # noqa: E402

dev = "cuda:0"
sizes = [4099, 5, (1 << 20) + 17]
for mode in ("red", "slot", "fixed"):
    for engine in ("tma", "ldg"):
        eng = OdcEngine(sizes, push_mode=mode, fetch_engine=engine, timeout_s=120)
        for l, n in enumerate(sizes):
            eng.set_params(l, torch.randn(n, device=dev))
        for mb in range(2):
            for l, n in enumerate(sizes):
                out = torch.empty(n, dtype=torch.bfloat16, device=dev)
                eng.fetch(l, out)
                eng.push(l, torch.randn(n, device=dev), 0.5)
                eng.push(l, torch.randn(n, device=dev).to(torch.bfloat16), 0.25)
                if n > 3:
                    eng.push_slice(l, 0, 1, torch.randn(min(n - 1, 100), device=dev), 0.5)
            eng.minibatch_end()
            for l in range(len(sizes)):
                eng.read_grad_shard(l)
            eng.adam_step(lr=1e-3)
        eng.check()
        eng.close()
        print("engine ok", mode, engine, flush=True)
for dt in (np.int64, np.float32):
    f = ShardFabric(4, 1001, dt)
    f.set_params("w", np.arange(1001).astype(dt))
    f.gather(1, "w")
    for c in (0, 3, 0, 2):
        f.scatter_accumulate(c, np.ones(1001, dt), dt(2))
    f.push_slice(1, 2, 3, np.ones(10, dt), dt(1))
    f.finalize_minibatch()
    print("fabric ok", np.dtype(dt).name, flush=True)
torch.cuda.synchronize()
print("sanitize driver done")
