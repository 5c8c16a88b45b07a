"""Times one SFT microbatch of a BASELINE model shape with fewer layers at N=1
(the per-layer cost does not depend on the layer count), phase by phase, so a
shape that is slow or hangs in the full bench can be isolated quickly.

usage: python tools/shape_probe.py MODEL LAYERS RECOMPUTE LEN[,LEN...]
"""
import dataclasses
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200 import shapes  # noqa: E402
from paper_2601_19362_b200 import worker as W  # noqa: E402
from paper_2601_19362_b200.engine import OdcEngine  # noqa: E402


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


name, layers, rc, lens = sys.argv[1], int(sys.argv[2]), sys.argv[3], [int(x) for x in sys.argv[4].split(",")]

if "--trace-calls" in sys.argv:  # synchronise after every libodc call and log it (finds a hanging kernel)
    from paper_2601_19362_b200 import _lib

    real = _lib.lib()

    class _Tracing:
        def __getattr__(self, n):
            fn = getattr(real, n)

            def call(*a):
                print(f"  -> {n}", flush=True)
                r = fn(*a)
                torch.cuda.synchronize()
                print(f"  <- {n} = {r}", flush=True)
                return r
            return call

    _lib._lib = _Tracing()
S = dataclasses.replace(shapes.SHAPES[name], layers=layers)
dev = torch.device("cuda", 0)
sizes = W.unit_sizes(S)
log("units", sizes)
eng = OdcEngine(sizes)
gen = torch.Generator(device=dev).manual_seed(0)
for u in range(len(sizes)):
    eng.set_params(u, W.init_unit(S, u, gen, dev))
torch.cuda.synchronize()
log("params set; arena GB", eng.arena_bytes() / 1e9)
wk = W.Worker(S, W.OdcComm(eng), dev, recompute=rc)
b = W.make_batch(lens, list(range(len(lens))), S.vocab, dev, heads=S.heads, kv_heads=S.kv_heads)
torch.cuda.synchronize()
log("batch built, tokens", b.tokens)
for it in range(3):
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    loss = wk.microbatch(b, 1.0)
    z.record()
    torch.cuda.synchronize()
    log(f"microbatch {it}: {a.elapsed_time(z):.1f} ms loss {loss.item():.4f} "
        f"peak mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB")
eng.minibatch_end()
eng.adam_step()
eng.check()
log("minibatch end + adam ok")
