"""One SFT microbatch of the Qwen2.5-1.5B worker at N=1 (for ncu captures of
the step's own kernels: gemm_kernel, attn_fwd/bwd, fetch, push, adam)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200 import partition as P  # noqa: E402
from paper_2601_19362_b200 import worker as W  # noqa: E402
from paper_2601_19362_b200.engine import OdcEngine  # noqa: E402
from paper_2601_19362_b200.shapes import QWEN25_1_5B as S  # noqa: E402

dev = torch.device("cuda", 0)
sizes = W.unit_sizes(S)
eng = OdcEngine(sizes)
gen = torch.Generator(device=dev).manual_seed(0)
for u in range(len(sizes)):
    eng.set_params(u, W.init_unit(S, u, gen, dev))
wk = W.Worker(S, W.OdcComm(eng), dev)
lens = [8192, 6000, 3000, 1500]
b = W.make_batch(lens, [0, 1, 2, 3], S.vocab, dev, heads=S.heads, kv_heads=S.kv_heads)
wk.microbatch(b, 1.0)
wk.minibatch_end()
torch.cuda.synchronize()
print("ok")
