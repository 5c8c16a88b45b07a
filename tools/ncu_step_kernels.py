"""One ODC SFT minibatch for ncu captures of the step's own kernels at N=1:
the Qwen2.5-1.5B layer / embedding / LM-head shapes (2 decoder layers so the
backward comes within a short capture) on the bench's largest microbatch, a
single 32,768-token sequence: fetch, tcgen05 GEMMs (incl. the fused gate_up +
SwiGLU), attention fwd/bwd, the glue, push, barrier and AdamW.

Every GEMM launch's (M, N, K, kind) is written in launch order to
gpurun_out/ncu_gemm_launches.json so tools/ncu_traffic.py can attach shapes and
algorithmic FLOPs to the ncu rows.

usage: python tools/ncu_step_kernels.py [tokens]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_19362_b200 import gemm as G  # noqa: E402
from paper_2601_19362_b200 import worker as W  # noqa: E402
from paper_2601_19362_b200.engine import OdcEngine  # noqa: E402
from paper_2601_19362_b200.shapes import QWEN25_1_5B, Shape  # noqa: E402

S0 = QWEN25_1_5B
S = Shape(S0.name + "-L2", S0.d, S0.ffn, 2, S0.heads, S0.kv_heads, S0.vocab, S0.qkv_bias, S0.tied)
dev = torch.device("cuda", 0)
sizes = W.unit_sizes(S)
eng = OdcEngine(sizes)
gen = torch.Generator(device=dev).manual_seed(0)
for u in range(len(sizes)):
    eng.set_params(u, W.init_unit(S, u, gen, dev))
wk = W.Worker(S, W.OdcComm(eng), dev)
lens = [int(sys.argv[1])] if len(sys.argv) > 1 else [32768]
b = W.make_batch(lens, list(range(len(lens))), S.vocab, dev, heads=S.heads, kv_heads=S.kv_heads)
G.recorder = G.Recorder()
wk.microbatch(b, 1.0)
wk.minibatch_end()
torch.cuda.synchronize()
rows = [{"M": k[0], "N": k[1], "K": k[2], "flops": fl, "kind": k[-1] if k[-1] == "glu" else
         ("wgrad" if k[3] else ("fwd" if not k[4] else "dgrad"))} for fl, _, _, k in G.recorder.rows]
G.recorder = None
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/ncu_gemm_launches.json", "w") as f:
    json.dump(rows, f)
print("ok", len(rows), "gemm launches")
