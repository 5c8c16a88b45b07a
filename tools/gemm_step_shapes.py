"""Per-shape TFLOP/s of every GEMM launched by one Qwen2.5-1.5B SFT microbatch
(fwd + bwd) at N=1, timed live with CUDA events (gemm.Recorder). Shows which
GEMM shapes (residual epilogue, split-K, wave tail) are below the rest.

usage: python tools/gemm_step_shapes.py [tokens_per_sequence ...]
"""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200 import gemm as G  # noqa: E402
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
lens = [int(x) for x in sys.argv[1:]] or [8192, 6000, 3000, 1500]
b = W.make_batch(lens, list(range(len(lens))), S.vocab, dev, heads=S.heads, kv_heads=S.kv_heads)
wk.microbatch(b, 1.0)  # warm-up
torch.cuda.synchronize()
G.recorder = G.Recorder()
wk.microbatch(b, 1.0)
torch.cuda.synchronize()
rows = G.recorder.rows
G.recorder = None
agg = defaultdict(lambda: [0, 0.0, 0.0])
for fl, e0, e1, key in rows:
    a = agg[key]
    a[0] += 1
    a[1] += fl
    a[2] += e0.elapsed_time(e1)
tot_ms = sum(a[2] for a in agg.values())
print(f"{'M':>7} {'N':>7} {'K':>6} amn bmn f32 acc res  n   ms    share  TF/s")
for key, (n, fl, ms) in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    M, N, K, amn, bmn, f32, acc, res = key
    print(f"{M:7d} {N:7d} {K:6d}  {amn}   {bmn}   {int(f32)}   {int(acc)}   {int(res)} {n:3d} {ms:6.2f} {ms / tot_ms:6.3f} "
          f"{fl / ms / 1e9:6.0f}")
print(f"total {tot_ms:.2f} ms, {sum(a[1] for a in agg.values()) / tot_ms / 1e9:.0f} TF/s")
