"""One call each of the tcgen05 attention fwd and bwd (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200 import fused as F  # noqa: E402

lens = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192").split(",")]
H, KV = 12, 2
T = sum(lens)
q = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
k = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
v = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
do = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
sc = 128 ** -0.5
for _ in range(2):
    o, lse = F.attn_fwd(q, k, v, F.attn_items(lens, H, "cuda"), sc)
    F.attn_bwd(q, k, v, o, do, lse, F.attn_bwd_items(lens, H, KV, "cuda"), sc)
torch.cuda.synchronize()
print("ok")
