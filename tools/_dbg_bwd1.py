import sys, torch
sys.path.insert(0, ".")
from paper_2601_19362_b200 import fused as F
lens=[128]; H, KV = 2, 1
T=sum(lens)
q = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
k = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
v = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
do = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
o, lse = F.attn_fwd(q, k, v, F.attn_items(lens, H, "cuda"), 128**-0.5)
torch.cuda.synchronize(); print("fwd ok", flush=True)
bi = F.attn_bwd_items(lens, H, KV, "cuda")
print(bi.cpu().tolist(), flush=True)
F.attn_bwd(q, k, v, o, do, lse, bi, 128**-0.5)
torch.cuda.synchronize(); print("bwd ok")
