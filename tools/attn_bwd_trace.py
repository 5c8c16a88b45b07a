"""Per-iteration timeline of the transposed-score attention backward
(attn_bwd_t_kernel, specialised warpgroups) in CTA 0, from SM clock stamps recorded by the
ODC_ATTN_TRACE build (`python -m paper_2601_19362_b200.build --variant trace
ODC_ATTN_TRACE`). Prints each event's median offset (SM cycles) from the
iteration's dP^T issue, and the median iteration period.

usage: ODC_LIB_PATH=paper_2601_19362_b200/lib/variants/trace/libodc.so python tools/attn_bwd_trace.py
"""
import ctypes as C
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_19362_b200 import fused as F  # noqa: E402
from paper_2601_19362_b200._lib import lib  # noqa: E402

EV = ["mma:dP_issue", "mma:dV_issue(p_full)", "mma:S_next_issue(p_read)", "mma:dQ_issue(ds_full)",
      "mma:dK_issued", "A:start(s_full)", "A:end(p_full)", "B:start(dp_full,p_full)", "B:p_read",
      "B:end(ds_full)", "B:dQ_start(dq_full)", "B:dq_read", "B:sent_to_peer", "B:peer_half_added", "B:dQ_reduce_issued",
      "B:prev_dQ_drained"]
NI = 64

lens, H, KV = [int(x) for x in os.environ.get("LENS", "32768").split(",")], 12, 2
T = sum(lens)
q = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
k = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
v = torch.randn(T, KV, 128, device="cuda").to(torch.bfloat16)
do = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
sc = 128 ** -0.5
o, lse = F.attn_fwd(q, k, v, F.attn_items(lens, H, "cuda"), sc)
bi = F.attn_bwd_items(lens, H, KV, "cuda")
for _ in range(3):
    F.attn_bwd(q, k, v, o, do, lse, bi, sc)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (len(EV) * NI))()
assert lib().odc_attn_trace_read(buf) == 0
tr = [[buf[e * NI + n] for n in range(NI)] for e in range(len(EV))]
rows = []
for e, name in enumerate(EV):
    offs = [tr[e][n] - tr[0][n] for n in range(8, NI - 1) if tr[e][n] and tr[0][n]]
    rows.append((name, statistics.median(offs) if offs else None))
period = statistics.median(tr[0][n + 1] - tr[0][n] for n in range(8, NI - 1))
out = {"lens": lens, "period_clk": period, "events": {n: (round(x) if x is not None else None) for n, x in rows}}
print(json.dumps(out))
for name, x in rows:
    print(f"{name:28s} {x}")
