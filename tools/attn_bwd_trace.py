"""Per-iteration timeline of the attention backward (attn_bwd_kernel) in CTA 0, from SM clock stamps recorded by the
ODC_ATTN_TRACE build (`python -m paper_2601_19362_b200.build --variant trace
ODC_ATTN_TRACE`). Prints each event's median offset (SM cycles) from the
iteration's dP issue, and the median iteration period.

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

EV = ["mma:dP_issue", "mma:S_next_issue(s_read)", "mma:dV_issue(p_full)", "mma:dQ_issue(ds_full)", "mma:dK_issued",
      "wg0:sdp_full", "wg0:P_drain_wait_start", "wg0:P_drain_wait_end", "wg0:p_full", "wg0:ds_full", "wg0:dq_full",
      "wg0:stage_start", "wg0:reduce_issued", "wg1:sdp_full", "wg1:p_full", "wg1:dS_drain_wait_start",
      "wg1:dS_drain_wait_end", "wg1:ds_full", "wg1:dq_full", "wg1:dk_done(stage_start)", "wg1:reduce_issued"]
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
