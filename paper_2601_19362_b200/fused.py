"""ctypes wrappers of the worker's fused sm_100a elementwise kernels
(csrc/worker_kernels.cu). bf16 activations, fp32 statistics/gradients."""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import check, lib


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def rmsnorm_fwd(x, w, eps=1e-6):
    T, d = x.shape
    y = torch.empty_like(x)
    rstd = torch.empty(T, dtype=torch.float32, device=x.device)
    check(lib().odc_w_rmsnorm_fwd(_p(x), _p(w), _p(y), _p(rstd), T, d, eps, _s()))
    return y, rstd


def rmsnorm_bwd(dy, x, w, rstd, dw_accum, resid=None):
    """returns resid + dx (bf16); dw_accum (fp32 [d]) += sum_rows dy * xhat."""
    T, d = x.shape
    out = torch.empty_like(x)
    check(lib().odc_w_rmsnorm_bwd(_p(dy), _p(x), _p(w), _p(rstd), _p(resid), _p(out), _p(dw_accum), T, d, _s()))
    return out


def rope_table(max_pos, head_dim, theta, device):
    inv = 1.0 / (theta ** (torch.arange(0, head_dim, 2, dtype=torch.float64) / head_dim))
    ang = torch.arange(max_pos, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.stack([torch.cos(ang), torch.sin(ang)], -1).float().contiguous().to(device)  # [P, hd/2, 2]


def qkv_rope_fwd(qkv, bias, table, pos, H, KV, hd):
    T = qkv.shape[0]
    q = torch.empty(T, H, hd, dtype=torch.bfloat16, device=qkv.device)
    k = torch.empty(T, KV, hd, dtype=torch.bfloat16, device=qkv.device)
    v = torch.empty(T, KV, hd, dtype=torch.bfloat16, device=qkv.device)
    check(lib().odc_w_qkv_rope_fwd(_p(qkv), _p(bias), _p(table), _p(pos), _p(q), _p(k), _p(v), T, H, KV, hd, _s()))
    return q, k, v


def qkv_rope_bwd(dq, dk, dv, table, pos, H, KV, hd):
    T = dq.shape[0]
    out = torch.empty(T, (H + 2 * KV) * hd, dtype=torch.bfloat16, device=dq.device)
    check(lib().odc_w_qkv_rope_bwd(_p(dq), _p(dk), _p(dv), _p(table), _p(pos), _p(out), T, H, KV, hd, _s()))
    return out


def col_sum_(m, out):
    T, n = m.shape
    check(lib().odc_w_col_sum(_p(m), _p(out), T, n, _s()))
    return out


def swiglu_fwd(gu, ffn):
    T = gu.shape[0]
    m = torch.empty(T, ffn, dtype=torch.bfloat16, device=gu.device)
    check(lib().odc_w_swiglu_fwd(_p(gu), _p(m), T, ffn, _s()))
    return m


def swiglu_bwd(dm, gu, ffn):
    T = gu.shape[0]
    dgu = torch.empty_like(gu)
    check(lib().odc_w_swiglu_bwd(_p(dm), _p(gu), _p(dgu), T, ffn, _s()))
    return dgu


def ce_fwd_bwd_(logits, labels, scale, loss_accum):
    rows, V = logits.shape
    check(lib().odc_w_ce_fwd_bwd(_p(logits), _p(labels), rows, V, float(scale), _p(loss_accum), _s()))
    return logits


def attn_items(lens, H: int, device) -> torch.Tensor:
    """Work list of the tcgen05 attention forward: one item per (sequence,
    256-query tile = two 128-row tiles, head), heaviest (most causal KV tiles)
    first."""
    items, start = [], 0
    for n in lens:
        for qt in range((n + 255) // 256):
            for h in range(H):
                items.append((start, n, qt, h))
        start += n
    items.sort(key=lambda t: -t[2])
    t = torch.tensor(items, dtype=torch.int32)
    return (t.pin_memory() if torch.device(device).type == "cuda" else t).to(device, non_blocking=True)


def attn_fwd(q, k, v, items, scale):
    """causal varlen attention, q [T,H,128], k/v [T,KV,128] -> out [T,H,128], lse [H,T]."""
    T, H, hd = q.shape
    KV = k.shape[1]
    out = torch.empty_like(q)
    lse = torch.empty(H, T, dtype=torch.float32, device=q.device)
    check(lib().odc_attn_fwd(_p(q), _p(k), _p(v), _p(out), _p(lse), _p(items), items.shape[0], T, H, KV, hd,
                             float(scale), _s()))
    return out, lse


def attn_bwd_items(lens, H: int, KV: int, device, sms: int = 148) -> torch.Tensor:
    """Backward work list: per (sequence, 128-key tile, kv head) the causal loop
    over (query head of the GQA group, query tile >= key tile). Loops longer
    than ~1/(2*SMs) of the total are cut into chunks (their dK/dV partials meet
    in fp32 accumulators) so the grid load-balances; largest first (LPT)."""
    G = H // KV
    loops, start = [], 0
    for n in lens:
        nt = (n + 127) // 128
        for kt in range(nt):
            loops.append((start, n, kt, G * (nt - kt)))
        start += n
    total = sum(t for *_, t in loops) * KV
    chunk = max(32, -(-total // (2 * sms)))
    items = []
    for st, n, kt, t in loops:
        pieces = -(-t // chunk)
        for pc in range(pieces):
            b, e = t * pc // pieces, t * (pc + 1) // pieces
            for h in range(KV):
                items.append((st, n, kt, h, b, e, 0, 0))
    items.sort(key=lambda x: x[4] - x[5])
    t = torch.tensor(items, dtype=torch.int32)
    return (t.pin_memory() if torch.device(device).type == "cuda" else t).to(device, non_blocking=True)


def attn_bwd(q, k, v, o, dout, lse, items, scale):
    T, H, hd = q.shape
    KV = k.shape[1]
    dq = torch.empty_like(q)
    dk = torch.empty_like(k)
    dv = torch.empty_like(v)
    ws = torch.empty((H * T + 63) // 64 * 64 + T * H * hd + 2 * T * KV * hd, dtype=torch.float32, device=q.device)
    check(lib().odc_attn_bwd(_p(q), _p(k), _p(v), _p(o), _p(dout), _p(lse), _p(dq), _p(dk), _p(dv), _p(ws),
                             _p(items), items.shape[0], T, H, KV, hd, float(scale), _s()))
    return dq, dk, dv


def attn_bwd_qkv(q, k, v, o, dout, lse, items, scale, table, pos):
    """The attention backward straight to the packed qkv gradient [T, (H+2KV)*hd]
    with the inverse RoPE applied (= attn_bwd + qkv_rope_bwd, bit-identical)."""
    T, H, hd = q.shape
    KV = k.shape[1]
    dqkv = torch.empty(T, (H + 2 * KV) * hd, dtype=torch.bfloat16, device=q.device)
    ws = torch.empty((H * T + 63) // 64 * 64 + T * H * hd + 2 * T * KV * hd, dtype=torch.float32, device=q.device)
    check(lib().odc_attn_bwd_qkv(_p(q), _p(k), _p(v), _p(o), _p(dout), _p(lse), _p(table), _p(pos), _p(dqkv), _p(ws),
                                 _p(items), items.shape[0], T, H, KV, hd, float(scale), _s()))
    return dqkv
