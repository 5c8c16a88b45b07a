"""fp32 torch references that scale to the benchmarked configuration (test
infrastructure): causal varlen attention chunked over query blocks (never a
full [n, n] score matrix, so 32K/64K-token sequences fit), and the SFT
decoder's loss with that attention and a chunked, recomputed LM head + CE (the
[T, 151,936] fp32 logits are never all alive at once).

Everything runs in fp32 with TF32 disabled; the kernels under test compute in
bf16 with fp32 accumulation, so the tests compare with norm-wise tolerances.
"""
from __future__ import annotations

import torch
import torch.nn.functional as TF
from torch.utils.checkpoint import checkpoint

from paper_2601_19362_b200 import worker as W

QCHUNK = 512


def _blocks(lens):
    s0 = 0
    for n in lens:
        yield s0, n
        s0 += n


@torch.no_grad()
def attn_fwd_ref(q, k, v, lens, scale):
    """q [T,H,D], k/v [T,KV,D] (any float dtype, computed in fp32) ->
    o [T,H,D] fp32, lse [H,T] fp32 (natural log), causal per sequence."""
    T, H, D = q.shape
    KV = k.shape[1]
    G = H // KV
    o = torch.empty(T, H, D, device=q.device)
    lse = torch.empty(H, T, device=q.device)
    for s0, n in _blocks(lens):
        for kh in range(KV):
            ks = k[s0:s0 + n, kh].float()
            vs = v[s0:s0 + n, kh].float()
            for qb in range(0, n, QCHUNK):
                c = min(QCHUNK, n - qb)
                kend = qb + c
                qs = q[s0 + qb:s0 + kend, kh * G:(kh + 1) * G].float().transpose(0, 1)  # [G, c, D]
                S = torch.matmul(qs, ks[:kend].t()) * scale  # [G, c, kend]
                S[:, :, qb:].masked_fill_(torch.triu(torch.ones(c, c, dtype=torch.bool, device=q.device), 1),
                                          float("-inf"))
                l = torch.logsumexp(S, -1)  # [G, c]
                P = torch.exp(S - l[..., None])
                o[s0 + qb:s0 + kend, kh * G:(kh + 1) * G] = torch.matmul(P, vs[:kend]).transpose(0, 1)
                lse[kh * G:(kh + 1) * G, s0 + qb:s0 + kend] = l
    return o, lse


@torch.no_grad()
def attn_bwd_ref(q, k, v, o, do, lse, lens, scale):
    """Gradients of attn_fwd_ref (flash-attention backward algebra, fp32)."""
    T, H, D = q.shape
    KV = k.shape[1]
    G = H // KV
    dq = torch.zeros(T, H, D, device=q.device)
    dk = torch.zeros(T, KV, D, device=q.device)
    dv = torch.zeros(T, KV, D, device=q.device)
    Dsum = (do.float() * o.float()).sum(-1)  # [T, H]
    for s0, n in _blocks(lens):
        for kh in range(KV):
            ks = k[s0:s0 + n, kh].float()
            vs = v[s0:s0 + n, kh].float()
            dks = dk[s0:s0 + n, kh]
            dvs = dv[s0:s0 + n, kh]
            for qb in range(0, n, QCHUNK):
                c = min(QCHUNK, n - qb)
                kend = qb + c
                sl = slice(s0 + qb, s0 + kend)
                hs = slice(kh * G, (kh + 1) * G)
                qs = q[sl, hs].float().transpose(0, 1)  # [G, c, D]
                dos = do[sl, hs].float().transpose(0, 1)
                S = torch.matmul(qs, ks[:kend].t()) * scale
                S[:, :, qb:].masked_fill_(torch.triu(torch.ones(c, c, dtype=torch.bool, device=q.device), 1),
                                          float("-inf"))
                P = torch.exp(S - lse[hs, sl][..., None])
                dP = torch.matmul(dos, vs[:kend].t())
                dS = P * (dP - Dsum[sl, hs].t()[..., None])
                dq[sl, hs] = (torch.matmul(dS, ks[:kend]) * scale).transpose(0, 1)
                dks[:kend] += torch.einsum("gck,gcd->kd", dS, qs) * scale
                dvs[:kend] += torch.einsum("gck,gcd->kd", P, dos)
    return dq, dk, dv


class ChunkedAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, lens, scale):
        o, lse = attn_fwd_ref(q, k, v, lens, scale)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.lens, ctx.scale = lens, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        dq, dk, dv = attn_bwd_ref(q, k, v, o, do, lse, ctx.lens, ctx.scale)
        return dq, dk, dv, None, None


def _rms(x, w):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + W.EPS) * w


def _ce_chunk(hf, head, labels):
    logits = hf @ head.t()
    return TF.cross_entropy(logits, labels, ignore_index=-100, reduction="sum")


def ref_loss(shape, units, batch, ce_chunk=4096):
    """fp32 loss of the worker's decoder (same layouts, RoPE, GQA, tied/untied
    head) on `batch`; gradients flow into `units` (fp32 leaf tensors)."""
    s = shape
    E = W.views(units[0], W.embed_layout(s))
    T = batch.tokens
    h = E["emb"][batch.ids]
    cos, sin = W.rope_tables(batch.positions, s.head_dim)
    cu = batch.cu_seqlens.tolist()
    lens = [cu[i + 1] - cu[i] for i in range(len(cu) - 1)]

    def rope(x):
        hh = x.shape[-1] // 2
        x1, x2 = x[..., :hh], x[..., hh:]
        c, sn = cos[:, None], sin[:, None]
        return torch.cat([x1 * c - x2 * sn, x2 * c + x1 * sn], -1)

    hd, H, KV = s.head_dim, s.heads, s.kv_heads
    for l in range(1, s.layers + 1):
        P = W.views(units[l], W.layer_layout(s))
        a = _rms(h, P["ln1"])
        qkv = a @ P["qkv_w"].t()
        if s.qkv_bias:
            qkv = qkv + P["qkv_b"]
        q = rope(qkv[:, :H * hd].view(T, H, hd))
        k = rope(qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd))
        v = qkv[:, (H + KV) * hd:].reshape(T, KV, hd)
        o = ChunkedAttention.apply(q.contiguous(), k.contiguous(), v.contiguous(), lens, hd ** -0.5)
        h = h + o.reshape(T, H * hd) @ P["o_w"].t()
        bn = _rms(h, P["ln2"])
        gu = bn @ P["gu_w"].t()
        h = h + (TF.silu(gu[:, :s.ffn]) * gu[:, s.ffn:]) @ P["down_w"].t()
    hf = _rms(h, E["norm"])
    head = E["emb"] if s.tied else E["head"]
    n_valid = int((batch.labels >= 0).sum().item())
    loss = 0.0
    for c0 in range(0, T, ce_chunk):
        c1 = min(T, c0 + ce_chunk)
        loss = loss + checkpoint(_ce_chunk, hf[c0:c1], head, batch.labels[c0:c1], use_reentrant=False)
    return loss / n_valid


def rel_l2(got, want):
    return ((got.float() - want.float()).norm() / want.float().norm().clamp_min(1e-30)).item()


def cosine(got, want):
    return TF.cosine_similarity(got.float().flatten(), want.float().flatten(), dim=0).item()
