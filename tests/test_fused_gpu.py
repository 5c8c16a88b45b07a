"""Fused worker kernels (csrc/worker_kernels.cu) vs torch fp32 references of
the same ops. bf16 outputs: rtol/atol 2e-2 (bf16 rounding); fp32 reductions
(dw, bias grad, loss): rtol 1e-3."""
import math

import pytest
import torch
import torch.nn.functional as TF

from paper_2601_19362_b200 import fused as F
from paper_2601_19362_b200 import worker as W

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def bf(*s, scale=1.0):
    return (torch.randn(*s, device=DEV) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("T,d", [(5, 256), (1000, 1536), (64, 2048), (77, 4096), (3, 5120)])
def test_rmsnorm(T, d):
    x, w, dy, res = bf(T, d), bf(d, scale=0.3) + 1, bf(T, d), bf(T, d)
    y, rstd = F.rmsnorm_fwd(x, w)
    xf = x.float().requires_grad_(True)
    wf = w.float().requires_grad_(True)
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-6) * wf
    torch.testing.assert_close(y.float(), ref.detach(), rtol=2e-2, atol=2e-2)
    ref.backward(dy.float())
    dw = torch.zeros(d, device=DEV)
    out = F.rmsnorm_bwd(dy, x, w, rstd, dw, resid=res)
    torch.testing.assert_close(out.float(), res.float() + xf.grad, rtol=2e-2, atol=3e-2)
    torch.testing.assert_close(dw, wf.grad, rtol=1e-3, atol=1e-2)


def test_qkv_rope_roundtrip_and_reference():
    T, H, KV, hd = 300, 12, 2, 128
    qkv, bias = bf(T, (H + 2 * KV) * hd), bf((H + 2 * KV) * hd)
    pos = torch.cat([torch.arange(100), torch.arange(200)]).to(DEV)
    tab = F.rope_table(4096, hd, W.ROPE_THETA, DEV)
    q, k, v = F.qkv_rope_fwd(qkv, bias, tab, pos, H, KV, hd)
    cos, sin = W.rope_tables(pos, hd)
    full = (qkv.float() + bias.float())

    def rope(x):
        h = hd // 2
        x1, x2 = x[..., :h], x[..., h:]
        return torch.cat([x1 * cos[:, None] - x2 * sin[:, None], x2 * cos[:, None] + x1 * sin[:, None]], -1)

    torch.testing.assert_close(q.float(), rope(full[:, :H * hd].view(T, H, hd)), rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(k.float(), rope(full[:, H * hd:(H + KV) * hd].view(T, KV, hd)), rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(v.float(), full[:, (H + KV) * hd:].view(T, KV, hd), rtol=2e-2, atol=2e-2)
    back = F.qkv_rope_bwd(q, k, v, tab, pos, H, KV, hd)  # transpose of a rotation = its inverse
    torch.testing.assert_close(back.float(), full, rtol=3e-2, atol=3e-2)
    cs = torch.zeros((H + 2 * KV) * hd, device=DEV)
    F.col_sum_(back, cs)
    torch.testing.assert_close(cs, back.float().sum(0), rtol=1e-3, atol=1e-2)


def test_swiglu():
    T, ffn = 513, 8960
    gu, dm = bf(T, 2 * ffn), bf(T, ffn)
    m = F.swiglu_fwd(gu, ffn)
    g = gu.float()[:, :ffn].requires_grad_(True)
    u = gu.float()[:, ffn:].requires_grad_(True)
    ref = TF.silu(g) * u
    torch.testing.assert_close(m.float(), ref.detach(), rtol=2e-2, atol=2e-2)
    ref.backward(dm.float())
    dgu = F.swiglu_bwd(dm, gu, ffn)
    torch.testing.assert_close(dgu.float(), torch.cat([g.grad, u.grad], -1), rtol=2e-2, atol=2e-2)


def test_cross_entropy():
    rows, V = 257, 151936
    logits = bf(rows, V, scale=3.0)
    labels = torch.randint(0, V, (rows,), device=DEV)
    labels[::7] = -100
    lf = logits.float().requires_grad_(True)
    n_valid = int((labels >= 0).sum())
    ref = TF.cross_entropy(lf, labels, ignore_index=-100, reduction="sum")
    (ref / n_valid).backward()
    loss = torch.zeros((), device=DEV)
    dl = F.ce_fwd_bwd_(logits.clone(), labels, 1.0 / n_valid, loss)
    torch.testing.assert_close(loss, ref.detach(), rtol=1e-3, atol=1e-2)
    torch.testing.assert_close(dl.float(), lf.grad, rtol=2e-2, atol=1e-6 + 1e-2 / n_valid)
