"""tcgen05 GEMM parity vs torch fp32 matmul of the same bf16 operands.
Tolerance: bf16 outputs within bf16 rounding (rtol 1e-2 / atol 1e-2 on unit-
scale data); fp32 outputs (wgrad) within rtol 2e-3 of the fp32 reference
(accumulation order differs)."""
import pytest
import torch

from paper_2601_19362_b200 import gemm as G

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _r(*s):
    return (torch.randn(*s, device=DEV) * 0.5).to(torch.bfloat16)


@pytest.mark.parametrize("T,inn,out", [(128, 64, 128), (1000, 1536, 256), (4096, 1536, 8960), (333, 8960, 1536),
                                       (257, 192, 320), (4096, 256, 384), (16384, 1536, 1536)])
def test_fwd_dgrad_wgrad(T, inn, out):
    x, w, dy = _r(T, inn), _r(out, inn), _r(T, out)
    y = G.linear_fwd(x, w)
    torch.testing.assert_close(y.float(), x.float() @ w.float().t(), rtol=1e-2, atol=2e-2 * (inn / 64) ** 0.5)
    dx = G.linear_dgrad(dy, w)
    torch.testing.assert_close(dx.float(), dy.float() @ w.float(), rtol=1e-2, atol=2e-2 * (out / 64) ** 0.5)
    dw = G.linear_wgrad(dy, x)
    ref = dy.float().t() @ x.float()
    torch.testing.assert_close(dw, ref, rtol=2e-3, atol=2e-3 * (T / 64) ** 0.5)


@pytest.mark.parametrize("T,inn,out", [(512, 256, 384), (4096, 320, 640), (8192, 1536, 2048)])
def test_accumulate_f32(T, inn, out):
    """wgrad accumulation into an existing fp32 grad: covers the 1-CTA tile,
    and the 2-CTA tile with and without split-K (partials red.add-ed into D)."""
    x, dy = _r(T, inn), _r(T, out)
    acc = torch.randn(out, inn, device=DEV)
    want = acc + dy.float().t() @ x.float()
    G.linear_wgrad(dy, x, out=acc, accumulate=True)
    torch.testing.assert_close(acc, want, rtol=2e-3, atol=2e-3 * (T / 64) ** 0.5)


@pytest.mark.parametrize("T,inn,out", [(1000, 1536, 1536), (333, 256, 320), (4096, 512, 2048)])
def test_fwd_residual_epilogue(T, inn, out):
    """y = x·wᵀ + r fused in the epilogue (residual row prefetched into
    registers on the 2-CTA fast path; generic path on the ragged N tail)."""
    x, w, r = _r(T, inn), _r(out, inn), _r(T, out)
    y = G.linear_fwd(x, w, residual=r)
    want = x.float() @ w.float().t() + r.float()
    torch.testing.assert_close(y.float(), want, rtol=1e-2, atol=2e-2 * (inn / 64) ** 0.5)


def test_bf16_accumulate_in_place():
    T, inn, out = 1024, 384, 768
    x, w = _r(T, inn), _r(out, inn)
    y = _r(T, out)
    want = x.float() @ w.float().t() + y.float()
    G.gemm(x, w, y, T, out, inn, x.stride(0), w.stride(0), False, False, accumulate=True)
    torch.testing.assert_close(y.float(), want, rtol=1e-2, atol=2e-2 * (inn / 64) ** 0.5)


@pytest.mark.parametrize("T,d,ffn", [(100, 256, 512), (1000, 1536, 8960), (4097, 512, 1024), (32768, 1536, 8960)])
def test_gate_up_swiglu_fused_matches_unfused(T, d, ffn):
    """SwiGLU fused into the gate_up GEMM epilogue: gu bit-identical to the
    plain GEMM, m bit-identical to the standalone swiglu kernel on that gu
    (T < 256 runs the unfused pair itself)."""
    from paper_2601_19362_b200 import fused as F

    x, w = _r(T, d), (torch.randn(2 * ffn, d, device=DEV) * 0.05).to(torch.bfloat16)
    gu, m = G.gate_up_swiglu(x, w, ffn)
    gu_ref = G.linear_fwd(x, w)
    assert torch.equal(gu, gu_ref)
    assert torch.equal(m, F.swiglu_fwd(gu_ref, ffn))
    g, u = gu_ref.float()[:, :ffn], gu_ref.float()[:, ffn:]
    torch.testing.assert_close(m.float(), torch.nn.functional.silu(g) * u, rtol=2e-2, atol=2e-2)

