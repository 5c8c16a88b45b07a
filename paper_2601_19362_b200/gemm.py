"""Python entry to the tcgen05 bf16 GEMM of libodc.so (csrc/gemm.cu).

    linear_fwd(x, w)      y  = x · wᵀ          x [T, in], w [out, in]
    linear_dgrad(dy, w)   dx = dy · w          dy [T, out]
    linear_wgrad(dy, x)   dw = dyᵀ · x  (fp32) -> [out, in]
Operands are used in place (MN-major smem descriptors), never transposed.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check, lib


def _p(t):
    return C.c_void_p(t.data_ptr())


class Recorder:
    """Optional live timing of every GEMM launch (CUDA events on the launching
    stream) for the bench's roofline: records (flops, start, end, shape key)."""

    def __init__(self):
        self.rows = []

    @staticmethod
    def alg_bytes(key):
        """Operand + result bytes of one launch: bf16 A [M,K] and B [N,K], the output (fp32 or bf16, read
        too when accumulating), the fused residual; the SwiGLU launch writes gu [T,2F] and m [T,F]."""
        M, N, K, _, _, f32, acc, res = key
        if res == "glu":
            return 2 * (M * K + N * K) + 2 * M * N + 2 * M * (N // 2)
        out = (4 if f32 else 2) * M * N
        return 2 * (M * K + N * K) + out * (2 if acc else 1) + (2 * M * N if res else 0)

    def summary(self):
        if not self.rows:
            return None
        ms = [r[1].elapsed_time(r[2]) for r in self.rows]
        fl = sum(r[0] for r in self.rows)
        return {"launches": len(self.rows), "flops": fl, "ms": sum(ms),
                "alg_bytes": sum(self.alg_bytes(r[3]) for r in self.rows)}


recorder = None


def gemm(a, b, out, M, N, K, lda, ldb, a_mn, b_mn, accumulate=False, stream=None, residual=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    dt = _lib.ODC_F32 if out.dtype == torch.float32 else _lib.ODC_BF16
    rec = recorder
    if rec is not None:
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
    if residual is not None:
        assert residual.dtype == torch.bfloat16 and residual.stride(0) == out.stride(0)
    check(lib().odc_gemm_bf16(_p(a), _p(b), _p(out), None if residual is None else _p(residual), M, N, K, lda, ldb,
                              out.stride(0), int(a_mn), int(b_mn), dt, int(accumulate), C.c_void_p(s.cuda_stream)))
    if rec is not None:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(s)
        rec.rows.append((2.0 * M * N * K, e0, e1, (M, N, K, int(a_mn), int(b_mn), out.dtype == torch.float32,
                                                    bool(accumulate), residual is not None)))
    return out


def linear_fwd(x, w, out=None, residual=None):
    """y = x·wᵀ (+ residual, fused in the epilogue)."""
    T, K = x.shape
    N = w.shape[0]
    out = torch.empty(T, N, dtype=torch.bfloat16, device=x.device) if out is None else out
    return gemm(x, w, out, T, N, K, x.stride(0), w.stride(0), 0, 0, residual=residual)


def linear_dgrad(dy, w, out=None):
    T, N_out = dy.shape
    K_in = w.shape[1]
    out = torch.empty(T, K_in, dtype=torch.bfloat16, device=dy.device) if out is None else out
    return gemm(dy, w, out, T, K_in, N_out, dy.stride(0), w.stride(0), 0, 1)


def linear_wgrad(dy, x, out=None, accumulate=False):
    T, N_out = dy.shape
    K_in = x.shape[1]
    out = torch.empty(N_out, K_in, dtype=torch.float32, device=dy.device) if out is None else out
    return gemm(dy, x, out, N_out, K_in, T, dy.stride(0), x.stride(0), 1, 1, accumulate=accumulate)


def gate_up_swiglu(x, w, ffn):
    """gu = x·wᵀ (w = [gate; up], [2*ffn, d]) and m = silu(gate)·up fused in the
    GEMM epilogue (csrc/gemm.cu glu mode). Returns (gu [T, 2*ffn], m [T, ffn])."""
    T, d = x.shape
    assert w.shape == (2 * ffn, d) and x.is_contiguous() and w.is_contiguous()
    gu = torch.empty(T, 2 * ffn, dtype=torch.bfloat16, device=x.device)
    m = torch.empty(T, ffn, dtype=torch.bfloat16, device=x.device)
    s = torch.cuda.current_stream()
    rec = recorder
    if rec is not None:
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
    check(lib().odc_gemm_gate_up_swiglu(_p(x), _p(w), _p(gu), _p(m), T, ffn, d, C.c_void_p(s.cuda_stream)))
    if rec is not None:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(s)
        rec.rows.append((2.0 * T * 2 * ffn * d, e0, e1, (T, 2 * ffn, d, 0, 0, False, False, "glu")))
    return gu, m

