// worker_kernels.cu — fused elementwise kernels of the SFT worker (the caller
// of the ODC path; no reference counterpart). bf16 in/out, fp32 math, 16-byte
// vector access, one kernel per fused op instead of a chain of torch ops:
//   rmsnorm_fwd        y = x * rsqrt(mean(x^2)+eps) * w, rstd saved
//   rmsnorm_bwd        out = resid + dx, dw += sum_rows dy * xhat   (fused residual)
//   qkv_rope_fwd       (+bias) split packed qkv, RoPE(q, k) from a cos/sin table
//   qkv_rope_bwd       inverse RoPE(dq, dk), pack [dq|dk|dv]
//   col_sum            bias gradient (fp32 column sums)
//   swiglu_fwd/bwd     m = silu(g) * u and its gradient
//   ce_fwd_bwd         per row: online logsumexp, loss, dlogits = (softmax - onehot)*scale in place
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "common.hpp"
#include "kernels.cuh"

namespace odc {
namespace wk {

__device__ __forceinline__ float bf(unsigned short h) { return __uint_as_float(static_cast<unsigned>(h) << 16); }
__device__ __forceinline__ unsigned short tobf(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }

__device__ __forceinline__ void unpack8(const uint4& v, float* f) {
    const unsigned* w = reinterpret_cast<const unsigned*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
    uint4 v;
    unsigned* w = reinterpret_cast<unsigned*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = static_cast<unsigned>(tobf(f[2 * i])) | (static_cast<unsigned>(tobf(f[2 * i + 1])) << 16);
    return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- RMSNorm
__global__ void rmsnorm_fwd_kernel(const uint4* __restrict__ x, const uint4* __restrict__ w, uint4* __restrict__ y,
                                   float* __restrict__ rstd, long long T, int dv, float eps) {
    const int lane = threadIdx.x % 32;
    const long long row = static_cast<long long>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= T) return;
    const uint4* xr = x + row * dv;
    float ss = 0.f;
    for (int i = lane; i < dv; i += 32) {
        float f[8];
        unpack8(xr[i], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
    }
    ss = warp_sum(ss);
    const float r = rsqrtf(ss / (dv * 8) + eps);
    if (lane == 0) rstd[row] = r;
    for (int i = lane; i < dv; i += 32) {
        float f[8], g[8];
        unpack8(xr[i], f);
        unpack8(w[i], g);
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = f[j] * r * g[j];
        y[row * dv + i] = pack8(f);
    }
}

// Register variant for d <= 32*8*KMAX: every 16 B load of the row is issued
// before the reduction and the row is normalised from registers (no re-read).
template <int KMAX>
__global__ void rmsnorm_fwd_reg_kernel(const uint4* __restrict__ x, const uint4* __restrict__ w, uint4* __restrict__ y,
                                       float* __restrict__ rstd, long long T, int dv, float eps) {
    const int lane = threadIdx.x % 32;
    const long long row = static_cast<long long>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= T) return;
    const uint4* xr = x + row * dv;
    uint4 q[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        const int i = lane + 32 * k;
        if (i < dv) q[k] = xr[i];
    }
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        if (lane + 32 * k < dv) {
            float f[8];
            unpack8(q[k], f);
#pragma unroll
            for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
        }
    }
    ss = warp_sum(ss);
    const float r = rsqrtf(ss / (dv * 8) + eps);
    if (lane == 0) rstd[row] = r;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        const int i = lane + 32 * k;
        if (i < dv) {
            float f[8], g[8];
            unpack8(q[k], f);
            unpack8(__ldg(w + i), g);
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = f[j] * r * g[j];
            y[row * dv + i] = pack8(f);
        }
    }
}

// one warp per row, 8 warps per block; dw partials in smem, then global atomics
__global__ void rmsnorm_bwd_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ x, const uint4* __restrict__ w,
                                   const float* __restrict__ rstd, const uint4* __restrict__ resid, uint4* __restrict__ out,
                                   float* __restrict__ dw, long long T, int dv) {
    extern __shared__ float sdw[];
    const int d = dv * 8;
    for (int i = threadIdx.x; i < d; i += blockDim.x) sdw[i] = 0.f;
    __syncthreads();
    const int lane = threadIdx.x % 32, wid = threadIdx.x / 32, nw = blockDim.x / 32;
    for (long long row = static_cast<long long>(blockIdx.x) * nw + wid; row < T; row += static_cast<long long>(gridDim.x) * nw) {
        const float r = rstd[row];
        float dot = 0.f;
        for (int i = lane; i < dv; i += 32) {
            float a[8], b[8], g[8];
            unpack8(dy[row * dv + i], a);
            unpack8(x[row * dv + i], b);
            unpack8(w[i], g);
#pragma unroll
            for (int j = 0; j < 8; ++j) dot += a[j] * g[j] * b[j] * r;
        }
        const float c = warp_sum(dot) / d;
        for (int i = lane; i < dv; i += 32) {
            float a[8], b[8], g[8], o[8];
            unpack8(dy[row * dv + i], a);
            unpack8(x[row * dv + i], b);
            unpack8(w[i], g);
            if (resid) unpack8(resid[row * dv + i], o);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float xh = b[j] * r;
                const float dxh = a[j] * g[j];
                o[j] = (resid ? o[j] : 0.f) + r * (dxh - xh * c);
                atomicAdd(&sdw[i * 8 + j], a[j] * xh);
            }
            out[row * dv + i] = pack8(o);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += blockDim.x) atomicAdd(&dw[i], sdw[i]);
}

// Register-accumulator variant: lane l of every warp owns the uint4 columns l, l+32, .. (KMAX per lane), so
// the dw partial of the rows a warp handles stays in registers; one shared-memory reduction per block at the end.
template <int KMAX>
__global__ void __launch_bounds__(256, KMAX > 4 ? 1 : 2) rmsnorm_bwd_reg_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ x,
                                                                const uint4* __restrict__ w, const float* __restrict__ rstd,
                                                                const uint4* __restrict__ resid, uint4* __restrict__ out,
                                                                float* __restrict__ dw, long long T, int dv) {
    extern __shared__ float sdw[];
    const int d = dv * 8;
    for (int i = threadIdx.x; i < d; i += blockDim.x) sdw[i] = 0.f;
    const int lane = threadIdx.x % 32, wid = threadIdx.x / 32, nw = blockDim.x / 32;
    float acc[KMAX][8];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[k][j] = 0.f;
    }
    for (long long row = static_cast<long long>(blockIdx.x) * nw + wid; row < T; row += static_cast<long long>(gridDim.x) * nw) {
        const float r = rstd[row];
        const uint4* dyr = dy + row * dv;
        const uint4* xr = x + row * dv;
        const uint4* rr = resid ? resid + row * dv : nullptr;
        // every load of the row (dy, x and the residual) in flight at once, kept in registers for both passes
        uint4 ra[KMAX], rb[KMAX], rc[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int i = lane + 32 * k;
            if (i < dv) {
                ra[k] = dyr[i];
                rb[k] = xr[i];
                if (rr) rc[k] = rr[i];
            }
        }
        float dot = 0.f;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int i = lane + 32 * k;
            if (i < dv) {
                float a[8], bb[8], g[8];
                unpack8(ra[k], a);
                unpack8(rb[k], bb);
                unpack8(__ldg(w + i), g);
#pragma unroll
                for (int j = 0; j < 8; ++j) dot += a[j] * g[j] * bb[j];
            }
        }
        const float c = warp_sum(dot) * r / d;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {  // residual, output, dw partial from the registers
            const int i = lane + 32 * k;
            if (i < dv) {
                float a[8], bb[8], g[8], o[8];
                unpack8(ra[k], a);
                unpack8(rb[k], bb);
                unpack8(__ldg(w + i), g);
                if (rr) unpack8(rc[k], o);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float xh = bb[j] * r;
                    o[j] = (rr ? o[j] : 0.f) + r * (a[j] * g[j] - xh * c);
                    acc[k][j] += a[j] * xh;  // dw += dy * xhat
                }
                out[row * dv + i] = pack8(o);
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        const int i = lane + 32 * k;
        if (i < dv) {
#pragma unroll
            for (int j = 0; j < 8; ++j) atomicAdd(&sdw[i * 8 + j], acc[k][j]);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += blockDim.x) atomicAdd(&dw[i], sdw[i]);
}

// ------------------------------------------------------------------- RoPE
// rotate-half convention: y1 = x1 c - x2 s, y2 = x2 c + x1 s (inverse: s -> -s)
// table: [max_pos][hd/2] float2 {cos, sin}
__global__ void qkv_rope_fwd_kernel(const unsigned short* __restrict__ qkv, const unsigned short* __restrict__ bias,
                                    const float2* __restrict__ table, const long long* __restrict__ pos,
                                    unsigned short* __restrict__ q, unsigned short* __restrict__ k,
                                    unsigned short* __restrict__ v, long long T, int H, int KV, int hd) {
    const int half = hd / 2, groups = half / 8;  // 8 pairs per thread
    const int heads = H + 2 * KV;
    const long long total = T * heads * groups;
    for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int gi = static_cast<int>(idx % groups);
        const int h = static_cast<int>((idx / groups) % heads);
        const long long t = idx / (static_cast<long long>(groups) * heads);
        const long long src = t * heads * hd + static_cast<long long>(h) * hd + gi * 8;
        float a[8], b[8];
        unpack8(__ldg(reinterpret_cast<const uint4*>(qkv + src)), a);
        unpack8(__ldg(reinterpret_cast<const uint4*>(qkv + src + half)), b);
        if (bias) {
            float ba[8], bb[8];
            unpack8(__ldg(reinterpret_cast<const uint4*>(bias + h * hd + gi * 8)), ba);
            unpack8(__ldg(reinterpret_cast<const uint4*>(bias + h * hd + gi * 8 + half)), bb);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                a[j] += ba[j];
                b[j] += bb[j];
            }
        }
        unsigned short* dst;
        long long off;
        if (h < H) {
            dst = q;
            off = (t * H + h) * hd;
        } else if (h < H + KV) {
            dst = k;
            off = (t * KV + (h - H)) * hd;
        } else {
            dst = v;
            off = (t * KV + (h - H - KV)) * hd;
        }
        if (h < H + KV) {
            // 8 (cos, sin) pairs as four 16 B loads (the table row is 64 B aligned)
            const float4* cs4 = reinterpret_cast<const float4*>(table + pos[t] * half + gi * 8);
            float cc[8], sn[8];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                const float4 u = __ldg(cs4 + q4);
                cc[2 * q4] = u.x;
                sn[2 * q4] = u.y;
                cc[2 * q4 + 1] = u.z;
                sn[2 * q4 + 1] = u.w;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float c = cc[j], s = sn[j];
                const float x1 = a[j], x2 = b[j];
                a[j] = x1 * c - x2 * s;
                b[j] = x2 * c + x1 * s;
            }
        }
        *reinterpret_cast<uint4*>(dst + off + gi * 8) = pack8(a);
        *reinterpret_cast<uint4*>(dst + off + gi * 8 + half) = pack8(b);
    }
}

__global__ void qkv_rope_bwd_kernel(const unsigned short* __restrict__ dq, const unsigned short* __restrict__ dk,
                                    const unsigned short* __restrict__ dv, const float2* __restrict__ table,
                                    const long long* __restrict__ pos, unsigned short* __restrict__ dqkv, long long T,
                                    int H, int KV, int hd) {
    const int half = hd / 2, groups = half / 8;
    const int heads = H + 2 * KV;
    const long long total = T * heads * groups;
    for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int gi = static_cast<int>(idx % groups);
        const int h = static_cast<int>((idx / groups) % heads);
        const long long t = idx / (static_cast<long long>(groups) * heads);
        const unsigned short* src;
        if (h < H) src = dq + (t * H + h) * hd;
        else if (h < H + KV) src = dk + (t * KV + (h - H)) * hd;
        else src = dv + (t * KV + (h - H - KV)) * hd;
        float a[8], b[8];
        unpack8(*reinterpret_cast<const uint4*>(src + gi * 8), a);
        unpack8(*reinterpret_cast<const uint4*>(src + gi * 8 + half), b);
        if (h < H + KV) {
            // 8 (cos, sin) pairs as four 16 B loads (the table row is 64 B aligned)
            const float4* cs4 = reinterpret_cast<const float4*>(table + pos[t] * half + gi * 8);
            float cc[8], sn[8];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                const float4 u = __ldg(cs4 + q4);
                cc[2 * q4] = u.x;
                sn[2 * q4] = u.y;
                cc[2 * q4 + 1] = u.z;
                sn[2 * q4 + 1] = u.w;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float c = cc[j], s = sn[j];
                const float y1 = a[j], y2 = b[j];
                a[j] = y1 * c + y2 * s;
                b[j] = y2 * c - y1 * s;
            }
        }
        const long long dst = t * heads * hd + static_cast<long long>(h) * hd + gi * 8;
        *reinterpret_cast<uint4*>(dqkv + dst) = pack8(a);
        *reinterpret_cast<uint4*>(dqkv + dst + half) = pack8(b);
    }
}

// column sums of a [T, n] bf16 matrix into fp32 out (out += sums)
__global__ void col_sum_kernel(const unsigned short* __restrict__ m, float* __restrict__ out, long long T, int n,
                               int rows_per_block) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= n) return;
    const long long r0 = static_cast<long long>(blockIdx.y) * rows_per_block;
    const long long r1 = r0 + rows_per_block < T ? r0 + rows_per_block : T;
    float acc = 0.f;
    for (long long r = r0; r < r1; ++r) acc += bf(m[r * n + col]);
    atomicAdd(&out[col], acc);
}

// ----------------------------------------------------------------- SwiGLU
// one row per block-iteration, columns across the threads: no 64-bit division per element
// The backward takes two 16-byte column groups per thread per step, every load
// issued before any math (6 independent 16 B loads in flight instead of 3):
// 350 -> 292 us at T=19K (4.86 -> 5.83 TB/s). The same change made the
// forward slower (174 -> 190 us), so it keeps one group per step.
constexpr int kGluThreads = 256;

__global__ void swiglu_fwd_kernel(const uint4* __restrict__ gu, uint4* __restrict__ m, long long T, int fv) {
    for (long long t = blockIdx.x; t < T; t += gridDim.x) {
        const uint4* gr = gu + t * 2 * fv;
        uint4* mr = m + t * fv;
        for (int c = threadIdx.x; c < fv; c += blockDim.x) {
            float g[8], u[8];
            unpack8(gr[c], g);
            unpack8(gr[fv + c], u);
#pragma unroll
            for (int j = 0; j < 8; ++j) g[j] = __fdividef(g[j], 1.f + __expf(-g[j])) * u[j];
            mr[c] = pack8(g);
        }
    }
}

__device__ __forceinline__ void swiglu_bwd8(const uint4& dv, const uint4& gv, const uint4& uv, uint4& dgo, uint4& duo) {
    float d[8], g[8], u[8], dg[8], du[8];
    unpack8(dv, d);
    unpack8(gv, g);
    unpack8(uv, u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float sg = __frcp_rn(1.f + __expf(-g[j]));
        dg[j] = d[j] * u[j] * sg * (1.f + g[j] * (1.f - sg));
        du[j] = d[j] * g[j] * sg;
    }
    dgo = pack8(dg);
    duo = pack8(du);
}

__global__ void __launch_bounds__(kGluThreads) swiglu_bwd_kernel(const uint4* __restrict__ dm,
                                                                 const uint4* __restrict__ gu,
                                                                 uint4* __restrict__ dgu, long long T, int fv) {
    for (long long t = blockIdx.x; t < T; t += gridDim.x) {
        const uint4* gr = gu + t * 2 * fv;
        const uint4* dr = dm + t * fv;
        uint4* orow = dgu + t * 2 * fv;
        for (int c = threadIdx.x; c < fv; c += 2 * kGluThreads) {
            const int c2 = c + kGluThreads;
            const bool two = c2 < fv;
            const uint4 d0 = dr[c], g0 = gr[c], u0 = gr[fv + c];
            uint4 d1 = d0, g1 = g0, u1 = u0;
            if (two) {
                d1 = dr[c2];
                g1 = gr[c2];
                u1 = gr[fv + c2];
            }
            uint4 a, b;
            swiglu_bwd8(d0, g0, u0, a, b);
            orow[c] = a;
            orow[fv + c] = b;
            if (two) {
                swiglu_bwd8(d1, g1, u1, a, b);
                orow[c2] = a;
                orow[fv + c2] = b;
            }
        }
    }
}

// ------------------------------------------------------- cross entropy
// one CTA per row; logits row overwritten by dlogits = (softmax - onehot) * scale
constexpr int kCeThreadsDefault = 512;
constexpr int kCeUnroll = 1;  // 4 measured slower (1.27 vs 1.21 ms per 8K rows)
template <int kCeThreads>
__global__ void __launch_bounds__(kCeThreads) ce_kernel(uint4* __restrict__ logits, const long long* __restrict__ labels,
                                                        long long rows, int vv, float scale, float* __restrict__ loss) {
    const long long row = blockIdx.x;
    uint4* L = logits + row * vv;
    const long long lab = labels[row];
    __shared__ float red_m[kCeThreads / 32], red_s[kCeThreads / 32];
    __shared__ float s_lse;
    // online (max, sum) per 16 B chunk: one max over the 8 values, one
    // rescale, 8 exps, no data-dependent branches
    float mx = -INFINITY, sm = 0.f;
    // kCeUnroll 16 B loads in flight per thread before any math
    int i0 = threadIdx.x;
    for (; i0 + (kCeUnroll - 1) * kCeThreads < vv; i0 += kCeUnroll * kCeThreads) {
        uint4 q[kCeUnroll];
#pragma unroll
        for (int u = 0; u < kCeUnroll; ++u) q[u] = L[i0 + u * kCeThreads];
#pragma unroll
        for (int u = 0; u < kCeUnroll; ++u) {
            float f[8];
            unpack8(q[u], f);
            const float cm = fmaxf(fmaxf(fmaxf(f[0], f[1]), fmaxf(f[2], f[3])),
                                   fmaxf(fmaxf(f[4], f[5]), fmaxf(f[6], f[7])));
            const float m = fmaxf(mx, cm);
            float cs = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) cs += __expf(f[j] - m);
            sm = (mx == -INFINITY ? 0.f : sm * __expf(mx - m)) + cs;
            mx = m;
        }
    }
    for (int i = i0; i < vv; i += kCeThreads) {
        float f[8];
        unpack8(L[i], f);
        float cm = fmaxf(fmaxf(fmaxf(f[0], f[1]), fmaxf(f[2], f[3])), fmaxf(fmaxf(f[4], f[5]), fmaxf(f[6], f[7])));
        const float m = fmaxf(mx, cm);
        float cs = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) cs += __expf(f[j] - m);
        sm = (mx == -INFINITY ? 0.f : sm * __expf(mx - m)) + cs;
        mx = m;
    }
    // warp then block reduction of (max, sum)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, mx, o), s2 = __shfl_xor_sync(0xffffffffu, sm, o);
        const float m = fmaxf(mx, m2);
        sm = (mx == -INFINITY ? 0.f : sm * __expf(mx - m)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - m));
        mx = m;
    }
    if (threadIdx.x % 32 == 0) {
        red_m[threadIdx.x / 32] = mx;
        red_s[threadIdx.x / 32] = sm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = red_m[0], S = red_s[0];
        for (int w = 1; w < kCeThreads / 32; ++w) {
            const float m = fmaxf(M, red_m[w]);
            S = S * __expf(M - m) + red_s[w] * __expf(red_m[w] - m);
            M = m;
        }
        s_lse = M + logf(S);
        if (lab >= 0) {
            const unsigned short* Ls = reinterpret_cast<const unsigned short*>(L);
            atomicAdd(loss, s_lse - bf(Ls[lab]));
        }
    }
    __syncthreads();
    const float lse = s_lse;
    const float sc = lab >= 0 ? scale : 0.f;
    int i1 = threadIdx.x;
    for (; i1 + (kCeUnroll - 1) * kCeThreads < vv; i1 += kCeUnroll * kCeThreads) {
        uint4 q[kCeUnroll];
#pragma unroll
        for (int u = 0; u < kCeUnroll; ++u) q[u] = L[i1 + u * kCeThreads];
#pragma unroll
        for (int u = 0; u < kCeUnroll; ++u) {
            float f[8];
            unpack8(q[u], f);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const long long col = static_cast<long long>(i1 + u * kCeThreads) * 8 + j;
                f[j] = (__expf(f[j] - lse) - (col == lab ? 1.f : 0.f)) * sc;
            }
            L[i1 + u * kCeThreads] = pack8(f);
        }
    }
    for (int i = i1; i < vv; i += kCeThreads) {
        float f[8];
        unpack8(L[i], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const long long col = static_cast<long long>(i) * 8 + j;
            f[j] = (__expf(f[j] - lse) - (col == lab ? 1.f : 0.f)) * sc;
        }
        L[i] = pack8(f);
    }
}

int grid_for(long long n, int threads) {
    long long g = (n + threads - 1) / threads;
    return static_cast<int>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

void ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void need(bool c, const char* what) {
    if (!c) throw odcsim::ParamError(what);
}

}  // namespace wk
}  // namespace odc

using namespace odc::wk;

extern "C" {

odc_status odc_w_rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, std::int64_t T, int d, float eps,
                             void* stream) {
    return odc::guard([&] {
        need(d % 8 == 0, "rmsnorm: d % 8 == 0");
        odc::count_launch();
        const int dv = d / 8;
        auto go = [&](auto kern) {
            kern<<<static_cast<int>((T + 7) / 8), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
                static_cast<const uint4*>(x), static_cast<const uint4*>(w), static_cast<uint4*>(y), rstd, T, dv, eps);
        };
        if (dv <= 32 * 6) go(rmsnorm_fwd_reg_kernel<6>);
        else if (dv <= 32 * 16) go(rmsnorm_fwd_reg_kernel<16>);
        else if (dv <= 32 * 20) go(rmsnorm_fwd_reg_kernel<20>);
        else go(rmsnorm_fwd_kernel);
        ok(cudaGetLastError(), "rmsnorm_fwd");
    });
}

odc_status odc_w_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd, const void* resid,
                             void* out, float* dw, std::int64_t T, int d, void* stream) {
    return odc::guard([&] {
        need(d % 8 == 0, "rmsnorm: d % 8 == 0");
        const int kmax = (d / 8 + 31) / 32;  // uint4 columns per lane
        // register kernels: one wave of exactly the resident CTAs (1 per SM for KMAX > 4, else 2) — every
        // extra CTA pays the dw reduction again (T=19K: 79 -> 60 us, T=4K: 39 -> 21 us vs 4 per SM)
        const int grid_per_sm = kmax > 6 ? 4 : kmax > 4 ? 1 : 2;
        const int blocks = static_cast<int>(std::min<long long>((T + 7) / 8, 148 * grid_per_sm));
        odc::count_launch();
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        auto args = [&](auto kern) {
            kern<<<blocks, 256, d * sizeof(float), st>>>(static_cast<const uint4*>(dy), static_cast<const uint4*>(x),
                                                         static_cast<const uint4*>(w), rstd,
                                                         static_cast<const uint4*>(resid), static_cast<uint4*>(out), dw,
                                                         T, d / 8);
        };
        switch (kmax) {
            case 1: args(rmsnorm_bwd_reg_kernel<1>); break;
            case 2: args(rmsnorm_bwd_reg_kernel<2>); break;
            case 3: args(rmsnorm_bwd_reg_kernel<3>); break;
            case 4: args(rmsnorm_bwd_reg_kernel<4>); break;
            case 5: args(rmsnorm_bwd_reg_kernel<5>); break;
            case 6: args(rmsnorm_bwd_reg_kernel<6>); break;
            default: args(rmsnorm_bwd_kernel); break;  // wide rows: shared-memory dw accumulation
        }
        ok(cudaGetLastError(), "rmsnorm_bwd");
    });
}

odc_status odc_w_qkv_rope_fwd(const void* qkv, const void* bias, const void* table, const std::int64_t* pos, void* q,
                              void* k, void* v, std::int64_t T, int H, int KV, int hd, void* stream) {
    return odc::guard([&] {
        need(hd % 16 == 0, "rope: head_dim % 16 == 0");
        const long long n = T * (H + 2 * KV) * (hd / 16);
        odc::count_launch();
        qkv_rope_fwd_kernel<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
            static_cast<const unsigned short*>(qkv), static_cast<const unsigned short*>(bias),
            static_cast<const float2*>(table), reinterpret_cast<const long long*>(pos), static_cast<unsigned short*>(q),
            static_cast<unsigned short*>(k), static_cast<unsigned short*>(v), T, H, KV, hd);
        ok(cudaGetLastError(), "qkv_rope_fwd");
    });
}

odc_status odc_w_qkv_rope_bwd(const void* dq, const void* dk, const void* dv, const void* table,
                              const std::int64_t* pos, void* dqkv, std::int64_t T, int H, int KV, int hd, void* stream) {
    return odc::guard([&] {
        need(hd % 16 == 0, "rope: head_dim % 16 == 0");
        const long long n = T * (H + 2 * KV) * (hd / 16);
        odc::count_launch();
        qkv_rope_bwd_kernel<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
            static_cast<const unsigned short*>(dq), static_cast<const unsigned short*>(dk),
            static_cast<const unsigned short*>(dv), static_cast<const float2*>(table),
            reinterpret_cast<const long long*>(pos), static_cast<unsigned short*>(dqkv), T, H, KV, hd);
        ok(cudaGetLastError(), "qkv_rope_bwd");
    });
}

odc_status odc_w_col_sum(const void* m, float* out, std::int64_t T, int n, void* stream) {
    return odc::guard([&] {
        const int rpb = 256;
        dim3 grid((n + 255) / 256, static_cast<unsigned>((T + rpb - 1) / rpb));
        odc::count_launch();
        col_sum_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(static_cast<const unsigned short*>(m),
                                                                                out, T, n, rpb);
        ok(cudaGetLastError(), "col_sum");
    });
}

odc_status odc_w_swiglu_fwd(const void* gu, void* m, std::int64_t T, int ffn, void* stream) {
    return odc::guard([&] {
        need(ffn % 8 == 0, "swiglu: ffn % 8 == 0");
        odc::count_launch();
        swiglu_fwd_kernel<<<static_cast<unsigned>(std::min<long long>(T, 148 * 8)), 256, 0,
                            reinterpret_cast<cudaStream_t>(stream)>>>(
            static_cast<const uint4*>(gu), static_cast<uint4*>(m), T, ffn / 8);
        ok(cudaGetLastError(), "swiglu_fwd");
    });
}

odc_status odc_w_swiglu_bwd(const void* dm, const void* gu, void* dgu, std::int64_t T, int ffn, void* stream) {
    return odc::guard([&] {
        need(ffn % 8 == 0, "swiglu: ffn % 8 == 0");
        odc::count_launch();
        swiglu_bwd_kernel<<<static_cast<unsigned>(std::min<long long>(T, 148 * 8)), 256, 0,
                            reinterpret_cast<cudaStream_t>(stream)>>>(
            static_cast<const uint4*>(dm), static_cast<const uint4*>(gu), static_cast<uint4*>(dgu), T, ffn / 8);
        ok(cudaGetLastError(), "swiglu_bwd");
    });
}

odc_status odc_w_ce_fwd_bwd(void* logits, const std::int64_t* labels, std::int64_t rows, std::int64_t vocab,
                            float scale, float* loss, void* stream) {
    return odc::guard([&] {
        need(vocab % 8 == 0, "ce: vocab % 8 == 0");
        if (rows <= 0) return;
        odc::count_launch();
        // threads per row-CTA (ODC_CE_THREADS 256/512/1024 for A/B). Fewer
        // resident CTAs via extra shared memory (so the gradient pass re-reads
        // from L2) measured slower (profiles/r01/ce_occupancy_ab.jsonl).
        static const int nt = [] {
            const char* e = std::getenv("ODC_CE_THREADS");
            return e ? std::atoi(e) : kCeThreadsDefault;
        }();
        auto go = [&](auto kern, int threads) {
            kern<<<static_cast<unsigned>(rows), threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
                static_cast<uint4*>(logits), reinterpret_cast<const long long*>(labels), rows,
                static_cast<int>(vocab / 8), scale, loss);
        };
        if (nt == 256) go(ce_kernel<256>, 256);
        else if (nt == 1024) go(ce_kernel<1024>, 1024);
        else go(ce_kernel<512>, 512);
        ok(cudaGetLastError(), "ce");
    });
}

}  // extern "C"
