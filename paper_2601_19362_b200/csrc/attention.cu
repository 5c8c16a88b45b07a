// attention.cu — causal varlen flash-attention on tcgen05 (the worker's
// attention; no reference counterpart — the reference models its cost as
// alpha*s^2, src/cost_model.cpp:14-18). head_dim 128, bf16 in/out, fp32
// softmax statistics, GQA (H query heads share H/KV kv heads).
//
// FORWARD. One CTA per (sequence, 256-query tile, query head), heaviest
// items first. The 256 queries are two 128-row tiles Q0, Q1 that ping-pong on
// the tensor core: while the softmax warpgroup of one tile works, the MMA
// warp runs the other tile's MMAs, so each softmax hides behind 1024 clk of
// tensor work.
//   warp 0     TMA: Q0, Q1 once; K_j and V_j through separate 2-stage rings.
//   warp 1     single-thread tcgen05.mma issuer, per KV tile j:
//                PV0_{j-1}.. order: S0_j, S1_j, then O0 += P0_j V_j, S0_{j+1},
//                O1 += P1_j V_j, S1_{j+1}.  P_t is read from TMEM (the A
//                operand of a TS-MMA), V from smem.
//   warps 4-7  softmax of Q0, warps 8-11 softmax of Q1 (setmaxnreg gives them
//              the registers of warpgroup 0): one query row per thread,
//              tcgen05.ld of the S row, causal / sequence-end mask, online
//              max / sum in the exp2 domain with lazy rescaling (O_t is
//              rescaled in TMEM only when the running max grows by more than
//              2^8), P_t (bf16 pairs) stored with tcgen05.st over the first 64
//              columns of S_t; finally O_t / l -> bf16, and the LSE.
// TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "common.hpp"
#include "kernels.cuh"

namespace odc {
namespace attn {

constexpr int HD = 128;
constexpr int BQ = 128, BKV = 128;
constexpr int kTile = BQ * HD * 2;              // 32 KB: one 128 x 128 bf16 tile (two 16 KB swizzle halves)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;       // log2 units

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
#ifdef ODC_ATTN_DEBUG
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    bool said = false;
    while (true) {
        unsigned ok;
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(su32(b)), "r"(parity)
            : "memory");
        if (ok) return;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (!said && t - t0 > 2000000000ull) {
            if (threadIdx.x % 32 == 0)
                printf("attn hang: block %d thread %d bar smem 0x%x parity %u\n", blockIdx.x, threadIdx.x, su32(b), parity);
            said = true;
        }
        if (t - t0 > 6000000000ull) asm volatile("trap;");
    }
}
#else
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
#endif
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, unsigned long long* bar, void* smem, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(smem)),
        "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ std::uint64_t sdesc(unsigned addr, unsigned lbo, unsigned sbo) {
    std::uint64_t d = static_cast<std::uint64_t>((addr & 0x3FFFF) >> 4);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
// bf16 x bf16 -> f32, M=128, N=128
__host__ __device__ constexpr unsigned idesc(int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<unsigned>(b_mn_major) << 16) | ((128u >> 3) << 17) |
           ((128u >> 4) << 24);
}
__host__ __device__ constexpr unsigned instr(int a_mn_major, int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<unsigned>(a_mn_major) << 15) |
           (static_cast<unsigned>(b_mn_major) << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma(unsigned d, std::uint64_t a, std::uint64_t b, unsigned id, unsigned acc) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// packed fp32x2 FMA / MUL (FFMA2 / FMUL2 on sm_100): two lanes of math per issue slot
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rc, {%6, %7};\n"
        "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    float2 d;
    asm("{\n.reg .b64 ra, rb, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmul.rn.f32x2 rd, ra, rb;\n"
        "mov.b64 {%0, %1}, rd;\n}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{\n.reg .b64 ra, rb, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nadd.rn.f32x2 rd, ra, rb;\n"
        "mov.b64 {%0, %1}, rd;\n}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// 2^x on the FMA pipe (takes load off MUFU.EX2): round-to-nearest split x = j + f via the 1.5*2^23 trick,
// degree-3 minimax of 2^f on [-0.5, 0.5] (max rel. error 7.5e-5, far below the bf16 rounding of P), then j
// added to the exponent field. x is clamped at -125 (masked scores give ~2^-125 instead of 0).
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
    x.x = fmaxf(x.x, -125.f);  // keeps the exponent field of the result >= 1 (2^f >= 0.707 has exponent 126)
    x.y = fmaxf(x.y, -125.f);
    const float2 magic = make_float2(12582912.f, 12582912.f);
    const float2 t = fadd2(x, magic);
    const float2 jf = fadd2(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = fadd2(x, make_float2(-jf.x, -jf.y));
    float2 p = ffma2(f, make_float2(0.05517132f, 0.05517132f), make_float2(0.24261054f, 0.24261054f));
    p = ffma2(p, f, make_float2(0.69326099f, 0.69326099f));
    p = ffma2(p, f, make_float2(0.99992811f, 0.99992811f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}
__device__ __forceinline__ unsigned pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<unsigned*>(&h);
}
__device__ __forceinline__ void sts128(const void* p, unsigned a, unsigned b, unsigned c, unsigned d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(su32(p)), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}

#define TM_LD32(taddr, r)                                                                                        \
    asm volatile(                                                                                                \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                       \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),      \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), \
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),            \
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),            \
          "=r"(r[30]), "=r"(r[31])                                                                               \
        : "r"(taddr))
#define TM_ST32(taddr, r)                                                                                          \
    asm volatile(                                                                                                  \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                              \
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),        \
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), \
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]),           \
        "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                                     \
        : "memory")

#ifdef ODC_ATTN_TRACE
// per-iteration SM clock stamps of the backward's CTA 0 (tools/attn_bwd_trace.py): [event][iteration]
constexpr int kTrEvents = 21, kTrIters = 64;
__device__ unsigned long long g_attn_trace[kTrEvents * kTrIters];
#define TR(ev, n)                                                                                  \
    do {                                                                                           \
        if (blockIdx.x == 0 && (n) < kTrIters) g_attn_trace[(ev) * kTrIters + (n)] = clock64();    \
    } while (0)
#else
#define TR(ev, n) \
    do {          \
    } while (0)
#endif

struct Item {
    int seq_start, seq_len, q_tile, head;
};

struct Args {
    const Item* items;
    int n_items;
    int H, KV;
    float scale_log2;  // softmax scale * log2(e)
    __nv_bfloat16* out;  // [T][H][HD]
    float* lse;          // [H][T] natural-log LSE
    long long T;
};

constexpr int kFwdThreads = 384;
constexpr int BQ2 = 2 * BQ;                       // queries per forward CTA
constexpr int kFwdSmem = kTile * 6 + 1024;         // Q0, Q1, K x2, V x2

// bf16 x bf16 -> f32, M=128, N=128, A (P) from TMEM (K-major), B (V) MN-major
__device__ __forceinline__ void mma_ts(unsigned d, unsigned a_tmem, std::uint64_t b, unsigned id, unsigned acc) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(id), "r"(acc)
        : "memory");
}

__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, Args g) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    char* sQ = smem;               // Q0 | Q1
    char* sK = smem + 2 * kTile;   // stage s at sK + s * kTile
    char* sV = smem + 4 * kTile;
    __shared__ __align__(8) unsigned long long q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2],
        p_full[2], o_done[2];
    __shared__ unsigned tmem_base;

    const Item it = g.items[blockIdx.x];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int kvh = it.head / (g.H / g.KV);
    const int q0 = it.q_tile * BQ2;  // first query row within the sequence
    const int n_kv_seq = (it.seq_len + BKV - 1) / BKV;
    // causal: Q tile t (rows q0 + 128t ..) sees KV tiles 0 .. 2*q_tile + t
    const int n0 = min(n_kv_seq, 2 * it.q_tile + 1), n1 = min(n_kv_seq, 2 * it.q_tile + 2);

    if (warp == 0 && lane == 0) {
        mbar_init(&q_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], 4);
            mbar_init(&o_done[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_q) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_k) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_v) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base;

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 80;" ::: "memory");
        if (warp == 0 && lane == 0) {  // ---- TMA
            const int row0 = it.seq_start + q0;
            mbar_expect_tx(&q_full, 2 * kTile);
            tma_2d(&map_q, &q_full, sQ, it.head * HD, row0);
            tma_2d(&map_q, &q_full, sQ + kTile / 2, it.head * HD + 64, row0);
            tma_2d(&map_q, &q_full, sQ + kTile, it.head * HD, row0 + BQ);
            tma_2d(&map_q, &q_full, sQ + kTile + kTile / 2, it.head * HD + 64, row0 + BQ);
            for (int j = 0; j < n1; ++j) {
                const int s = j & 1, k0 = it.seq_start + j * BKV;
                if (j >= 2) mbar_wait(&k_empty[s], ((j >> 1) - 1) & 1);
                mbar_expect_tx(&k_full[s], kTile);
                tma_2d(&map_k, &k_full[s], sK + s * kTile, kvh * HD, k0);
                tma_2d(&map_k, &k_full[s], sK + s * kTile + kTile / 2, kvh * HD + 64, k0);
                if (j >= 2) mbar_wait(&v_empty[s], ((j >> 1) - 1) & 1);
                mbar_expect_tx(&v_full[s], kTile);
                tma_2d(&map_v, &v_full[s], sV + s * kTile, kvh * HD, k0);
                tma_2d(&map_v, &v_full[s], sV + s * kTile + kTile / 2, kvh * HD + 64, k0);
            }
        } else if (warp == 1 && lane == 0) {  // ---- MMA issuer
            const unsigned id_qk = idesc(0), id_pv = idesc(1);
            mbar_wait(&q_full, 0);
            auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T into TMEM columns [128t, 128t + 128)
                const unsigned qa = su32(sQ + t * kTile), ka = su32(sK + (j & 1) * kTile);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const unsigned off = (kk >> 2) * (kTile / 2) + (kk & 3) * 32;
                    mma(tmem + t * 128, sdesc(qa + off, 16, 1024), sdesc(ka + off, 16, 1024), id_qk, kk > 0);
                }
                commit(&s_full[t]);
            };
            auto issue_pv = [&](int t, int j) {  // O_t += P_t V_j, P_t = bf16 pairs in TMEM columns [128t, 128t + 64)
                const unsigned va = su32(sV + (j & 1) * kTile);
                mbar_wait(&p_full[t], j & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk)
                    mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, sdesc(va + kk * 2048, kTile / 2, 1024), id_pv,
                           (j > 0 || kk > 0));
            };
            mbar_wait(&k_full[0], 0);
            issue_s(0, 0);
            issue_s(1, 0);
            commit(&k_empty[0]);
            for (int j = 0; j < n1; ++j) {
                const int s = j & 1;
                mbar_wait(&v_full[s], (j >> 1) & 1);
                if (j < n0) issue_pv(0, j);
                if (j + 1 == n0) commit(&o_done[0]);
                const bool more = j + 1 < n1;
                if (more) mbar_wait(&k_full[s ^ 1], ((j + 1) >> 1) & 1);
                if (j + 1 < n0) issue_s(0, j + 1);
                issue_pv(1, j);
                commit(&v_empty[s]);
                if (more) {
                    issue_s(1, j + 1);
                    commit(&k_empty[s ^ 1]);
                }
            }
            commit(&o_done[1]);
        }
    } else {  // ---- softmax / correction / epilogue: warpgroup t = Q tile t
        asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
        const int t = (warp - 4) >> 2;
        const int quad = warp % 4;
        const int r = quad * 32 + lane;          // query row within tile t
        const int qi = q0 + t * BQ + r;          // query index within the sequence
        const int n_t = t ? n1 : n0;
        const unsigned lane_base = static_cast<unsigned>(quad * 32) << 16;
        const unsigned t_s = tmem + lane_base + t * 128, t_o = tmem + lane_base + 256 + t * 128;
        const float sl2 = g.scale_log2;
        float m = -INFINITY, l0 = 0.f, l1 = 0.f;  // running max (scaled, log2 units), two partial row sums
        for (int j = 0; j < n_t; ++j) {
            mbar_wait(&s_full[t], j & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            unsigned v[128];
            TM_LD32(t_s + 0, (v + 0));
            TM_LD32(t_s + 32, (v + 32));
            TM_LD32(t_s + 64, (v + 64));
            TM_LD32(t_s + 96, (v + 96));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            // keys e <= lim are visible to this query (causal + sequence end)
            const int lim = min(qi, it.seq_len - 1) - j * BKV;
            if (lim < BKV - 1) {
#pragma unroll
                for (int e = 0; e < 128; ++e)
                    if (e > lim) v[e] = __float_as_uint(-INFINITY);
            }
            // row max: 8 independent chains of 3-input max (short dependency chains)
            float mxa[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) mxa[k] = -INFINITY;
#pragma unroll
            for (int e = 0; e < 128; e += 16) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mxa[k] = fmax3(mxa[k], __uint_as_float(v[e + 2 * k]), __uint_as_float(v[e + 2 * k + 1]));
            }
            float mx = fmax3(fmax3(mxa[0], mxa[1], mxa[2]), fmax3(mxa[3], mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7]));
            mx *= sl2;  // scale > 0: max commutes with the scaling
            float m_new = m;
            if (mx > m + kRescaleThreshold || m == -INFINITY) m_new = fmaxf(mx, m);
            // lazy rescale of O_t (PV_t of j-1 completed before S_t of j). tcgen05.ld/st are
            // warp-collective (.sync.aligned): the decision is a warp vote, rows whose max did
            // not move rescale by 1
            if (__any_sync(0xffffffffu, j > 0 && m_new != m)) {
                const float alpha = m_new != m ? ex2(m - m_new) : 1.f;
                l0 *= alpha;
                l1 *= alpha;
#pragma unroll 1
                for (int c = 0; c < HD; c += 32) {
                    unsigned o[32];
                    TM_LD32(t_o + c, o);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                    TM_ST32(t_o + c, o);
                }
            }
            m = m_new;
            const float mm = (m == -INFINITY) ? 0.f : m;
            // p = exp2(s*scale*log2e - m) -> bf16 pairs, packed in place into v[0..63]
            // one pair in four goes through the FMA-pipe exp2 so MUFU is not the bottleneck
            const float2 v_sl2 = make_float2(sl2, sl2), v_nm = make_float2(-mm, -mm);
            float2 acc[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = make_float2(0.f, 0.f);
#pragma unroll
            for (int e = 0; e < 128; e += 2) {
                const float2 x = ffma2(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), v_sl2, v_nm);
                const float2 p = ((e >> 1) & 3) == 3 ? ex2_fma2(x) : make_float2(ex2(x.x), ex2(x.y));
                acc[(e >> 1) & 3] = fadd2(acc[(e >> 1) & 3], p);
                v[e / 2] = pack_bf16(p.x, p.y);
            }
            const float2 acc01 = fadd2(acc[0], acc[1]), acc23 = fadd2(acc[2], acc[3]);
            l0 += acc01.x + acc23.x;
            l1 += acc01.y + acc23.y;
            TM_ST32(t_s + 0, (v + 0));
            TM_ST32(t_s + 32, (v + 32));
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[t]);
        }
        // epilogue: O_t / l -> bf16, LSE
        mbar_wait(&o_done[t], 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float l = l0 + l1;
        const bool valid = qi < it.seq_len;
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const long long tok = static_cast<long long>(it.seq_start) + qi;
        __nv_bfloat16* orow = g.out + (tok * g.H + it.head) * HD;
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
            unsigned v[32];
            TM_LD32(t_o + c, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (valid) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4 o;
                    o.x = pack_bf16(__uint_as_float(v[8 * q]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
                    o.y = pack_bf16(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
                    o.z = pack_bf16(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
                    o.w = pack_bf16(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
                    *reinterpret_cast<uint4*>(orow + c + 8 * q) = o;
                }
            }
        }
        if (valid) g.lse[static_cast<long long>(it.head) * g.T + tok] = (m + log2f(l)) / kLog2e;  // natural log
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// ======================================================================
// Backward. One CTA per (sequence, 128-key tile j, kv head): K_j and V_j stay
// in smem, dK_j / dV_j accumulate in TMEM over every query head of the GQA
// group and every query tile i >= j (causal), so they are written once, with
// no atomics. Per (head, i):
//   MMA  S = Q_i K_j^T, dP = dO_i V_j^T                      (TMEM S, dP)
//   SM   P = exp(scale*S - lse), dS = scale * P * (dP - D)    (bf16 -> smem)
//   MMA  dV += P^T dO_i, dK += dS^T Q_i  (A operands MN-major: P / dS stored
//        [q][key] are read transposed in place), dQ_i = dS K_j (into dP's cols)
//   SM   dQ_i rows -> red.global.add.v4.f32 into the fp32 dQ accumulator,
//        overlapping the next S = Q K^T (dP waits for the read-out)
// D = rowsum(dO * O) comes from attn_bwd_prep_kernel; dq_convert makes bf16.
// TMEM: dV [0,128) dK [128,256) S [256,384) dP/dQ [384,512).
// A backward work item: key tile kv_tile of one sequence for one kv head,
// iterations [it_begin, it_end) of the (query head of the group, query tile
// i >= kv_tile) loop. Long causal loops are split into several items so the
// grid load-balances; their dK / dV partials meet in fp32 accumulators.
struct BwdItem {
    int seq_start, seq_len, kv_tile, kv_head, it_begin, it_end, pad0, pad1;
};

struct BwdArgs {
    const BwdItem* items;
    int H, KV;
    float scale, scale_log2;
    const float* lse;  // [H][T]
    const float* D;    // [H][T]
    float* dq_acc;     // [T][H][HD] fp32
    float* dk_acc;     // [T][KV][HD] fp32
    float* dv_acc;
    long long T;
};

__device__ __forceinline__ void store_swizzled(char* tile, int r, int c, const unsigned* pk) {
    // 32 bf16 of row r, columns [c, c+32) of a [128][128] K-major SW128 tile (two 64-column halves)
    char* half = tile + (c >> 6) * (kTile / 2) + r * 128;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int chunk = ((c & 63) >> 3) + q;
        sts128(half + ((chunk ^ (r & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    }
}

// warp 0 TMA, warp 1 MMA (warpgroup 0, registers given away with setmaxnreg), warps 4.. elementwise:
// kEwWg warpgroups, each owning kCpt of the 128 columns and covering the four TMEM lane quadrants
#ifndef ODC_BWD_EW_WG
#define ODC_BWD_EW_WG 2
#endif
constexpr int kEwWg = ODC_BWD_EW_WG;
constexpr int kCpt = 128 / kEwWg;  // columns per elementwise thread
constexpr int kBwdThreads = 128 + 128 * kEwWg;
constexpr int kEwRegs = kEwWg == 2 ? 208 : 104;  // setmaxnreg of the elementwise warpgroups
constexpr int kProdRegs = kEwWg == 2 ? 88 : 56;  // ... and of the TMA / MMA warpgroup
constexpr int kBwdSmem = kTile * 7 + 1024;  // K, V, Q x2, dO, P, dS
static_assert(kEwWg == 2 || kEwWg == 4, "2 or 4 elementwise warpgroups");

__device__ __forceinline__ void bar_ew() {  // named barrier over the elementwise warps
    asm volatile("bar.sync 1, %0;" ::"n"(128 * kEwWg) : "memory");
}
__device__ __forceinline__ void tma_reduce_add(const CUtensorMap* map, const void* smem, int c0, int c1) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
                 "r"(c0), "r"(c1), "r"(su32(smem))
                 : "memory");
}
// 64 fp32 columns [c0, c0+64) of row r into an fp32 staging tile made of four [128 rows][32 fp32] 128B-swizzled
// chunks (the box layout of an f32 tensor map with SWIZZLE_128B): conflict-free 16-B stores.
template <int NCH = 2>
__device__ __forceinline__ void stage_f32(char* stage, int r, int c0, const unsigned* v) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        char* row = stage + ((c0 >> 5) + k) * (kTile / 2) + r * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            sts128(row + ((q ^ (r & 7)) << 4), v[32 * k + 4 * q], v[32 * k + 4 * q + 1], v[32 * k + 4 * q + 2],
                   v[32 * k + 4 * q + 3]);
    }
}

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_do,
                    const __grid_constant__ CUtensorMap map_dq, const __grid_constant__ CUtensorMap map_dk,
                    const __grid_constant__ CUtensorMap map_dv, BwdArgs g) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    char* sK = smem;
    char* sV = smem + kTile;
    char* sQ0 = smem + 2 * kTile;  // Q double-buffered (sQ0 + b * kTile): Q_{n+1} lands while n computes
    char* sdO = smem + 4 * kTile;
    char* sP = smem + 5 * kTile;
    char* sdS = smem + 6 * kTile;
    char* stage = sP;  // [sP, sdS] = 64 KB fp32 staging of dQ_n once every MMA of n is done
    // sdp_full: S_n and dP_n in TMEM; ds_full: P_n / dS_n in smem (S_n, dP_n consumed);
    // dq_full: every MMA of n done (dQ_n in the dP columns); dq_read: dQ_n read out
    // s_read: S_n, dP_n are in the elementwise warps' registers (S columns free for S_{n+1})
    // p_full: P_n in smem (dV_n may start; the dS store may still wait for the dQ staging drain)
    // dk_done: dK_n finished reading dS_n (warpgroup 1 may stage its dQ half into sdS)
    __shared__ __align__(8) unsigned long long kv_full, q_full[2], q_empty[2], do_full, do_empty, sdp_full, s_read,
        p_full, ds_full, dq_full, dq_read, dk_done;
    __shared__ unsigned tmem_base;

    const BwdItem it = g.items[blockIdx.x];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int j = it.kv_tile;  // key tile
    const int kvh = it.kv_head;
    const int G = g.H / g.KV;
    const int n_q = (it.seq_len + BQ - 1) / BQ;
    const int per_head = n_q - j;  // query tiles i = j .. n_q-1 for each head of the group
    const int n0 = it.it_begin;
    const int n_iter = it.it_end - it.it_begin;

    if (warp == 0 && lane == 0) {
        mbar_init(&kv_full, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&q_full[b], 1);
            mbar_init(&q_empty[b], 1);
        }
        mbar_init(&do_full, 1);
        mbar_init(&do_empty, 1);
        mbar_init(&sdp_full, 1);
        mbar_init(&s_read, 4 * kEwWg);
#ifdef ODC_ATTN_DEBUG
        if (blockIdx.x == 0)
            printf("bars: kv_full %x q_full %x %x q_empty %x %x do_full %x do_empty %x sdp_full %x s_read %x ds_full %x "
                   "dq_full %x dq_read %x n_iter %d\n",
                   su32(&kv_full), su32(&q_full[0]), su32(&q_full[1]), su32(&q_empty[0]), su32(&q_empty[1]),
                   su32(&do_full), su32(&do_empty), su32(&sdp_full), su32(&s_read), su32(&ds_full), su32(&dq_full),
                   su32(&dq_read), it.it_end - it.it_begin);
#endif
        mbar_init(&p_full, 4 * kEwWg);
        mbar_init(&dk_done, 1);
        mbar_init(&ds_full, 4 * kEwWg);
        mbar_init(&dq_full, 1);
        mbar_init(&dq_read, 4 * kEwWg);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base;
    const unsigned T_DV = 0, T_DK = 128, T_S = 256, T_DP = 384;  // dQ_n reuses T_DP

    if (warp < 4) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs) : "memory");
      if (warp == 0) {
        if (lane == 0) {  // ---- TMA
            const int k0 = it.seq_start + j * BKV;
            mbar_expect_tx(&kv_full, 2 * kTile);
            tma_2d(&map_k, &kv_full, sK, kvh * HD, k0);
            tma_2d(&map_k, &kv_full, sK + kTile / 2, kvh * HD + 64, k0);
            tma_2d(&map_v, &kv_full, sV, kvh * HD, k0);
            tma_2d(&map_v, &kv_full, sV + kTile / 2, kvh * HD + 64, k0);
            for (int n = 0; n < n_iter; ++n) {
                const int h = kvh * G + (n0 + n) / per_head, i = j + (n0 + n) % per_head;
                const int q0 = it.seq_start + i * BQ, b = n & 1;
                if (n >= 2) mbar_wait(&q_empty[b], ((n >> 1) - 1) & 1);  // Q_{n-2} consumed by dK_{n-2}
                mbar_expect_tx(&q_full[b], kTile);
                tma_2d(&map_q, &q_full[b], sQ0 + b * kTile, h * HD, q0);
                tma_2d(&map_q, &q_full[b], sQ0 + b * kTile + kTile / 2, h * HD + 64, q0);
                if (n >= 1) mbar_wait(&do_empty, (n - 1) & 1);  // dO_{n-1} consumed by dV_{n-1}
                mbar_expect_tx(&do_full, kTile);
                tma_2d(&map_do, &do_full, sdO, h * HD, q0);
                tma_2d(&map_do, &do_full, sdO + kTile / 2, h * HD + 64, q0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            const unsigned id_kk = instr(0, 0), id_mm = instr(1, 1), id_km = instr(0, 1);
            mbar_wait(&kv_full, 0);
            const unsigned doa = su32(sdO), ka = su32(sK), va = su32(sV), pa = su32(sP), dsa = su32(sdS);
            auto issue_s = [&](int n) {  // S_n = Q_n K^T
                const int b = n & 1;
                const unsigned qa = su32(sQ0 + b * kTile);
                mbar_wait(&q_full[b], (n >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const unsigned off = (kk >> 2) * (kTile / 2) + (kk & 3) * 32;
                    mma(tmem + T_S, sdesc(qa + off, 16, 1024), sdesc(ka + off, 16, 1024), id_kk, kk > 0);
                }
            };
            issue_s(0);
            for (int n = 0; n < n_iter; ++n) {
                const int b = n & 1;
                const unsigned qa = su32(sQ0 + b * kTile);
                if (n > 0) mbar_wait(&dq_read, (n - 1) & 1);  // dP columns free again
                mbar_wait(&do_full, n & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                TR(0, n);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {  // dP = dO V^T
                    const unsigned off = (kk >> 2) * (kTile / 2) + (kk & 3) * 32;
                    mma(tmem + T_DP, sdesc(doa + off, 16, 1024), sdesc(va + off, 16, 1024), id_kk, kk > 0);
                }
                commit(&sdp_full);
                if (n + 1 < n_iter) {  // S_{n+1} overlaps the elementwise work of n once S_n is in registers
                    mbar_wait(&s_read, n & 1);
                    TR(1, n);
                    issue_s(n + 1);
                }
                mbar_wait(&p_full, n & 1);  // P in smem (dS may still be waiting for the staging drain)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                TR(2, n);
#pragma unroll
                for (int kk = 0; kk < BQ / 16; ++kk)  // K = query rows: MN-major A (P^T) and B (dO)
                    mma(tmem + T_DV, sdesc(pa + kk * 2048, kTile / 2, 1024), sdesc(doa + kk * 2048, kTile / 2, 1024),
                        id_mm, (n > 0 || kk > 0));
                commit(&do_empty);  // dO_n consumed: the TMA refills it while dK, dQ run
                mbar_wait(&ds_full, n & 1);  // dS in smem
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                TR(3, n);
                // dQ first: its read-out (and dP_{n+1}'s wait for it) overlaps dK
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {  // dQ = dS K into the dP columns
                    const unsigned aoff = (kk >> 2) * (kTile / 2) + (kk & 3) * 32;
                    mma(tmem + T_DP, sdesc(dsa + aoff, 16, 1024), sdesc(ka + kk * 2048, kTile / 2, 1024), id_km, kk > 0);
                }
                commit(&dq_full);  // also: P consumed (dV was issued before)
#pragma unroll
                for (int kk = 0; kk < BQ / 16; ++kk)  // dK += dS^T Q
                    mma(tmem + T_DK, sdesc(dsa + kk * 2048, kTile / 2, 1024), sdesc(qa + kk * 2048, kTile / 2, 1024),
                        id_mm, (n > 0 || kk > 0));
                commit(&q_empty[b]);
                commit(&dk_done);  // dS consumed
                TR(4, n);
            }
        }
      }
    } else {  // ---- elementwise / dQ / dK dV epilogue: row quadrant warp%4, column half
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEwRegs) : "memory");
#ifdef ODC_ATTN_DEBUG
        if (lane == 0 && blockIdx.x == 0) printf("ew warp %d start\n", warp);
#endif
        const int quad = warp % 4;
        const int wg = (warp - 4) >> 2;
        const int c0 = wg * kCpt;  // this warp's kCpt columns
        const bool first_half = wg < kEwWg / 2;  // stages its dQ part into sP (else into sdS, after dK)
        const bool lead = (warp & 3) == 0 && lane == 0;  // per warpgroup: issues its half's TMA reductions
        const int r = quad * 32 + lane;  // row: query within tile i (loop) / key within tile j (epilogue)
        const unsigned lane_base = static_cast<unsigned>(quad * 32) << 16;
        const float sl2 = g.scale_log2, sc = g.scale;
        auto stats = [&](int n, float& lse_raw, float& d_raw) {  // row statistics of iteration n (prefetched)
            const int h = kvh * G + (n0 + n) / per_head, i = j + (n0 + n) % per_head;
            const int qi = i * BQ + r;
            const long long idx = static_cast<long long>(h) * g.T + it.seq_start + qi;
            const bool ok = n < n_iter && qi < it.seq_len;
            lse_raw = ok ? __ldg(g.lse + idx) : 0.f;
            d_raw = ok ? __ldg(g.D + idx) : 0.f;
        };
        float lse_nx, d_nx;
        stats(0, lse_nx, d_nx);
        for (int n = 0; n < n_iter; ++n) {
            const int h = kvh * G + (n0 + n) / per_head, i = j + (n0 + n) % per_head;
            const int qi = i * BQ + r;  // query index within the sequence
            const bool q_ok = qi < it.seq_len;
            const float lse2 = lse_nx * kLog2e;
            const float Ds = d_nx * sc;
            stats(n + 1, lse_nx, d_nx);
            const int lim = q_ok ? min(qi, it.seq_len - 1) - j * BKV - c0 : -1;  // visible keys among our columns
            mbar_wait(&sdp_full, n & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lead && wg < 2) TR(5 + 8 * wg, n);
            unsigned sv[kCpt], dp[kCpt];
#pragma unroll
            for (int k = 0; k < kCpt / 32; ++k) {
                TM_LD32(tmem + lane_base + T_S + c0 + 32 * k, (sv + 32 * k));
                TM_LD32(tmem + lane_base + T_DP + c0 + 32 * k, (dp + 32 * k));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_read);
#ifdef ODC_ATTN_DEBUG
            if (lane == 0 && blockIdx.x == 0) printf("ew warp %d n %d s_read\n", warp, n);
#endif
            // P = exp2(S*scale*log2e - lse2) (0 where masked), dS = P * (dP*scale - D*scale); packed fp32x2
            // math, no mask work on tiles this row sees entirely. P first (kept in fp32 in sv, packed to pk),
            // stored and signalled so dV_n runs on the tensor pipe while dS is computed and stored.
            const float2 v_sl2 = make_float2(sl2, sl2), v_nlse = make_float2(-lse2, -lse2);
            const float2 v_sc = make_float2(sc, sc), v_nds = make_float2(-Ds, -Ds);
            unsigned pk[kCpt / 2];
            if (lim >= kCpt - 1) {
#pragma unroll
                for (int x = 0; x < kCpt; x += 2) {
                    const float2 t = ffma2(make_float2(__uint_as_float(sv[x]), __uint_as_float(sv[x + 1])), v_sl2, v_nlse);
                    const float2 pp = make_float2(ex2(t.x), ex2(t.y));
                    sv[x] = __float_as_uint(pp.x);
                    sv[x + 1] = __float_as_uint(pp.y);
                    pk[x / 2] = pack_bf16(pp.x, pp.y);
                }
            } else {
#pragma unroll
                for (int x = 0; x < kCpt; x += 2) {
                    const float2 t = ffma2(make_float2(__uint_as_float(sv[x]), __uint_as_float(sv[x + 1])), v_sl2, v_nlse);
                    const float2 pp = make_float2(x > lim ? 0.f : ex2(t.x), x + 1 > lim ? 0.f : ex2(t.y));
                    sv[x] = __float_as_uint(pp.x);
                    sv[x + 1] = __float_as_uint(pp.y);
                    pk[x / 2] = pack_bf16(pp.x, pp.y);
                }
            }
            // dQ_{n-1} was staged per warpgroup: warpgroup 0's half in sP, warpgroup 1's in sdS (each
            // lead committed its own bulk group). P waits for the sP half's read only, and dV_n runs
            // on P while the sdS half still drains into L2
            if (n > 0) {
                if (lead && first_half) {
                    if (wg == 0) TR(6, n);
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    if (wg == 0) TR(7, n);
                }
                bar_ew();
            }
#pragma unroll
            for (int k = 0; k < kCpt / 32; ++k) store_swizzled(sP, r, c0 + 32 * k, pk + 16 * k);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full);
            if (lead && wg < 2) TR(8 + 6 * wg, n);
#pragma unroll
            for (int x = 0; x < kCpt; x += 2) {
                const float2 u = ffma2(make_float2(__uint_as_float(dp[x]), __uint_as_float(dp[x + 1])), v_sc, v_nds);
                const float2 d = fmul2(make_float2(__uint_as_float(sv[x]), __uint_as_float(sv[x + 1])), u);
                dp[x / 2] = pack_bf16(d.x, d.y);
            }
            if (n > 0) {
                if (lead && !first_half) {
                    if (wg == 1) TR(15, n);
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    if (wg == 1) TR(16, n);
                }
                bar_ew();
            }
#pragma unroll
            for (int k = 0; k < kCpt / 32; ++k) store_swizzled(sdS, r, c0 + 32 * k, dp + 16 * k);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&ds_full);
            if (lead && wg < 2) TR(9 + 8 * wg, n);
            // dQ_n (fp32, already scaled) -> smem staging -> TMA reduce-add into the global accumulator,
            // while the MMA warp starts S_{n+1}
            mbar_wait(&dq_full, n & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lead && wg < 2) TR(10 + 8 * wg, n);
            unsigned v[kCpt];
#pragma unroll
            for (int k = 0; k < kCpt / 32; ++k) TM_LD32(tmem + lane_base + T_DP + c0 + 32 * k, (v + 32 * k));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&dq_read);
            // warpgroup 0's half goes to sP (free: dV_n read P before dQ_n), warpgroup 1's to sdS once
            // dK_n has read dS
            if (!first_half) mbar_wait(&dk_done, n & 1);
            if (lead && wg < 2) TR(11 + 8 * wg, n);
            stage_f32<kCpt / 32>(stage, r, c0, v);  // rows past the sequence end hold exact zeros (P = dS = 0)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync %0, 128;" ::"r"(2 + wg) : "memory");
            if (lead) {
                const int row0 = it.seq_start + i * BQ;
#pragma unroll
                for (int k = 0; k < kCpt / 32; ++k)
                    tma_reduce_add(&map_dq, stage + (c0 / 32 + k) * (kTile / 2), h * HD + c0 + 32 * k, row0);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                if (wg < 2) TR(12 + 8 * wg, n);
            }
        }
        // dK, dV of the key tile (every MMA done once the last dK finished) -> staging -> TMA reduce-add
        if (n_iter > 0) mbar_wait(&dk_done, (n_iter - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lead) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        bar_ew();
        char* st_dv = sP;  // [sP, sdS]
        char* st_dk = sQ0;  // both Q buffers: Q is no longer read
        {
            unsigned v[kCpt];
#pragma unroll
            for (int k = 0; k < kCpt / 32; ++k) TM_LD32(tmem + lane_base + T_DV + c0 + 32 * k, (v + 32 * k));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            stage_f32<kCpt / 32>(st_dv, r, c0, v);
#pragma unroll
            for (int k = 0; k < kCpt / 32; ++k) TM_LD32(tmem + lane_base + T_DK + c0 + 32 * k, (v + 32 * k));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            stage_f32<kCpt / 32>(st_dk, r, c0, v);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_ew();
        if (lead && wg == 0) {
            const int krow0 = it.seq_start + j * BKV;  // key rows past the sequence end hold exact zeros
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                tma_reduce_add(&map_dv, st_dv + k * (kTile / 2), kvh * HD + 32 * k, krow0);
                tma_reduce_add(&map_dk, st_dk + k * (kTile / 2), kvh * HD + 32 * k, krow0);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (lead) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// D[h][t] = sum_c dO[t][h][c] * O[t][h][c]; one warp per (t, h) row; also zeroes dq_acc rows
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                     float* __restrict__ D, float* __restrict__ dq_acc, long long T, int H) {
    const long long row = static_cast<long long>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (row >= T * H) return;
    const uint2 a = reinterpret_cast<const uint2*>(o + row * HD)[lane];
    const uint2 b = reinterpret_cast<const uint2*>(dout + row * HD)[lane];
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
    float acc = __low2float(a2[0]) * __low2float(b2[0]) + __high2float(a2[0]) * __high2float(b2[0]) +
                __low2float(a2[1]) * __low2float(b2[1]) + __high2float(a2[1]) * __high2float(b2[1]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    const long long t = row / H;
    const int h = static_cast<int>(row % H);
    if (lane == 0) D[static_cast<long long>(h) * T + t] = acc;
    reinterpret_cast<float4*>(dq_acc + row * HD)[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void dq_convert_kernel(const float4* __restrict__ acc, uint2* __restrict__ dq, long long n4) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float4 v = acc[i];
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
        dq[i] = make_uint2(*reinterpret_cast<unsigned*>(&a), *reinterpret_cast<unsigned*>(&b));
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap rows_map(const void* base, long long cols, long long rows) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw odcsim::ParamError("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

// fp32 [rows][cols] accumulator as the target of TMA reduce-add: box {32 fp32 = 128 B, 128 rows}, 128B swizzle
CUtensorMap f32_rows_map(void* base, long long cols, long long rows) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw odcsim::ParamError("cuTensorMapEncodeTiled (f32) failed (" + std::to_string(r) + ")");
    return m;
}

}  // namespace attn
}  // namespace odc

extern "C" odc_status odc_attn_fwd(const void* q, const void* k, const void* v, void* out, float* lse, const void* items,
                                   int n_items, std::int64_t T, int H, int KV, int head_dim, float scale, void* stream) {
    return odc::guard([&] {
        using namespace odc::attn;
        if (head_dim != HD) throw odcsim::ParamError("attn_fwd: head_dim must be 128");
        if (KV < 1 || H % KV) throw odcsim::ParamError("attn_fwd: H must be a multiple of KV");
        if (n_items <= 0) return;
        static thread_local int configured = -1;
        int dev = 0;
        cudaGetDevice(&dev);
        if (configured != dev) {
            cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
            if (e != cudaSuccess) throw std::runtime_error(std::string("attn smem attr: ") + cudaGetErrorString(e));
            configured = dev;
        }
        // q: [T][H*HD], k / v: [T][KV*HD] (the RoPE kernel's outputs)
        CUtensorMap mq = rows_map(q, static_cast<long long>(H) * HD, T);
        CUtensorMap mk = rows_map(k, static_cast<long long>(KV) * HD, T);
        CUtensorMap mv = rows_map(v, static_cast<long long>(KV) * HD, T);
        Args a{};
        a.items = static_cast<const Item*>(items);
        a.n_items = n_items;
        a.H = H;
        a.KV = KV;
        a.scale_log2 = scale * kLog2e;
        a.out = static_cast<__nv_bfloat16*>(out);
        a.lse = lse;
        a.T = T;
        odc::count_launch();
        attn_fwd_kernel<<<n_items, kFwdThreads, kFwdSmem, reinterpret_cast<cudaStream_t>(stream)>>>(mq, mk, mv, a);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(std::string("attn_fwd launch: ") + cudaGetErrorString(e));
    });
}

namespace odc {
namespace attn {

// fp32 dQ/dK/dV accumulators -> the packed qkv gradient [T][(H+2KV)*128] bf16 with the inverse
// RoPE applied to the q and k heads: dq_convert (x3) + qkv_rope_bwd in one pass. Each value is
// rounded to bf16 first, exactly as the two-kernel path stores dq/dk/dv, so the result is
// bit-identical to it (csrc/worker_kernels.cu qkv_rope_bwd_kernel).
__global__ void qkv_grad_kernel(const float* __restrict__ dq, const float* __restrict__ dk, const float* __restrict__ dv,
                                const float2* __restrict__ table, const long long* __restrict__ pos,
                                unsigned short* __restrict__ dqkv, long long T, int H, int KV) {
    constexpr int half = HD / 2, groups = half / 8;
    const int heads = H + 2 * KV;
    const long long total = T * heads * groups;
    for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int gi = static_cast<int>(idx % groups);
        const int h = static_cast<int>((idx / groups) % heads);
        const long long t = idx / (static_cast<long long>(groups) * heads);
        const float* src;
        if (h < H) src = dq + (t * H + h) * HD;
        else if (h < H + KV) src = dk + (t * KV + (h - H)) * HD;
        else src = dv + (t * KV + (h - H - KV)) * HD;
        float a[8], b[8];
#pragma unroll
        for (int q4 = 0; q4 < 2; ++q4) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(src + gi * 8) + q4);
            const float4 y = __ldg(reinterpret_cast<const float4*>(src + gi * 8 + half) + q4);
            const float xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // the bf16 the unfused path stores
                a[4 * q4 + e] = __bfloat162float(__float2bfloat16_rn(xs[e]));
                b[4 * q4 + e] = __bfloat162float(__float2bfloat16_rn(ys[e]));
            }
        }
        if (h < H + KV) {
            const float4* cs4 = reinterpret_cast<const float4*>(table + pos[t] * half + gi * 8);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                const float4 u = __ldg(cs4 + q4);
                const float c0 = u.x, s0 = u.y, c1 = u.z, s1 = u.w;
                const float y1 = a[2 * q4], y2 = b[2 * q4], z1 = a[2 * q4 + 1], z2 = b[2 * q4 + 1];
                a[2 * q4] = y1 * c0 + y2 * s0;
                b[2 * q4] = y2 * c0 - y1 * s0;
                a[2 * q4 + 1] = z1 * c1 + z2 * s1;
                b[2 * q4 + 1] = z2 * c1 - z1 * s1;
            }
        }
        const long long dst = t * heads * HD + static_cast<long long>(h) * HD + gi * 8;
        uint4 pa, pb;
        pa.x = pack_bf16(a[0], a[1]);
        pa.y = pack_bf16(a[2], a[3]);
        pa.z = pack_bf16(a[4], a[5]);
        pa.w = pack_bf16(a[6], a[7]);
        pb.x = pack_bf16(b[0], b[1]);
        pb.y = pack_bf16(b[2], b[3]);
        pb.z = pack_bf16(b[4], b[5]);
        pb.w = pack_bf16(b[6], b[7]);
        *reinterpret_cast<uint4*>(dqkv + dst) = pa;
        *reinterpret_cast<uint4*>(dqkv + dst + half) = pb;
    }
}

}  // namespace attn
}  // namespace odc

namespace {
// the backward up to the fp32 accumulators; returns (dq_acc, dk_acc, dv_acc) in the workspace
void attn_bwd_accumulate(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
                         void* workspace, const void* items, int n_items, std::int64_t T, int H, int KV, int head_dim,
                         float scale, cudaStream_t st, float** dq_out, float** dk_out, float** dv_out) {
    using namespace odc::attn;
    {
        if (head_dim != HD) throw odcsim::ParamError("attn_bwd: head_dim must be 128");
        if (KV < 1 || H % KV) throw odcsim::ParamError("attn_bwd: H must be a multiple of KV");
        static thread_local int configured = -1;
        int dev = 0;
        cudaGetDevice(&dev);
        if (configured != dev) {
            cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
            if (e != cudaSuccess) throw std::runtime_error(std::string("attn bwd smem attr: ") + cudaGetErrorString(e));
            configured = dev;
        }
        // workspace (fp32): D [H][T] | dq_acc [T][H][HD] | dk_acc, dv_acc [T][KV][HD]
        float* D = static_cast<float*>(workspace);
        float* dq_acc = D + (static_cast<long long>(H) * T + 63) / 64 * 64;  // keep the accumulators 256B-aligned
        float* dk_acc = dq_acc + T * H * HD;
        float* dv_acc = dk_acc + T * KV * HD;
        const long long rows = T * H;
        cudaError_t z = cudaMemsetAsync(dk_acc, 0, static_cast<size_t>(2 * T * KV * HD) * 4, st);
        if (z != cudaSuccess) throw std::runtime_error(std::string("attn_bwd zero: ") + cudaGetErrorString(z));
        odc::count_launch();
        attn_bwd_prep_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(
            static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), D, dq_acc, T, H);
        // zero dK / dV rows no key tile writes (tokens past every sequence end never exist here; all rows covered)
        if (n_items > 0) {
            CUtensorMap mq = rows_map(q, static_cast<long long>(H) * HD, T);
            CUtensorMap mk = rows_map(k, static_cast<long long>(KV) * HD, T);
            CUtensorMap mv = rows_map(v, static_cast<long long>(KV) * HD, T);
            CUtensorMap mdo = rows_map(dout, static_cast<long long>(H) * HD, T);
            CUtensorMap mdq = f32_rows_map(dq_acc, static_cast<long long>(H) * HD, T);
            CUtensorMap mdk = f32_rows_map(dk_acc, static_cast<long long>(KV) * HD, T);
            CUtensorMap mdv = f32_rows_map(dv_acc, static_cast<long long>(KV) * HD, T);
            BwdArgs a{};
            a.items = static_cast<const BwdItem*>(items);
            a.H = H;
            a.KV = KV;
            a.scale = scale;
            a.scale_log2 = scale * kLog2e;
            a.lse = lse;
            a.D = D;
            a.dq_acc = dq_acc;
            a.dk_acc = dk_acc;
            a.dv_acc = dv_acc;
            a.T = T;
            odc::count_launch();
            attn_bwd_kernel<<<n_items, kBwdThreads, kBwdSmem, st>>>(mq, mk, mv, mdo, mdq, mdk, mdv, a);
        }
        *dq_out = dq_acc;
        *dk_out = dk_acc;
        *dv_out = dv_acc;
    }
}
}  // namespace

#ifdef ODC_ATTN_TRACE
extern "C" int odc_attn_trace_read(unsigned long long* dst) {
    return cudaMemcpyFromSymbol(dst, odc::attn::g_attn_trace, sizeof(odc::attn::g_attn_trace)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" odc_status odc_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                                   const float* lse, void* dq, void* dk, void* dv, void* workspace,
                                   const void* items, int n_items, std::int64_t T, int H, int KV, int head_dim,
                                   float scale, void* stream) {
    return odc::guard([&] {
        using namespace odc::attn;
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        float *dq_acc, *dk_acc, *dv_acc;
        attn_bwd_accumulate(q, k, v, o, dout, lse, workspace, items, n_items, T, H, KV, head_dim, scale, st, &dq_acc,
                            &dk_acc, &dv_acc);
        auto convert = [&](const float* acc, void* out, long long n) {
            odc::count_launch();
            const long long n4 = n / 4;
            dq_convert_kernel<<<static_cast<unsigned>(std::min<long long>((n4 + 255) / 256, 148 * 8)), 256, 0, st>>>(
                reinterpret_cast<const float4*>(acc), static_cast<uint2*>(out), n4);
        };
        convert(dq_acc, dq, T * H * HD);
        convert(dk_acc, dk, T * KV * HD);
        convert(dv_acc, dv, T * KV * HD);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(std::string("attn_bwd launch: ") + cudaGetErrorString(e));
    });
}

extern "C" odc_status odc_attn_bwd_qkv(const void* q, const void* k, const void* v, const void* o, const void* dout,
                                       const float* lse, const void* table, const int64_t* pos, void* dqkv,
                                       void* workspace, const void* items, int n_items, std::int64_t T, int H, int KV,
                                       int head_dim, float scale, void* stream) {
    return odc::guard([&] {
        using namespace odc::attn;
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        float *dq_acc, *dk_acc, *dv_acc;
        attn_bwd_accumulate(q, k, v, o, dout, lse, workspace, items, n_items, T, H, KV, head_dim, scale, st, &dq_acc,
                            &dk_acc, &dv_acc);
        const long long n = T * (H + 2 * KV) * (HD / 16);
        odc::count_launch();
        qkv_grad_kernel<<<static_cast<unsigned>(std::min<long long>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(
            dq_acc, dk_acc, dv_acc, static_cast<const float2*>(table), reinterpret_cast<const long long*>(pos),
            static_cast<unsigned short*>(dqkv), T, H, KV);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(std::string("attn_bwd_qkv launch: ") + cudaGetErrorString(e));
    });
}
