// gemm.cu — bf16 GEMM on the 5th-generation tensor cores (tcgen05) for the
// worker's dense layers (fwd X·Wᵀ, dgrad dY·W, wgrad dYᵀ·X). No reference
// counterpart (the reference only has the cost model, src/cost_model.cpp:14-18).
//
//   D[M,N] (+)= A·Bᵀ,  A: [M][K] (K-major) or [K][M] (M-major)
//                      B: [N][K] (K-major) or [K][N] (N-major)
//
// Structure (one 128 x BN output tile per CTA, warp-specialised):
//   warp 0       TMA producer: 2D tensor-map loads (128B swizzle) of the A/B
//                k-slices into a kStages-deep smem ring (mbarrier full/empty)
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer
//                (kind::f16, M=128, N=BN, K=16 per instruction, fp32 accum in
//                TMEM); tcgen05.commit releases smem stages / signals epilogue
//   warps 2..5   epilogue: tcgen05.ld 32x32b TMEM -> registers -> bf16/fp32
//                vector stores (each warp owns its TMEM lane quadrant)
// Operand majorness is handled entirely by the UMMA smem descriptors and the
// TMA boxes (K-major: box {64 K, rows}; MN-major: boxes {64 MN, 64 K}), so no
// operand is ever transposed in memory.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "common.hpp"
#include "kernels.cuh"

namespace odc {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int kThreads = 192;

template <int BN>
struct Cfg {
    static constexpr int kStages = BN == 256 ? 4 : 6;
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kSmem = kStages * kStageBytes + 1024;  // + alignment slack
    static constexpr int kTmemCols = BN;                         // fp32 accumulator columns
};

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, unsigned long long* bar, void* smem, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(smem)),
        "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_128B, sm100 version bits = 1
__device__ __forceinline__ std::uint64_t smem_desc(unsigned addr, unsigned lbo, unsigned sbo) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((addr & 0x3FFFF) >> 4);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version
    d |= 2ull << 61;  // layout: SWIZZLE_128B
    return d;
}

// instruction descriptor: bf16 x bf16 -> f32, M=128, N=BN
__host__ __device__ constexpr unsigned instr_desc(int bn, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<unsigned>(a_mn_major) << 15) |
           (static_cast<unsigned>(b_mn_major) << 16) | (static_cast<unsigned>(bn >> 3) << 17) |
           (static_cast<unsigned>(BM >> 4) << 24);
}

struct Args {
    void* D;
    const void* C;  // optional bf16 residual: D = A·Bᵀ + C (same shape / ldd as D)
    long long M, N, K, ldd;
    int d_f32, accumulate;
    int a_mn, b_mn;  // 1 = MN-major operand
    int tiles_m, tiles_n;
    int splits;  // split-K factor (fp32 output only): partial tiles are red.add-ed into D
    int group;   // raster: M-tiles per group (N swept inside a group); see raster_group()
    // fused SwiGLU (gate_up projection, 2-CTA kernel only): B = [gate; up] (2*ffn rows); output tile n
    // pairs gate rows [128n, 128n+128) (leader CTA's B half) with up rows ffn + [128n, 128n+128) (peer's),
    // so one TMEM row holds g and u of the same 128 ffn columns. D = gu [M][2*ffn] as unfused,
    // glu_m = silu(g) * u [M][ffn] (from the bf16-rounded g, u: bit-identical to swiglu_fwd)
    void* glu_m;
    int ffn;
};

// Tile raster (L2 reuse). Tiles are walked in groups of `group` M-tiles, the
// N-tiles swept inside a group, so the group's A rows stay in L2 while B
// streams past; B is then read tiles_m / group times from DRAM. group = 1 is
// row-major (B reused from L2 by every M-tile: right when all of B fits in L2,
// e.g. the 27.5 MB down-proj weight), group = tiles_m is column-major (A
// resident). Otherwise the group is sized so its A rows take ~budget bytes of
// L2 (the gate_up weight, 55 MB, is then read ~3x at 32K tokens instead of
// 16x with a fixed group of 8). ODC_GEMM_GROUP forces a group,
// ODC_GEMM_L2_MB sets the budget (default 40 MB of the 126 MB L2).
// process-wide raster settings (ODC_GEMM_GROUP / ODC_GEMM_L2_MB at first use;
// odc_gemm_set_raster overrides them, for interleaved A/B timing)
inline std::atomic<int>& raster_forced() {
    static std::atomic<int> v{[] {
        const char* e = std::getenv("ODC_GEMM_GROUP");
        return e ? std::atoi(e) : 0;
    }()};
    return v;
}
inline std::atomic<long long>& raster_budget() {
    static std::atomic<long long> v{[] {
        const char* e = std::getenv("ODC_GEMM_L2_MB");
        return (e ? std::atoll(e) : 40LL) << 20;
    }()};
    return v;
}
inline int raster_group(long long K, int tiles_m, int tiles_n, int tile_rows_a, int tile_rows_b) {
    const int forced = raster_forced().load(std::memory_order_relaxed);
    const long long budget = raster_budget().load(std::memory_order_relaxed);
    if (forced > 0) return forced < tiles_m ? forced : tiles_m;
    const long long a_tile = static_cast<long long>(tile_rows_a) * K * 2, b_tile = static_cast<long long>(tile_rows_b) * K * 2;
    if (b_tile * tiles_n <= budget) return 1;
    if (a_tile * tiles_m <= budget) return tiles_m;
    long long g = budget / a_tile;
    if (g < 8) g = 8;
    return static_cast<int>(g < tiles_m ? g : tiles_m);
}

template <int BN>
__device__ __forceinline__ void tile_coords(int tile, const Args& g, int& m0, int& n0) {
    // grouped rasterisation (raster_group): `group` M-tiles share the same N-tiles for L2 reuse
    const int group = g.group;
    const int per_group = group * g.tiles_n;
    const int gid = tile / per_group, first_m = gid * group;
    const int gsize = min(group, g.tiles_m - first_m);
    m0 = (first_m + (tile % per_group) % gsize) * BM;
    n0 = ((tile % per_group) / gsize) * BN;
}

// Persistent: each CTA walks tiles blockIdx.x, +gridDim.x, ... The TMEM
// accumulator is double-buffered (2 x BN fp32 columns), so the epilogue of
// tile i (warps 2..5) overlaps the MMAs of tile i+1 (warp 1) while warp 0
// keeps the smem ring full across tile boundaries.
template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, Args g) {
    using C = Cfg<BN>;
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) unsigned long long full_bar[C::kStages], empty_bar[C::kStages];
    __shared__ __align__(8) unsigned long long tmem_full[2], tmem_empty[2];
    __shared__ unsigned tmem_base;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int num_items = g.tiles_m * g.tiles_n * g.splits;
    const int k_tiles = static_cast<int>((g.K + BK - 1) / BK);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 4);  // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                     "n"(2 * C::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            int it = 0;
            for (int w = blockIdx.x; w < num_items; w += gridDim.x) {
                int m0, n0;
                tile_coords<BN>(w / g.splits, g, m0, n0);
                const int sp = w % g.splits;
                const int kb = k_tiles * sp / g.splits, ke = k_tiles * (sp + 1) / g.splits;
                for (int kt = kb; kt < ke; ++kt, ++it) {
                    const int s = it % C::kStages;
                    if (it >= C::kStages) mbar_wait(&empty_bar[s], ((it / C::kStages) - 1) & 1);
                    char* sa = smem + s * C::kStageBytes;
                    char* sb = sa + C::kABytes;
                    mbar_expect_tx(&full_bar[s], C::kStageBytes);
                    const int k0 = kt * BK;
                    if (!g.a_mn) {
                        tma_load_2d(&map_a, &full_bar[s], sa, k0, m0);
                    } else {
                        tma_load_2d(&map_a, &full_bar[s], sa, m0, k0);
                        tma_load_2d(&map_a, &full_bar[s], sa + 64 * BK * 2, m0 + 64, k0);
                    }
                    if (!g.b_mn) {
                        tma_load_2d(&map_b, &full_bar[s], sb, k0, n0);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            tma_load_2d(&map_b, &full_bar[s], sb + j * 64 * BK * 2, n0 + 64 * j, k0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            const unsigned idesc = instr_desc(BN, g.a_mn, g.b_mn);
            // K-major: rows of 128 B, 8-row atoms 1024 B apart (SBO), k-step +32 B
            // MN-major: 64-element MN runs, 8-k-row atoms 1024 B apart (SBO),
            //           next 64 MN at LBO = BK*128 B, k-step +2048 B
            const unsigned a_lbo = g.a_mn ? BK * 128 : 16, b_lbo = g.b_mn ? BK * 128 : 16;
            const unsigned a_step = g.a_mn ? 2048 : 32, b_step = g.b_mn ? 2048 : 32;
            int it = 0, j = 0;
            for (int w = blockIdx.x; w < num_items; w += gridDim.x, ++j) {
                const int sp = w % g.splits;
                const int kb = k_tiles * sp / g.splits, ke = k_tiles * (sp + 1) / g.splits;
                const int acc = j & 1, use = j >> 1;
                if (use > 0) mbar_wait(&tmem_empty[acc], (use - 1) & 1);  // epilogue drained this buffer
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned d_tmem = tmem + static_cast<unsigned>(acc * BN);
                for (int kt = kb; kt < ke; ++kt, ++it) {
                    const int s = it % C::kStages;
                    mbar_wait(&full_bar[s], (it / C::kStages) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const unsigned sa = su32(smem + s * C::kStageBytes);
                    const unsigned sb = sa + C::kABytes;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        const std::uint64_t da = smem_desc(sa + kk * a_step, a_lbo, 1024);
                        const std::uint64_t db = smem_desc(sb + kk * b_step, b_lbo, 1024);
                        const unsigned accum = (kt > kb || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
                            "l"(da), "l"(db), "r"(idesc), "r"(accum)
                            : "memory");
                    }
                    // frees the smem stage once these MMAs have read it
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     su32(&empty_bar[s]))
                                 : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 su32(&tmem_full[acc]))
                             : "memory");
            }
        }
    } else {  // ---- epilogue warps 2..5
        const int quad = warp % 4;  // TMEM lane quadrant this warp may access
        int j = 0;
        for (int w = blockIdx.x; w < num_items; w += gridDim.x, ++j) {
            const int acc = j & 1, use = j >> 1;
            int m0, n0;
            tile_coords<BN>(w / g.splits, g, m0, n0);
            mbar_wait(&tmem_full[acc], use & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const long long row = m0 + quad * 32 + lane;
            const bool row_ok = row < g.M;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                unsigned r[32];
                const unsigned taddr =
                    tmem + (static_cast<unsigned>(quad * 32) << 16) + static_cast<unsigned>(acc * BN + c);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c + 32 >= BN) {  // whole accumulator now in registers: hand the buffer back early
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&tmem_empty[acc])) : "memory");
                }
                if (!row_ok) continue;
                const long long col0 = n0 + c;
                if (col0 >= g.N) continue;
                const bool full = col0 + 32 <= g.N;
                if (g.d_f32) {
                    float* out = static_cast<float*>(g.D) + row * g.ldd + col0;
                    if (g.splits > 1) {  // partial K range: reduce into D (zeroed or accumulated by the host)
                        if (full && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                            for (int q = 0; q < 32; q += 4)
                                asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(out + q), "f"(__uint_as_float(r[q])),
                                             "f"(__uint_as_float(r[q + 1])), "f"(__uint_as_float(r[q + 2])),
                                             "f"(__uint_as_float(r[q + 3]))
                                             : "memory");
                        } else {
                            for (int q = 0; q < 32 && col0 + q < g.N; ++q) atomicAdd(out + q, __uint_as_float(r[q]));
                        }
                    } else if (full && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < 32; q += 4) {
                            float4 v = make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]),
                                                   __uint_as_float(r[q + 2]), __uint_as_float(r[q + 3]));
                            if (g.accumulate) {
                                const float4 o = *reinterpret_cast<const float4*>(out + q);
                                v.x += o.x;
                                v.y += o.y;
                                v.z += o.z;
                                v.w += o.w;
                            }
                            *reinterpret_cast<float4*>(out + q) = v;
                        }
                    } else {
                        for (int q = 0; q < 32 && col0 + q < g.N; ++q)
                            out[q] = __uint_as_float(r[q]) + (g.accumulate ? out[q] : 0.f);
                    }
                } else {
                    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(g.D) + row * g.ldd + col0;
                    const __nv_bfloat16* add = g.C ? static_cast<const __nv_bfloat16*>(g.C) + row * g.ldd + col0
                                                   : (g.accumulate ? out : nullptr);
                    if (full && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < 32; q += 8) {
                            uint4 v, a4 = make_uint4(0, 0, 0, 0);
                            if (add) a4 = *reinterpret_cast<const uint4*>(add + q);
                            const unsigned* aw = reinterpret_cast<const unsigned*>(&a4);
                            unsigned* w = reinterpret_cast<unsigned*>(&v);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float lo = __uint_as_float(r[q + 2 * e]) + __uint_as_float(aw[e] << 16);
                                const float hi = __uint_as_float(r[q + 2 * e + 1]) + __uint_as_float(aw[e] & 0xffff0000u);
                                __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
                                w[e] = *reinterpret_cast<unsigned*>(&h);
                            }
                            *reinterpret_cast<uint4*>(out + q) = v;
                        }
                    } else {
                        for (int q = 0; q < 32 && col0 + q < g.N; ++q) {
                            float x = __uint_as_float(r[q]) + (add ? __bfloat162float(add[q]) : 0.f);
                            out[q] = __float2bfloat16_rn(x);
                        }
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * C::kTmemCols)
                     : "memory");
    }
}

// ------------------------------------------------------------------ host
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

// 2D bf16 tensor map: inner dim (contiguous) x outer dim, row pitch in elements
CUtensorMap make_map(const void* base, long long inner, long long outer, long long pitch, int box_inner, int box_outer) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw odcsim::ParamError("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

// ---------------------------------------------------------------- 2-CTA
// cta_group::2: a CTA pair (cluster of 2 on one TPC) computes a 256 x 256
// tile with M=256 UMMAs issued by the leader. Each CTA stages only its half of
// A (128 rows) and its half of B (128 of the 256 N rows) per k-slice, so per-
// SM smem traffic per MMA halves vs the 1-CTA 128 x 256 tile; each CTA's TMEM
// holds its 128 accumulator rows x 256 columns (double-buffered).
constexpr int kStages2 = 6;
constexpr int kHalfBytes = 128 * BK * 2;          // 16 KB: 128 rows x 64 bf16
constexpr int kStage2Bytes = 2 * kHalfBytes;      // A half + B half per CTA
constexpr int kSmem2 = kStages2 * kStage2Bytes + 1024;

__device__ __forceinline__ unsigned cta_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(const CUtensorMap* map, unsigned long long* bar, void* smem, int c0,
                                                int c1) {
    // both CTAs load into their own smem; transaction bytes land on the leader's barrier
    const unsigned mbar = su32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(su32(smem)),
        "l"(map), "r"(c0), "r"(c1), "r"(mbar)
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(unsigned taddr, unsigned* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
// Pins the registers of an asynchronous tcgen05.ld after its wait::ld: every use depends on this asm.
__device__ __forceinline__ void reg_fence32(unsigned* r) {
    asm volatile(""
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

// epilogue variants of the 2-CTA kernel, one instantiation each (a fused epilogue's registers
// never burden the plain GEMM)
enum Epi : int { kEpiPlain = 0, kEpiGluFwd = 1 };

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, Args g) {
    constexpr int BN2 = 256;
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) unsigned long long full_bar[kStages2], empty_bar[kStages2];
    __shared__ __align__(8) unsigned long long tmem_full[2], tmem_empty[2];
    __shared__ unsigned tmem_base;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const unsigned rank = cta_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x / 2, n_pairs = gridDim.x / 2;
    const int num_items = g.tiles_m * g.tiles_n * g.splits;  // 256 x 256 tiles x K splits
    const int k_tiles = static_cast<int>((g.K + BK - 1) / BK);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(&full_bar[s], 1);   // leader: one arrive.expect_tx for both CTAs' bytes
            mbar_init(&empty_bar[s], 1);  // one multicast commit per use
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 8);  // leader: 4 epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                     "n"(2 * BN2)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base;

    auto coords = [&](int tile, int& m0, int& n0) {
        const int group = g.group;
        const int per_group = group * g.tiles_n;
        const int gid = tile / per_group, first_m = gid * group;
        const int gsize = min(group, g.tiles_m - first_m);
        m0 = (first_m + (tile % per_group) % gsize) * 256;
        n0 = ((tile % per_group) / gsize) * BN2;
    };

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (both CTAs: own A half, own B half)
            int it = 0;
            for (int w = pair; w < num_items; w += n_pairs) {
                int m0, n0;
                coords(w / g.splits, m0, n0);
                const int sp = w % g.splits;
                const int kb = k_tiles * sp / g.splits, ke = k_tiles * (sp + 1) / g.splits;
                const int ma = m0 + static_cast<int>(rank) * 128;
                const int nb = EPI == kEpiGluFwd ? (rank ? g.ffn : 0) + n0 / 2 : n0 + static_cast<int>(rank) * 128;
                for (int kt = kb; kt < ke; ++kt, ++it) {
                    const int s = it % kStages2;
                    if (it >= kStages2) mbar_wait(&empty_bar[s], ((it / kStages2) - 1) & 1);
                    char* sa = smem + s * kStage2Bytes;
                    char* sb = sa + kHalfBytes;
                    if (leader) mbar_expect_tx(&full_bar[s], 2 * kStage2Bytes);
                    const int k0 = kt * BK;
                    if (!g.a_mn) {
                        tma_load_2d_2sm(&map_a, &full_bar[s], sa, k0, ma);
                    } else {
                        tma_load_2d_2sm(&map_a, &full_bar[s], sa, ma, k0);
                        tma_load_2d_2sm(&map_a, &full_bar[s], sa + 64 * BK * 2, ma + 64, k0);
                    }
                    if (!g.b_mn) {
                        tma_load_2d_2sm(&map_b, &full_bar[s], sb, k0, nb);
                    } else {
                        tma_load_2d_2sm(&map_b, &full_bar[s], sb, nb, k0);
                        tma_load_2d_2sm(&map_b, &full_bar[s], sb + 64 * BK * 2, nb + 64, k0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {  // ---- MMA issuer (leader only; M = 256 over both CTAs)
            const unsigned idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<unsigned>(g.a_mn) << 15) |
                                   (static_cast<unsigned>(g.b_mn) << 16) | (static_cast<unsigned>(BN2 >> 3) << 17) |
                                   (static_cast<unsigned>(256 >> 4) << 24);
            const unsigned a_lbo = g.a_mn ? BK * 128 : 16, b_lbo = g.b_mn ? BK * 128 : 16;
            const unsigned a_step = g.a_mn ? 2048 : 32, b_step = g.b_mn ? 2048 : 32;
            int it = 0, j = 0;
            for (int w = pair; w < num_items; w += n_pairs, ++j) {
                const int sp = w % g.splits;
                const int kb = k_tiles * sp / g.splits, ke = k_tiles * (sp + 1) / g.splits;
                const int acc = j & 1, use = j >> 1;
                if (use > 0) mbar_wait(&tmem_empty[acc], (use - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned d_tmem = tmem + static_cast<unsigned>(acc * BN2);
                for (int kt = kb; kt < ke; ++kt, ++it) {
                    const int s = it % kStages2;
                    mbar_wait(&full_bar[s], (it / kStages2) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const unsigned sa = su32(smem + s * kStage2Bytes);
                    const unsigned sb = sa + kHalfBytes;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        const std::uint64_t da = smem_desc(sa + kk * a_step, a_lbo, 1024);
                        const std::uint64_t db = smem_desc(sb + kk * b_step, b_lbo, 1024);
                        const unsigned accum = (kt > kb || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
                            "l"(da), "l"(db), "r"(idesc), "r"(accum)
                            : "memory");
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                        "%1;" ::"r"(su32(&empty_bar[s])),
                        "h"(static_cast<unsigned short>(3))
                        : "memory");
                }
                asm volatile(
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                        su32(&tmem_full[acc])),
                    "h"(static_cast<unsigned short>(3))
                    : "memory");
            }
        }
    } else {  // ---- epilogue warps 2..5: this CTA's 128 rows x 256 columns
        const int quad = warp % 4;
        unsigned leader_empty0;  // the leader CTA's tmem_empty[0] (tmem_empty[1] is 8 bytes above)
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(leader_empty0) : "r"(su32(&tmem_empty[0])));
        int j = 0;
        for (int w = pair; w < num_items; w += n_pairs, ++j) {
            const int acc = j & 1, use = j >> 1;
            int m0, n0;
            coords(w / g.splits, m0, n0);
            const long long row = m0 + static_cast<long long>(rank) * 128 + quad * 32 + lane;
            const bool row_ok = row < g.M;
            // fast path (bf16 output, whole 256-column row in range, 16-B aligned): the residual row is
            // prefetched into registers while the MMAs run, TMEM loads are double-buffered.
            __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(g.D) + row * g.ldd + n0;
            const __nv_bfloat16* arow = g.C ? static_cast<const __nv_bfloat16*>(g.C) + row * g.ldd + n0
                                            : (g.accumulate ? orow : nullptr);
            const bool fast = !g.d_f32 && n0 + BN2 <= g.N && (reinterpret_cast<uintptr_t>(orow) & 15) == 0 &&
                              (arow == nullptr || (reinterpret_cast<uintptr_t>(arow) & 15) == 0);
            if constexpr (EPI == kEpiGluFwd) {  // fused SwiGLU (host guarantees the fast-path conditions)
                mbar_wait(&tmem_full[acc], use & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned tbase = tmem + (static_cast<unsigned>(quad * 32) << 16) + static_cast<unsigned>(acc * BN2);
                __nv_bfloat16* grow = static_cast<__nv_bfloat16*>(g.D) + row * g.ldd + n0 / 2;
                __nv_bfloat16* urow = grow + g.ffn;
                __nv_bfloat16* mrow = static_cast<__nv_bfloat16*>(g.glu_m) + row * g.ffn + n0 / 2;
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    unsigned ra[32], rb[32];
                    tmem_ld32(tbase + c * 32, ra);        // gate columns
                    tmem_ld32(tbase + 128 + c * 32, rb);  // up columns
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    reg_fence32(ra);
                    reg_fence32(rb);
                    if (c == 3) {  // accumulator in registers: release the buffer to the leader's MMA
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0)
                            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                             leader_empty0 + 8u * acc)
                                         : "memory");
                    }
                    if (!row_ok) continue;
#pragma unroll
                    for (int q = 0; q < 32; q += 8) {
                        uint4 vg, vu, vm;
                        unsigned* wg = reinterpret_cast<unsigned*>(&vg);
                        unsigned* wu = reinterpret_cast<unsigned*>(&vu);
                        unsigned* wm = reinterpret_cast<unsigned*>(&vm);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            __nv_bfloat162 hg = __floats2bfloat162_rn(__uint_as_float(ra[q + 2 * e]), __uint_as_float(ra[q + 2 * e + 1]));
                            __nv_bfloat162 hu = __floats2bfloat162_rn(__uint_as_float(rb[q + 2 * e]), __uint_as_float(rb[q + 2 * e + 1]));
                            wg[e] = *reinterpret_cast<unsigned*>(&hg);
                            wu[e] = *reinterpret_cast<unsigned*>(&hu);
                            const float g0 = __low2float(hg), g1 = __high2float(hg);  // swiglu_fwd_kernel's formula
                            const float m0v = __fdividef(g0, 1.f + __expf(-g0)) * __low2float(hu);
                            const float m1v = __fdividef(g1, 1.f + __expf(-g1)) * __high2float(hu);
                            __nv_bfloat162 hm = __floats2bfloat162_rn(m0v, m1v);
                            wm[e] = *reinterpret_cast<unsigned*>(&hm);
                        }
                        *reinterpret_cast<uint4*>(grow + c * 32 + q) = vg;
                        *reinterpret_cast<uint4*>(urow + c * 32 + q) = vu;
                        *reinterpret_cast<uint4*>(mrow + c * 32 + q) = vm;
                    }
                }
                continue;
            }
            if (fast) {
                uint4 cb[BN2 / 8];
                if (arow && row_ok) {
#pragma unroll
                    for (int i = 0; i < BN2 / 8; ++i) cb[i] = __ldg(reinterpret_cast<const uint4*>(arow) + i);
                }
                mbar_wait(&tmem_full[acc], use & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned tbase = tmem + (static_cast<unsigned>(quad * 32) << 16) + static_cast<unsigned>(acc * BN2);
                unsigned ra[32], rb[32];
                tmem_ld32(tbase, ra);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                reg_fence32(ra);
#pragma unroll
                for (int c = 0; c < BN2 / 32; ++c) {
                    unsigned* cur = (c & 1) ? rb : ra;
                    unsigned* nxt = (c & 1) ? ra : rb;
                    if (c + 1 < BN2 / 32) tmem_ld32(tbase + (c + 1) * 32, nxt);
                    if (c + 1 == BN2 / 32) {  // last chunk in registers: release the buffer to the leader's MMA
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0)
                            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                             leader_empty0 + 8u * acc)
                                         : "memory");
                    }
                    if (row_ok) {
#pragma unroll
                        for (int q = 0; q < 32; q += 8) {
                            uint4 v;
                            const uint4 a4 = arow ? cb[c * 4 + q / 8] : make_uint4(0, 0, 0, 0);
                            const unsigned* aw = reinterpret_cast<const unsigned*>(&a4);
                            unsigned* w = reinterpret_cast<unsigned*>(&v);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float lo = __uint_as_float(cur[q + 2 * e]) + __uint_as_float(aw[e] << 16);
                                const float hi = __uint_as_float(cur[q + 2 * e + 1]) + __uint_as_float(aw[e] & 0xffff0000u);
                                __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
                                w[e] = *reinterpret_cast<unsigned*>(&h);
                            }
                            *reinterpret_cast<uint4*>(orow + c * 32 + q) = v;
                        }
                    }
                    if (c + 1 < BN2 / 32) {
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        reg_fence32(nxt);
                    }
                }
                continue;
            }
            mbar_wait(&tmem_full[acc], use & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int c = 0; c < BN2; c += 32) {
                unsigned r[32];
                const unsigned taddr =
                    tmem + (static_cast<unsigned>(quad * 32) << 16) + static_cast<unsigned>(acc * BN2 + c);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c + 32 >= BN2) {  // accumulator in registers: release the buffer to the leader's MMA
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_empty0 + 8u * acc)
                                     : "memory");
                }
                if (!row_ok) continue;
                const long long col0 = n0 + c;
                if (col0 >= g.N) continue;
                const bool full = col0 + 32 <= g.N;
                if (g.d_f32) {
                    float* out = static_cast<float*>(g.D) + row * g.ldd + col0;
                    if (g.splits > 1) {  // partial K range: reduce into D (zeroed or accumulated by the host)
                        if (full && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                            for (int q = 0; q < 32; q += 4)
                                asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(out + q), "f"(__uint_as_float(r[q])),
                                             "f"(__uint_as_float(r[q + 1])), "f"(__uint_as_float(r[q + 2])),
                                             "f"(__uint_as_float(r[q + 3]))
                                             : "memory");
                        } else {
                            for (int q = 0; q < 32 && col0 + q < g.N; ++q) atomicAdd(out + q, __uint_as_float(r[q]));
                        }
                    } else if (full && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < 32; q += 4) {
                            float4 v = make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]),
                                                   __uint_as_float(r[q + 2]), __uint_as_float(r[q + 3]));
                            if (g.accumulate) {
                                const float4 o = *reinterpret_cast<const float4*>(out + q);
                                v.x += o.x;
                                v.y += o.y;
                                v.z += o.z;
                                v.w += o.w;
                            }
                            *reinterpret_cast<float4*>(out + q) = v;
                        }
                    } else {
                        for (int q = 0; q < 32 && col0 + q < g.N; ++q)
                            out[q] = __uint_as_float(r[q]) + (g.accumulate ? out[q] : 0.f);
                    }
                } else {
                    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(g.D) + row * g.ldd + col0;
                    const __nv_bfloat16* add = g.C ? static_cast<const __nv_bfloat16*>(g.C) + row * g.ldd + col0
                                                   : (g.accumulate ? out : nullptr);
                    if (full && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < 32; q += 8) {
                            uint4 v, a4 = make_uint4(0, 0, 0, 0);
                            if (add) a4 = *reinterpret_cast<const uint4*>(add + q);
                            const unsigned* aw = reinterpret_cast<const unsigned*>(&a4);
                            unsigned* w = reinterpret_cast<unsigned*>(&v);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float lo = __uint_as_float(r[q + 2 * e]) + __uint_as_float(aw[e] << 16);
                                const float hi = __uint_as_float(r[q + 2 * e + 1]) + __uint_as_float(aw[e] & 0xffff0000u);
                                __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
                                w[e] = *reinterpret_cast<unsigned*>(&h);
                            }
                            *reinterpret_cast<uint4*>(out + q) = v;
                        }
                    } else {
                        for (int q = 0; q < 32 && col0 + q < g.N; ++q) {
                            float x = __uint_as_float(r[q]) + (add ? __bfloat162float(add[q]) : 0.f);
                            out[q] = __float2bfloat16_rn(x);
                        }
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync();  // the peer is done with our barriers / TMEM before dealloc
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN2) : "memory");
    }
}

cudaError_t launch2(const void* A, const void* B, Args g, long long lda, long long ldb, cudaStream_t s) {
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
        for (auto fn : {gemm2_kernel<kEpiPlain>, gemm2_kernel<kEpiGluFwd>}) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
            if (e != cudaSuccess) return e;
        }
        configured = dev;
    }
    // per CTA: A half = 128 rows (box 64 x 128 K-major / 2 boxes 64 x 64 MN-major), B half = 128 rows likewise
    CUtensorMap ma = g.a_mn ? make_map(A, g.M, g.K, lda, 64, BK) : make_map(A, g.K, g.M, lda, BK, 128);
    CUtensorMap mb = g.b_mn ? make_map(B, g.N, g.K, ldb, 64, BK) : make_map(B, g.K, g.N, ldb, BK, 128);
    static int sms = 0;
    if (!sms) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (const char* r = std::getenv("ODC_GEMM_RESERVE_SMS")) sms -= std::atoi(r);
        sms &= ~1;
        if (sms < 2) sms = 2;
    }
    g.tiles_m = static_cast<int>((g.M + 255) / 256);
    g.tiles_n = static_cast<int>((g.N + 255) / 256);
    g.group = raster_group(g.K, g.tiles_m, g.tiles_n, 256, 256);
    const int pairs = g.tiles_m * g.tiles_n * g.splits;
    const int grid = 2 * (pairs < sms / 2 ? pairs : sms / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem2;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    count_launch();
    if (g.glu_m) return cudaLaunchKernelEx(&cfg, gemm2_kernel<kEpiGluFwd>, ma, mb, g);
    return cudaLaunchKernelEx(&cfg, gemm2_kernel<kEpiPlain>, ma, mb, g);
}

template <int BN>
cudaError_t launch(const void* A, const void* B, const Args& g, long long lda, long long ldb, cudaStream_t s) {
    using C = Cfg<BN>;
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
        cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        configured = dev;
    }
    // A: K-major [M][K] (box 64 x 128) or M-major [K][M] (box 64 x 64)
    CUtensorMap ma = g.a_mn ? make_map(A, g.M, g.K, lda, 64, BK) : make_map(A, g.K, g.M, lda, BK, BM);
    CUtensorMap mb = g.b_mn ? make_map(B, g.N, g.K, ldb, 64, BK) : make_map(B, g.K, g.N, ldb, BK, BN);
    static int sms = 0;
    if (!sms) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (const char* r = std::getenv("ODC_GEMM_RESERVE_SMS")) sms -= std::atoi(r);  // leave SMs to comm kernels
        if (sms < 1) sms = 1;
    }
    const int tiles = g.tiles_m * g.tiles_n;
    const int items = tiles * g.splits;
    Args ga = g;
    ga.group = raster_group(g.K, g.tiles_m, g.tiles_n, BM, BN);
    count_launch();
    gemm_kernel<BN><<<items < sms ? items : sms, kThreads, C::kSmem, s>>>(ma, mb, ga);
    return cudaGetLastError();
}

}  // namespace gemm
}  // namespace odc

extern "C" odc_status odc_gemm_set_raster(int group, int l2_budget_mb) {
    return odc::guard([&] {
        if (group < 0 || l2_budget_mb < 0) throw odcsim::ParamError("raster: group and budget must be >= 0");
        odc::gemm::raster_forced().store(group);
        if (l2_budget_mb > 0) odc::gemm::raster_budget().store(static_cast<long long>(l2_budget_mb) << 20);
    });
}

extern "C" odc_status odc_gemm_gate_up_swiglu(const void* X, const void* W, void* gu, void* m, std::int64_t T,
                                               std::int64_t ffn, std::int64_t d, void* stream) {
    return odc::guard([&] {
        using odcsim::ParamError;
        if (T < 1 || ffn < 1 || d < 1) throw ParamError("gate_up: dims must be >= 1");
        if (ffn % 128 || d % 8) throw ParamError("gate_up: ffn must be a multiple of 128 and d of 8");
        if (reinterpret_cast<uintptr_t>(X) % 16 || reinterpret_cast<uintptr_t>(W) % 16 ||
            reinterpret_cast<uintptr_t>(gu) % 16 || reinterpret_cast<uintptr_t>(m) % 16)
            throw ParamError("gate_up: operands must be 16-byte aligned");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        if (T < 256 || std::getenv("ODC_GEMM_1CTA")) {  // below one 2-CTA tile: the unfused sm_100a pair
            const odc_status e = odc_gemm_bf16(X, W, gu, nullptr, T, 2 * ffn, d, d, d, 2 * ffn, 0, 0, ODC_BF16, 0, stream);
            if (e != ODC_OK) throw std::runtime_error(odc_last_error());
            const odc_status e2 = odc_w_swiglu_fwd(gu, m, T, static_cast<int>(ffn), stream);
            if (e2 != ODC_OK) throw std::runtime_error(odc_last_error());
            return;
        }
        odc::gemm::Args g{};
        g.D = gu;
        g.M = T;
        g.N = 2 * ffn;
        g.K = d;
        g.ldd = 2 * ffn;
        g.splits = 1;
        g.glu_m = m;
        g.ffn = static_cast<int>(ffn);
        const cudaError_t e = odc::gemm::launch2(X, W, g, d, d, st);
        if (e != cudaSuccess) throw std::runtime_error(std::string("gate_up launch: ") + cudaGetErrorString(e));
    });
}

extern "C" odc_status odc_gemm_bf16(const void* A, const void* B, void* D, const void* C, std::int64_t M,
                                    std::int64_t N, std::int64_t K, std::int64_t lda, std::int64_t ldb, std::int64_t ldd,
                                    int a_mn_major, int b_mn_major, int d_dtype, int accumulate, void* stream) {
    return odc::guard([&] {
        using odcsim::ParamError;
        if (M < 1 || N < 1 || K < 1) throw ParamError("gemm dims must be >= 1");
        if (d_dtype != ODC_BF16 && d_dtype != ODC_F32) throw ParamError("gemm output must be bf16 or f32");
        if ((lda * 2) % 16 || (ldb * 2) % 16) throw ParamError("gemm operand pitches must be multiples of 8 elements");
        if (reinterpret_cast<uintptr_t>(A) % 16 || reinterpret_cast<uintptr_t>(B) % 16)
            throw ParamError("gemm operands must be 16-byte aligned");
        odc::gemm::Args g{};
        if (C && d_dtype != ODC_BF16) throw ParamError("gemm residual C requires a bf16 output");
        g.D = D;
        g.C = C;
        g.M = M;
        g.N = N;
        g.K = K;
        g.ldd = ldd;
        g.d_f32 = d_dtype == ODC_F32;
        g.accumulate = accumulate;
        g.a_mn = a_mn_major ? 1 : 0;
        g.b_mn = b_mn_major ? 1 : 0;
        g.tiles_m = static_cast<int>((M + odc::gemm::BM - 1) / odc::gemm::BM);
        // split-K for fp32 outputs whose tile count cannot fill the GPU (wgrad of
        // d x d weights): partial tiles are reduced with red.global.add.v4.f32
        static const bool two_cta = !std::getenv("ODC_GEMM_1CTA");
        const bool use2 = two_cta && M >= 256 && N > 128;
        // split-K for fp32 outputs whose tile count cannot fill the GPU (wgrad of
        // d x d weights): partial tiles are reduced with red.global.add.v4.f32.
        // The factor maximises the fraction of (pair-)slots busy in the last wave.
        g.splits = 1;
        {
            const long long bm = use2 ? 256 : odc::gemm::BM, bn = (N <= 128 && !use2) ? 128 : 256;
            const long long tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
            const long long kt = (K + odc::gemm::BK - 1) / odc::gemm::BK;
            const long long slots = use2 ? 74 : 148;
            if (g.d_f32 && tiles * 10 < slots * 8 && kt >= 8) {
                double best = -1.0;
                for (long long sp = 1; sp <= 4 && sp <= kt / 4; ++sp) {
                    const long long items = tiles * sp, waves = (items + slots - 1) / slots;
                    const double eff = static_cast<double>(items) / static_cast<double>(waves * slots);
                    if (eff > best + 1e-9) {
                        best = eff;
                        g.splits = static_cast<int>(sp);
                    }
                }
            }
        }
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        if (g.splits > 1 && !accumulate) {
            cudaError_t z = cudaMemset2DAsync(D, static_cast<size_t>(ldd) * 4, 0, static_cast<size_t>(N) * 4,
                                              static_cast<size_t>(M), st);
            if (z != cudaSuccess) throw std::runtime_error(std::string("gemm split-K zero: ") + cudaGetErrorString(z));
        }
        cudaError_t e;
        if (use2) {
            e = odc::gemm::launch2(A, B, g, lda, ldb, st);
        } else if (N <= 128) {
            g.tiles_n = static_cast<int>((N + 127) / 128);
            e = odc::gemm::launch<128>(A, B, g, lda, ldb, st);
        } else {
            g.tiles_n = static_cast<int>((N + 255) / 256);
            e = odc::gemm::launch<256>(A, B, g, lda, ldb, st);
        }
        if (e != cudaSuccess) throw std::runtime_error(std::string("gemm launch: ") + cudaGetErrorString(e));
    });
}
