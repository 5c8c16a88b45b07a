// odc_kernels.cu — sm_100a kernels of the ODC hot path.
//
//   copy_segments   fetch (a3): N owner shards (peer HBM over NVLink + local)
//                   -> one full-layer buffer. 16-byte vector loads, UNROLL
//                   independent loads in flight per thread, chunked over a
//                   small CTA budget so fetch stays non-intrusive.
//                   replaces ShardState::gather inc/primitives.hpp:70-77
//   push_red        push (a6), RED mode: red.relaxed.sys.global.add.v4.f32
//                   straight into each owner's fp32 grad shard (NVLink).
//                   replaces split_gradient + try_stage + consume :80-136
//   push_bulk       push (a6) through TMA bulk ops into peer HBM: RED (fp32
//                   reductions into the owner's grad shard), SLOT (w*g stored,
//                   then added, into this client's slot AT THE OWNER),
//                   FIXED (int64 fixed-point reductions)
//   slot_reduce     SLOT mode owner reduce in fixed rank order (barrier step)
//   push_fixed      push (a6), FIXED mode: w*g rounded to int64 fixed point,
//                   TMA bulk .add.u64 reductions into the owner (deterministic
//                   in any order, 8 B per owned element); fixed_finalize
//                   converts back to fp32 at the barrier
//   barrier         (a8) finalize_minibatch :199-203 as sys-scope flags
//   adam            (a19) fused AdamW over owned shards, bf16 shard out
//   accumulate<T>   ShardState::consume :125-136 exactly (mul, then add)
//   red_accumulate<T> red.add.{u64,f64,f32} form of consume
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "kernels.cuh"

namespace odc {

namespace {
std::atomic<std::uint64_t> g_launches{0};
}
std::uint64_t launches() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

__host__ __device__ __forceinline__ std::int64_t i64min(std::int64_t a, std::int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ std::int64_t i64max(std::int64_t a, std::int64_t b) { return a > b ? a : b; }

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void red_sys_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void red_sys_f32(float* p, float a) {
    asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Bounded spin: returns false (and raises the error word) on timeout so a
// dead peer turns into ODC_ERR_TIMEOUT on the host instead of a hung GPU.
__device__ bool wait_geq(const unsigned long long* flag, unsigned long long need, unsigned long long* err,
                         long long timeout_ns) {
    if (ld_acquire_sys(flag) >= need) return true;
    const long long t0 = global_ns();
    unsigned ns = 32;
    while (true) {
        if (ld_acquire_sys(flag) >= need) return true;
        if (err && (*reinterpret_cast<volatile unsigned long long*>(err) & kErrTimeout)) return false;
        if (global_ns() - t0 > timeout_ns) {
            if (err) atomicOr(err, static_cast<unsigned long long>(kErrTimeout));
            return false;
        }
        __nanosleep(ns);
        if (ns < 1024) ns <<= 1;
    }
}

__device__ __forceinline__ float bf16_to_f32(unsigned short h) { return __uint_as_float(static_cast<unsigned>(h) << 16); }
__device__ __forceinline__ unsigned short f32_to_bf16(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// ------------------------------------------------------------ fetch / copy
constexpr int kCopyThreads = 512;
constexpr int kCopyUnroll = 8;
constexpr std::int64_t kChunkVec = kCopyThreads * kCopyUnroll;  // 4096 x 16 B = 64 KB per chunk

struct SegPlan {
    std::int64_t head, vecs, tail;  // bytes before the aligned body, 16B units, bytes after
    std::int64_t chunks;
    bool fast;
};

__device__ __forceinline__ SegPlan plan_seg(const char* src, const char* dst, std::int64_t bytes) {
    SegPlan p{};
    if (bytes <= 0) return p;
    const unsigned sa = static_cast<unsigned>(reinterpret_cast<uintptr_t>(src) & 15);
    const unsigned da = static_cast<unsigned>(reinterpret_cast<uintptr_t>(dst) & 15);
    p.fast = sa == da;
    if (p.fast) {
        p.head = i64min(bytes, (16 - da) & 15);
        p.vecs = (bytes - p.head) / 16;
        p.tail = bytes - p.head - p.vecs * 16;
        p.chunks = i64max(1, (p.vecs + kChunkVec - 1) / kChunkVec);
    } else {
        p.chunks = (bytes + kChunkVec * 16 - 1) / (kChunkVec * 16);
    }
    return p;
}

__global__ void __launch_bounds__(kCopyThreads) copy_segments_kernel(SegTable t) {
    __shared__ SegPlan plans[kMaxSeg];
    __shared__ std::int64_t first_chunk[kMaxSeg + 1];
    __shared__ int gate_ok;
    if (threadIdx.x == 0) {
        std::int64_t acc = 0;
        for (int i = 0; i < t.n; ++i) {
            plans[i] = plan_seg(t.src[i], t.dst[i], t.bytes[i]);
            first_chunk[i] = acc;
            acc += plans[i].chunks;
        }
        first_chunk[t.n] = acc;
    }
    __syncthreads();
    const std::int64_t total = first_chunk[t.n];
    int seg = 0;
    int gated_seg = -1;
    bool seg_ok = true;  // gate result of gated_seg, kept for the segment's later chunks
    for (std::int64_t c = blockIdx.x; c < total; c += gridDim.x) {
        while (c >= first_chunk[seg + 1]) ++seg;
        if (t.gate[seg]) {  // on-demand readiness of this owner's shard
            if (gated_seg != seg) {
                if (threadIdx.x == 0) gate_ok = wait_geq(t.gate[seg], t.need, t.err, t.timeout_ns);
                __syncthreads();
                seg_ok = gate_ok != 0;
                __syncthreads();  // gate_ok may be rewritten at the next segment switch
                gated_seg = seg;
            }
            if (!seg_ok) continue;  // a timed-out owner's chunks are never copied
        }
        const SegPlan p = plans[seg];
        const char* src = t.src[seg];
        char* dst = t.dst[seg];
        const std::int64_t j = c - first_chunk[seg];
        if (p.fast) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src + p.head);
            uint4* d4 = reinterpret_cast<uint4*>(dst + p.head);
            const std::int64_t beg = j * kChunkVec, end = i64min(p.vecs, beg + kChunkVec);
            std::int64_t i = beg + threadIdx.x;
            if (end - beg == kChunkVec) {
                uint4 r[kCopyUnroll];
#pragma unroll
                for (int u = 0; u < kCopyUnroll; ++u) r[u] = ld_stream_v4(s4 + i + u * kCopyThreads);
#pragma unroll
                for (int u = 0; u < kCopyUnroll; ++u) st_v4(d4 + i + u * kCopyThreads, r[u]);
            } else {
                for (; i < end; i += kCopyThreads) st_v4(d4 + i, ld_stream_v4(s4 + i));
            }
            if (j == 0) {
                if (threadIdx.x < p.head) dst[threadIdx.x] = src[threadIdx.x];
                const std::int64_t tb = p.head + p.vecs * 16;
                if (threadIdx.x < p.tail) dst[tb + threadIdx.x] = src[tb + threadIdx.x];
            }
        } else {
            const std::int64_t beg = j * kChunkVec * 16, end = i64min(t.bytes[seg], beg + kChunkVec * 16);
            for (std::int64_t b = beg + threadIdx.x; b < end; b += kCopyThreads) dst[b] = src[b];
        }
    }
}

cudaError_t launch_copy_segments(const SegTable& t, int ctas, cudaStream_t s) {
    if (t.n <= 0) return cudaSuccess;
    if (ctas <= 0) ctas = 148;
    count_launch();
    copy_segments_kernel<<<ctas, kCopyThreads, 0, s>>>(t);
    return cudaGetLastError();
}

// ---------------------------------------------------- fetch (TMA bulk)
// The fetch engine proper. One elected thread per CTA streams chunks
// peer HBM --cp.async.bulk--> smem --cp.async.bulk--> local HBM through a
// kTmaStages-deep mbarrier pipeline, so each CTA keeps kTmaSmem of NVLink reads
// in flight from a single thread; a small CTA budget leaves the SMs to the
// model's kernels. Every CTA owns a contiguous slice of EVERY owner's shard
// and walks the slices round-robin, so all owners (and the local shard) are
// served concurrently instead of one after the other. Bytes before the first
// 16-byte-aligned address and after the last one (ragged shards) are moved
// by a second warp.
// 4 x 32 KB per CTA: ~128 KB of NVLink reads in flight per CTA is what the
// link needs (64 CTAs: 645 GB/s at N=2). A 3 x 8 KB variant that fits next to
// a resident GEMM/attention CTA reached only 340 GB/s and did not change the
// SFT step (profiles/r01/p2p_n2_smallsmem.md), so the big ring stays.
constexpr int kTmaChunk = 32768;
constexpr int kTmaStages = 5;  // 4 peer loads in flight + 1 stage whose store to local HBM is still reading smem
constexpr int kTmaThreads = 64;
constexpr int kTmaSmem = kTmaChunk * kTmaStages;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

struct TmaJobs {
    // this CTA's slice of every segment, in 16-byte-aligned body chunks
    std::int64_t first[kMaxSeg], count[kMaxSeg], body0[kMaxSeg], body_bytes[kMaxSeg];
    int n;
    std::int64_t k;  // round
    int s;           // segment within the round
    __device__ bool next(int& seg, std::int64_t& off, int& bytes) {
        std::int64_t maxc = 0;
        for (int i = 0; i < n; ++i) maxc = count[i] > maxc ? count[i] : maxc;
        while (k < maxc) {
            while (s < n) {
                const int i = s++;
                if (k < count[i]) {
                    const std::int64_t c = first[i] + k;
                    seg = i;
                    off = body0[i] + c * kTmaChunk;
                    const std::int64_t rem = body0[i] + body_bytes[i] - off;
                    bytes = static_cast<int>(rem < kTmaChunk ? rem : kTmaChunk);
                    return true;
                }
            }
            s = 0;
            ++k;
        }
        return false;
    }
};

__global__ void __launch_bounds__(kTmaThreads, 1) fetch_tma_kernel(SegTable t) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) unsigned long long bar[kTmaStages];
    __shared__ int gate_ok;
    const int tid = threadIdx.x;
    if (tid == 0) gate_ok = 1;
    __syncthreads();
    // on-demand readiness: every owner published the parameter epoch we need
    if (tid < t.n && t.gate[tid] && !wait_geq(t.gate[tid], t.need, t.err, t.timeout_ns)) gate_ok = 0;
    __syncthreads();
    if (!gate_ok) return;
    asm volatile("fence.proxy.async.global;" ::: "memory");

    if (tid >= 32) {  // warp 1: ragged head/tail bytes and non-co-aligned segments
        const int lane = tid - 32;
        for (int i = 0; i < t.n; ++i) {
            const char* src = t.src[i];
            char* dst = t.dst[i];
            const std::int64_t bytes = t.bytes[i];
            if (bytes <= 0) continue;
            const unsigned sa = static_cast<unsigned>(reinterpret_cast<uintptr_t>(src) & 15);
            const unsigned da = static_cast<unsigned>(reinterpret_cast<uintptr_t>(dst) & 15);
            if (sa != da) {  // slow path: this CTA's byte slice
                const std::int64_t b0 = bytes * blockIdx.x / gridDim.x, b1 = bytes * (blockIdx.x + 1) / gridDim.x;
                for (std::int64_t b = b0 + lane; b < b1; b += 32) dst[b] = src[b];
                continue;
            }
            if (blockIdx.x != 0) continue;
            const std::int64_t head = i64min(bytes, (16 - da) & 15);
            const std::int64_t body = (bytes - head) & ~static_cast<std::int64_t>(15);
            if (lane < head) dst[lane] = src[lane];
            const std::int64_t tb = head + body;
            if (lane < bytes - tb) dst[tb + lane] = src[tb + lane];
        }
        return;
    }
    if (tid != 0) return;

    TmaJobs jobs{};
    jobs.n = t.n;
    for (int i = 0; i < t.n; ++i) {
        const std::int64_t bytes = t.bytes[i];
        const unsigned sa = static_cast<unsigned>(reinterpret_cast<uintptr_t>(t.src[i]) & 15);
        const unsigned da = static_cast<unsigned>(reinterpret_cast<uintptr_t>(t.dst[i]) & 15);
        if (bytes <= 0 || sa != da) {
            jobs.count[i] = 0;
            continue;
        }
        const std::int64_t head = i64min(bytes, (16 - da) & 15);
        jobs.body0[i] = head;
        jobs.body_bytes[i] = (bytes - head) & ~static_cast<std::int64_t>(15);
        const std::int64_t nch = (jobs.body_bytes[i] + kTmaChunk - 1) / kTmaChunk;
        jobs.first[i] = nch * blockIdx.x / gridDim.x;
        jobs.count[i] = nch * (blockIdx.x + 1) / gridDim.x - jobs.first[i];
    }
    for (int s = 0; s < kTmaStages; ++s)
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

    int seg[kTmaStages], nbytes[kTmaStages];
    std::int64_t off[kTmaStages];
    unsigned phase = 0;  // bit s = parity to wait for on stage s
    auto load = [&](int st) {
        const unsigned b = smem_u32(&bar[st]);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(nbytes[st]) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem + st * kTmaChunk)),
            "l"(t.src[seg[st]] + off[st]), "r"(nbytes[st]), "r"(b)
            : "memory");
    };
    // Stages are consumed in load-issue order (a FIFO of stage ids). A consumed
    // stage is stored to local HBM and refilled only one iteration later, after
    // `wait_group.read 1` (every store but the newest has read its smem): the
    // peer loads never wait for the store that was just issued.
    int fifo[kTmaStages];
    int head = 0, count = 0;
    for (int st = 0; st < kTmaStages - 1; ++st) {
        if (!jobs.next(seg[st], off[st], nbytes[st])) break;
        load(st);
        fifo[(head + count++) % kTmaStages] = st;
    }
    int spare = kTmaStages - 1;  // the stage kept free for the store in flight
    int stored = -1;             // stage whose store was issued last iteration (refill candidate)
    while (count > 0) {
        const int st = fifo[head];
        head = (head + 1) % kTmaStages;
        --count;
        asm volatile(
            "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(
                smem_u32(&bar[st])),
            "r"((phase >> st) & 1u)
            : "memory");
        phase ^= 1u << st;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(t.dst[seg[st]] + off[st]),
                     "r"(smem_u32(smem + st * kTmaChunk)), "r"(nbytes[st])
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // refill: the spare stage (never used yet) first, then the stage stored one iteration ago
        int refill = spare;
        if (refill < 0) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            refill = stored;
        }
        spare = -1;
        stored = st;
        if (refill >= 0 && jobs.next(seg[refill], off[refill], nbytes[refill])) {
            load(refill);
            fifo[(head + count++) % kTmaStages] = refill;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

cudaError_t launch_fetch_tma(const SegTable& t, int ctas, cudaStream_t s) {
    if (t.n <= 0) return cudaSuccess;
    static thread_local int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(fetch_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
        if (e != cudaSuccess) return e;
        configured_dev = dev;
    }
    if (ctas <= 0) ctas = 64;
    count_launch();
    fetch_tma_kernel<<<ctas, kTmaThreads, kTmaSmem, s>>>(t);
    return cudaGetLastError();
}

// ------------------------------------------------------------- push (RED)
constexpr int kPushThreads = 512;
constexpr int kPushUnroll = 4;
constexpr std::int64_t kPushChunk = kPushThreads * kPushUnroll;  // 4-element units per chunk

struct RedPlan {
    std::int64_t head, units, tail, chunks;  // head/tail in elements, units of 4 elements
    bool fast;
};

__device__ __forceinline__ RedPlan plan_red(const void* src, const float* dst, std::int64_t n, bool bf16) {
    RedPlan p{};
    if (n <= 0) return p;
    const unsigned da = static_cast<unsigned>(reinterpret_cast<uintptr_t>(dst) & 15);  // multiple of 4
    const std::int64_t head = i64min(n, ((16 - da) & 15) / 4);
    const uintptr_t s_after = reinterpret_cast<uintptr_t>(src) + head * (bf16 ? 2 : 4);
    p.fast = (da % 4 == 0) && (s_after % (bf16 ? 8 : 16) == 0);
    if (p.fast) {
        p.head = head;
        p.units = (n - head) / 4;
        p.tail = n - head - p.units * 4;
        p.chunks = i64max(1, (p.units + kPushChunk - 1) / kPushChunk);
    } else {
        p.chunks = (n + kPushChunk * 4 - 1) / (kPushChunk * 4);
    }
    return p;
}

template <bool BF16>
__device__ __forceinline__ float load_grad(const void* src, std::int64_t i) {
    if constexpr (BF16) return bf16_to_f32(reinterpret_cast<const unsigned short*>(src)[i]);
    else return reinterpret_cast<const float*>(src)[i];
}

template <bool BF16>
__device__ __forceinline__ float4 load_grad4(const void* src, std::int64_t e) {
    if constexpr (BF16) {
        const uint2 v = *reinterpret_cast<const uint2*>(reinterpret_cast<const unsigned short*>(src) + e);
        return make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u), __uint_as_float(v.y << 16),
                           __uint_as_float(v.y & 0xffff0000u));
    } else {
        return *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src) + e);
    }
}

template <bool BF16>
__global__ void __launch_bounds__(kPushThreads) push_red_kernel(RedTable t, float w) {
    // Every CTA owns a contiguous slice of every owner's shard and walks the
    // slices round-robin in kPushChunk-unit steps, so all owners (and the
    // local shard) receive reductions concurrently.
    __shared__ RedPlan plans[kMaxSeg];
    __shared__ std::int64_t lo[kMaxSeg], hi[kMaxSeg];
    __shared__ int gate_ok;
    if (threadIdx.x == 0) gate_ok = 1;
    __syncthreads();
    // the owner finished its previous AdamW (its grad shard is zeroed)
    if (threadIdx.x < t.n && t.gate[threadIdx.x] && !wait_geq(t.gate[threadIdx.x], t.need, t.err, t.timeout_ns))
        gate_ok = 0;
    if (threadIdx.x < t.n) {
        const int i = threadIdx.x;
        RedPlan p = plan_red(t.src[i], t.dst[i], t.elems[i], BF16);
        plans[i] = p;
        const std::int64_t n = p.fast ? p.units : t.elems[i];  // units of 4 (fast) or elements (slow)
        lo[i] = n * blockIdx.x / gridDim.x;
        hi[i] = n * (blockIdx.x + 1) / gridDim.x;
    }
    __syncthreads();
    if (!gate_ok) return;
    std::int64_t maxlen = 0;
    for (int i = 0; i < t.n; ++i) maxlen = i64max(maxlen, hi[i] - lo[i]);
    for (std::int64_t k = 0; k < maxlen; k += kPushChunk) {
        for (int i = 0; i < t.n; ++i) {
            const std::int64_t beg = lo[i] + k;
            const std::int64_t end = i64min(hi[i], beg + kPushChunk);
            if (beg >= end) continue;
            const RedPlan p = plans[i];
            const void* src = t.src[i];
            float* dst = t.dst[i];
            if (p.fast) {
                std::int64_t u = beg + threadIdx.x;
                if (end - beg == kPushChunk) {
                    float4 g[kPushUnroll];
#pragma unroll
                    for (int q = 0; q < kPushUnroll; ++q) g[q] = load_grad4<BF16>(src, p.head + 4 * (u + q * kPushThreads));
#pragma unroll
                    for (int q = 0; q < kPushUnroll; ++q)
                        red_sys_v4(dst + p.head + 4 * (u + q * kPushThreads), __fmul_rn(w, g[q].x), __fmul_rn(w, g[q].y),
                                   __fmul_rn(w, g[q].z), __fmul_rn(w, g[q].w));
                } else {
                    for (; u < end; u += kPushThreads) {
                        const float4 g = load_grad4<BF16>(src, p.head + 4 * u);
                        red_sys_v4(dst + p.head + 4 * u, __fmul_rn(w, g.x), __fmul_rn(w, g.y), __fmul_rn(w, g.z),
                                   __fmul_rn(w, g.w));
                    }
                }
            } else {
                for (std::int64_t e = beg + threadIdx.x; e < end; e += kPushThreads)
                    red_sys_f32(dst + e, __fmul_rn(w, load_grad<BF16>(src, e)));
            }
        }
    }
    if (blockIdx.x == 0) {  // ragged head / tail elements of the fast segments
        for (int i = 0; i < t.n; ++i) {
            const RedPlan p = plans[i];
            if (!p.fast) continue;
            if (threadIdx.x < p.head) red_sys_f32(t.dst[i] + threadIdx.x, __fmul_rn(w, load_grad<BF16>(t.src[i], threadIdx.x)));
            const std::int64_t tb = p.head + 4 * p.units;
            if (threadIdx.x < p.tail)
                red_sys_f32(t.dst[i] + tb + threadIdx.x, __fmul_rn(w, load_grad<BF16>(t.src[i], tb + threadIdx.x)));
        }
    }
    // order this thread's remote reductions before anything later in the
    // stream (the barrier kernel's release also covers them cumulatively)
    __threadfence_system();
}

cudaError_t launch_push_red(const RedTable& t, float w, bool src_bf16, int ctas, cudaStream_t s) {
    if (t.n <= 0) return cudaSuccess;
    if (ctas <= 0) ctas = 148;
    count_launch();
    if (src_bf16) push_red_kernel<true><<<ctas, kPushThreads, 0, s>>>(t, w);
    else push_red_kernel<false><<<ctas, kPushThreads, 0, s>>>(t, w);
    return cudaGetLastError();
}

// ------------------------------------------------------------ gates
struct GateList {
    const unsigned long long* g[kMaxSeg];
    int n;
    unsigned long long need;
    unsigned long long* err;
    long long timeout_ns;
};

__device__ __forceinline__ bool pass_gates(const GateList& gl) {
    __shared__ int ok;
    if (threadIdx.x == 0) ok = 1;
    __syncthreads();
    if (threadIdx.x < gl.n && !wait_geq(gl.g[threadIdx.x], gl.need, gl.err, gl.timeout_ns)) ok = 0;
    __syncthreads();
    return ok != 0;
}

// ------------------------------------------------------------ push (FIXED)
// Deterministic push in bounded memory: every pushed value is
// rounded once to a 64-bit fixed-point integer, q = rn(fl(w*g) * 2^S), and
// added into the owner's int64 accumulator with TMA bulk reductions
// (cp.reduce.async.bulk .add.u64, peer HBM over NVLink). Integer addition is
// associative, so the owner's sum is bit-identical for every arrival order,
// every interleaving of clients and every world size; the memory cost is
// 8 B per OWNED element (SLOT mode needs 4 B per element of every unit).
// cvt.rni.s64.f32 rounds to nearest even, clamps out-of-range values and maps
// NaN to 0. Range: |sum| < 2^(63-S) (2^23 at the default S = 40).
constexpr int kFixThreads = 256;


// Range: a single contribution must satisfy |w*g*2^S| < 2^kFixedMaxLog2 (2^55),
// leaving 8 guard bits so 256 maximal contributions cannot overflow the int64
// sum. A contribution outside that range (or NaN/Inf) sets `range`; a nonzero
// contribution that rounds to 0 sets `under` (resolution loss, not an error).
constexpr float kFixedMax = 36028797018963968.0f;  // 2^55
__device__ __forceinline__ long long to_fixed(float w, float g, float scale, bool& range, bool& under) {
    const float x = __fmul_rn(__fmul_rn(w, g), scale);
    if (!(fabsf(x) < kFixedMax)) range = true;
    const long long q = __float2ll_rn(x);
    if (q == 0 && x != 0.f) under = true;
    return q;
}
__device__ __forceinline__ void red_sys_u64(long long* p, long long v) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <bool BF16>
__device__ __forceinline__ float2 load_grad2(const void* src, std::int64_t e) {
    if constexpr (BF16) {
        const unsigned v = *reinterpret_cast<const unsigned*>(reinterpret_cast<const unsigned short*>(src) + e);
        return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));
    } else {
        return *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(src) + e);
    }
}

// One kernel body for the bulk pushes: every 16 B unit of the owner's shard
// (FIXED: 2 int64, F32: 4 fp32) is produced in registers, staged in a 3-deep
// shared-memory ring and added into peer HBM by one elected thread with
// cp.reduce.async.bulk (.add.u64 / .add.f32) — or, for an F32 segment marked
// `assign` (SLOT mode: the first push of a unit into this client's slot at the
// owner in this minibatch), STORED with cp.async.bulk (NVLink write
// bandwidth, no remote read-modify-write). 8 KB per bulk op, 25 KB of smem per
// CTA so four CTAs share an SM (and one fits next to a GEMM).
constexpr int kBulkUnits = 2;   // 16 B units per thread per chunk
constexpr int kBulkStages = 3;

template <bool BF16, bool FIXED>
__global__ void __launch_bounds__(kFixThreads) push_bulk_kernel(BulkTable t, float w, float scale) {
    constexpr int E = FIXED ? 2 : 4;                 // elements per 16 B unit of dst
    constexpr int kDstBytes = FIXED ? 8 : 4;
    constexpr std::int64_t kChunk = kFixThreads * kBulkUnits;  // units per chunk
    __shared__ __align__(128) uint4 stage[kBulkStages][kChunk];
    __shared__ std::int64_t head[kMaxSeg], lo[kMaxSeg], hi[kMaxSeg];
    __shared__ bool fast[kMaxSeg];
    __shared__ int gate_ok;
    bool range = false, under = false;  // FIXED conversion flags of this thread
    if (threadIdx.x == 0) gate_ok = 1;
    __syncthreads();
    // the owner consumed what the previous minibatch left in this push target (drain epoch)
    const bool my_gate = !(threadIdx.x < t.n && t.gate[threadIdx.x]) ||
                         wait_geq(t.gate[threadIdx.x], t.need, t.err, t.timeout_ns);
    if (!my_gate) gate_ok = 0;
    if (my_gate && blockIdx.x == 0 && threadIdx.x < t.n && t.mark[threadIdx.x])  // SLOT: "client pushed this unit"
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(t.mark[threadIdx.x]), "l"(t.mark_value) : "memory");
    if (threadIdx.x < t.n) {
        const int i = threadIdx.x;
        // the owner's shard is co-aligned with its position in the caller's full-layer
        // buffer (arena padding), so after < E head elements dst is 16 B aligned and the
        // grad body is aligned for E-element vector loads
        const std::int64_t n = t.elems[i];
        const uintptr_t d = reinterpret_cast<uintptr_t>(t.dst[i]);
        const std::int64_t h = i64min(n, static_cast<std::int64_t>(((16 - (d & 15)) & 15) / kDstBytes));
        const uintptr_t s_body = reinterpret_cast<uintptr_t>(t.src[i]) + h * (BF16 ? 2 : 4);
        fast[i] = d % kDstBytes == 0 && s_body % (E * (BF16 ? 2 : 4)) == 0;
        head[i] = fast[i] ? h : 0;
        const std::int64_t units = fast[i] ? (n - h) / E : 0;
        lo[i] = units * blockIdx.x / gridDim.x;
        hi[i] = units * (blockIdx.x + 1) / gridDim.x;
    }
    __syncthreads();
    if (!gate_ok) return;
    // the gates were acquired through the generic proxy; the reductions go through the async proxy
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
    std::int64_t maxlen = 0;
    for (int i = 0; i < t.n; ++i) maxlen = i64max(maxlen, hi[i] - lo[i]);
    int it = 0;
    for (std::int64_t k = 0; k < maxlen; k += kChunk) {
        for (int i = 0; i < t.n; ++i) {
            const std::int64_t beg = lo[i] + k;
            const std::int64_t end = i64min(hi[i], beg + kChunk);
            if (beg >= end) continue;
            uint4* buf = stage[it % kBulkStages];
            if (it >= kBulkStages) {  // the bulk reduction that last read this stage has finished reading it
                if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kBulkStages - 1) : "memory");
                __syncthreads();
            }
            const std::int64_t e0 = head[i] + E * beg;  // element offset of the chunk in the segment
            const std::int64_t nu = end - beg;
#pragma unroll
            for (int q = 0; q < kBulkUnits; ++q) {
                const std::int64_t u = threadIdx.x + q * kFixThreads;
                if (u < nu) {
                    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(buf + u));
                    if constexpr (FIXED) {
                        const float2 g = load_grad2<BF16>(t.src[i], e0 + E * u);
                        asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(sa), "l"(to_fixed(w, g.x, scale, range, under)),
                                     "l"(to_fixed(w, g.y, scale, range, under))
                                     : "memory");
                    } else {
                        const float4 g = load_grad4<BF16>(t.src[i], e0 + E * u);
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sa), "f"(__fmul_rn(w, g.x)),
                                     "f"(__fmul_rn(w, g.y)), "f"(__fmul_rn(w, g.z)), "f"(__fmul_rn(w, g.w))
                                     : "memory");
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) {
                char* dst = static_cast<char*>(t.dst[i]) + e0 * kDstBytes;
                const unsigned src = static_cast<unsigned>(__cvta_generic_to_shared(buf));
                const unsigned bytes = static_cast<unsigned>(nu * 16);
                if constexpr (FIXED)
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(dst),
                                 "r"(src), "r"(bytes)
                                 : "memory");
                else if (t.assign[i])
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
                                 "r"(bytes)
                                 : "memory");
                else
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                                 "r"(src), "r"(bytes)
                                 : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++it;
        }
    }
    if (threadIdx.x == 0) {  // reductions complete, then ordered before the barrier's release (later kernel)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __threadfence_system();
    }
    auto scalar = [&](int i, std::int64_t e) {
        const float g = load_grad<BF16>(t.src[i], e);
        if constexpr (FIXED) red_sys_u64(static_cast<long long*>(t.dst[i]) + e, to_fixed(w, g, scale, range, under));
        else if (t.assign[i]) static_cast<float*>(t.dst[i])[e] = __fmul_rn(w, g);
        else red_sys_f32(static_cast<float*>(t.dst[i]) + e, __fmul_rn(w, g));
    };
    for (int i = 0; i < t.n; ++i)  // segments whose src/dst alignment rules out the bulk path: scalar reductions
        if (!fast[i])
            for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * kFixThreads + threadIdx.x; e < t.elems[i];
                 e += static_cast<std::int64_t>(gridDim.x) * kFixThreads)
                scalar(i, e);
    if (blockIdx.x == gridDim.x - 1) {  // ragged head / tail elements of each bulk segment
        for (int i = 0; i < t.n; ++i) {
            const std::int64_t n = t.elems[i];
            if (n <= 0 || !fast[i]) continue;
            const std::int64_t body_end = head[i] + E * ((n - head[i]) / E);
            if (threadIdx.x < head[i]) scalar(i, threadIdx.x);
            if (body_end + threadIdx.x < n) scalar(i, body_end + threadIdx.x);
        }
    }
    if constexpr (FIXED) {  // sticky flags in the owner-independent local error word
        const int any_range = __syncthreads_or(range), any_under = __syncthreads_or(under);
        if (threadIdx.x == 0 && t.err && (any_range || any_under))
            atomicOr(t.err, (any_range ? kErrFixedRange : 0ull) | (any_under ? kWarnFixedUnderflow : 0ull));
    }
}

cudaError_t launch_push_bulk(const BulkTable& t, bool fixed, float w, float scale, bool src_bf16, int ctas,
                             cudaStream_t s) {
    if (t.n <= 0) return cudaSuccess;
    if (ctas <= 0) ctas = 148 * 4;
    count_launch();
    if (fixed) {
        if (src_bf16) push_bulk_kernel<true, true><<<ctas, kFixThreads, 0, s>>>(t, w, scale);
        else push_bulk_kernel<false, true><<<ctas, kFixThreads, 0, s>>>(t, w, scale);
    } else {
        if (src_bf16) push_bulk_kernel<true, false><<<ctas, kFixThreads, 0, s>>>(t, w, scale);
        else push_bulk_kernel<false, false><<<ctas, kFixThreads, 0, s>>>(t, w, scale);
    }
    return cudaGetLastError();
}

// SLOT mode, owner side, after the minibatch barrier: every unit's grad shard
// = the clients' slots summed in fixed rank order 0..N-1, counting only the
// clients whose mark says they pushed the unit in this minibatch (a slot that
// was not written this minibatch still holds an older one). Local HBM only:
// the slots were written over NVLink during the clients' backward passes.
__global__ void __launch_bounds__(512) slot_reduce_kernel(SlotReduce r) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (int u = 0; u < r.n; ++u) {
        const std::int64_t n = r.elems[u];
        if (n <= 0) continue;
        unsigned active = 0;  // clients that pushed this unit (N <= kMaxSeg)
        for (int c = 0; c < r.nsrc; ++c)
            if (*reinterpret_cast<volatile const unsigned long long*>(r.marks[u] + c) == r.epoch) active |= 1u << c;
        float* dst = r.dst[u];
        const float* s0 = r.slot0[u];
        const std::int64_t sst = r.slot_stride[u];
        const unsigned h = static_cast<unsigned>((reinterpret_cast<uintptr_t>(dst) >> 2) & 3);
        const std::int64_t head = i64min(n, (4 - h) & 3);
        const std::int64_t units = (n - head) / 4;
        for (std::int64_t k = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < units; k += stride) {
            const std::int64_t e = head + 4 * k;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
            bool first = true;
            for (int c = 0; c < r.nsrc; ++c) {  // rank order: deterministic
                if (!(active >> c & 1u)) continue;
                const float4 b = *reinterpret_cast<const float4*>(s0 + c * sst + e);
                if (first) {
                    a = b;
                    first = false;
                } else {
                    a.x = __fadd_rn(a.x, b.x);
                    a.y = __fadd_rn(a.y, b.y);
                    a.z = __fadd_rn(a.z, b.z);
                    a.w = __fadd_rn(a.w, b.w);
                }
            }
            *reinterpret_cast<float4*>(dst + e) = a;
        }
        if (blockIdx.x == 0) {  // ragged head / tail
            const std::int64_t tail = n - head - 4 * units;
            std::int64_t e = -1;
            if (threadIdx.x < head) e = threadIdx.x;
            else if (threadIdx.x >= 4 && threadIdx.x < 4 + tail) e = head + 4 * units + threadIdx.x - 4;
            if (e >= 0) {
                float a = 0.f;
                bool first = true;
                for (int c = 0; c < r.nsrc; ++c) {
                    if (!(active >> c & 1u)) continue;
                    a = first ? s0[c * sst + e] : __fadd_rn(a, s0[c * sst + e]);
                    first = false;
                }
                dst[e] = a;
            }
        }
    }
}

cudaError_t launch_slot_reduce(const SlotReduce& r, cudaStream_t s) {
    if (r.n <= 0) return cudaSuccess;
    count_launch();
    slot_reduce_kernel<<<148 * 2, 512, 0, s>>>(r);
    return cudaGetLastError();
}

// owner side, after the minibatch barrier: grad = fl(acc) * 2^-S, acc = 0
__global__ void __launch_bounds__(512) fixed_finalize_kernel(FixFinal f, float inv_scale) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (int s = 0; s < f.n; ++s) {
        float* g = f.grad[s];
        long long* a = f.acc[s];
        for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < f.elems[s];
             e += stride) {
            g[e] = __fmul_rn(__ll2float_rn(a[e]), inv_scale);
            a[e] = 0;
        }
    }
}

cudaError_t launch_fixed_finalize(const FixFinal& f, float inv_scale, cudaStream_t s) {
    if (f.n <= 0) return cudaSuccess;
    count_launch();
    fixed_finalize_kernel<<<148 * 4, 512, 0, s>>>(f, inv_scale);
    return cudaGetLastError();
}

// ------------------------------------------------ typed fabric accumulate
template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b) { return a * b; }
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b) { return a + b; }
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void accumulate_kernel(T* __restrict__ dst, const T* __restrict__ src, std::int64_t n, T w) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = add_rn(dst[i], mul_rn(w, src[i]));
}

template <typename T>
__device__ __forceinline__ void red_one(T* p, T v);
template <>
__device__ __forceinline__ void red_one<long long>(long long* p, long long v) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <>
__device__ __forceinline__ void red_one<double>(double* p, double v) {
    asm volatile("red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
template <>
__device__ __forceinline__ void red_one<float>(float* p, float v) {
    red_sys_f32(p, v);
}

template <typename T>
__global__ void red_accumulate_kernel(T* __restrict__ dst, const T* __restrict__ src, std::int64_t n, T w) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        red_one<T>(dst + i, mul_rn(w, src[i]));
}

static int small_grid(std::int64_t n) {
    std::int64_t g = (n + 255) / 256;
    return static_cast<int>(g < 1 ? 1 : (g > 592 ? 592 : g));
}

template <typename T>
cudaError_t launch_accumulate(T* dst, const T* src, std::int64_t n, T w, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    count_launch();
    accumulate_kernel<T><<<small_grid(n), 256, 0, s>>>(dst, src, n, w);
    return cudaGetLastError();
}
template <typename T>
cudaError_t launch_red_accumulate(T* dst, const T* src, std::int64_t n, T w, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    count_launch();
    red_accumulate_kernel<T><<<small_grid(n), 256, 0, s>>>(dst, src, n, w);
    return cudaGetLastError();
}
template cudaError_t launch_accumulate<long long>(long long*, const long long*, std::int64_t, long long, cudaStream_t);
template cudaError_t launch_accumulate<double>(double*, const double*, std::int64_t, double, cudaStream_t);
template cudaError_t launch_accumulate<float>(float*, const float*, std::int64_t, float, cudaStream_t);
template cudaError_t launch_red_accumulate<long long>(long long*, const long long*, std::int64_t, long long,
                                                      cudaStream_t);
template cudaError_t launch_red_accumulate<double>(double*, const double*, std::int64_t, double, cudaStream_t);
template cudaError_t launch_red_accumulate<float>(float*, const float*, std::int64_t, float, cudaStream_t);

// ------------------------------------------------------------- barrier
__global__ void barrier_kernel(BarrierArgs a) {
    const int t = threadIdx.x;
    // Every push this rank issued earlier on the stream completed before this
    // kernel started (kernel boundary); the sys-scope fence makes their
    // effects (remote red/bulk reductions, slot stores) ordered before the
    // flag stores below for every observer, independently of the cumulativity
    // of the release.
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (t < a.world) {
        // release: every push this rank issued earlier on the stream (kernel
        // boundaries order them before this thread) is visible to owner t
        // before it observes the flag. PTX release is cumulative.
        st_release_sys(a.peer_done[t] + a.rank, a.epoch);
    }
    if (t < a.world) wait_geq(a.my_done + t, a.epoch, a.err, a.timeout_ns);
    __syncthreads();
}

cudaError_t launch_barrier(const BarrierArgs& a, cudaStream_t s) {
    count_launch();
    barrier_kernel<<<1, 32 * ((a.world + 31) / 32), 0, s>>>(a);
    return cudaGetLastError();
}

__global__ void publish_kernel(unsigned long long* flag, unsigned long long v, unsigned long long* flag2,
                               unsigned long long v2) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release_sys(flag, v);
    if (flag2) st_release_sys(flag2, v2);
}

cudaError_t launch_publish(unsigned long long* flag, unsigned long long value, cudaStream_t s,
                           unsigned long long* flag2, unsigned long long value2) {
    count_launch();
    publish_kernel<<<1, 1, 0, s>>>(flag, value, flag2, value2);
    return cudaGetLastError();
}

struct ZeroList {
    float* p[64];
    std::int64_t n[64];
    int count;
};

__global__ void gated_zero_kernel(ZeroList z, GateList gl) {
    if (gl.n > 0 && !pass_gates(gl)) return;
    for (int k = 0; k < z.count; ++k) {
        const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
        for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < z.n[k]; i += stride)
            z.p[k][i] = 0.f;
    }
}

cudaError_t launch_gated_zero(float* const* ptrs, const std::int64_t* n, int count,
                              const unsigned long long* const* gates, int ngates, unsigned long long need,
                              unsigned long long* err, long long timeout_ns, cudaStream_t s) {
    GateList gl{};
    gl.n = ngates;
    for (int i = 0; i < ngates; ++i) gl.g[i] = gates[i];
    gl.need = need;
    gl.err = err;
    gl.timeout_ns = timeout_ns;
    if (count == 0) {  // gate only (copy-engine fetch waits on it in stream order)
        ZeroList z{};
        count_launch();
        gated_zero_kernel<<<1, 32, 0, s>>>(z, gl);
        return cudaGetLastError();
    }
    for (int base = 0; base < count; base += 64) {
        ZeroList z{};
        z.count = count - base < 64 ? count - base : 64;
        for (int k = 0; k < z.count; ++k) {
            z.p[k] = ptrs[base + k];
            z.n[k] = n[base + k];
        }
        count_launch();
        gated_zero_kernel<<<296, 512, 0, s>>>(z, gl);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ---------------------------------------------------------------- AdamW
// torch.optim.AdamW(foreach=False) update order:
//   p *= 1 - lr*wd;  m = lerp(m, g, 1-b1);  v = b2*v + (1-b2)*g*g
//   p -= step_size * m / (sqrt(v)/sqrt(bc2) + eps)
__device__ __forceinline__ void adam_one(float& p, float& m, float& v, float g, const AdamArgs& a) {
    p = p * (1.f - a.lr * a.wd);
    m = m + (1.f - a.beta1) * (g - m);
    v = a.beta2 * v + (1.f - a.beta2) * g * g;
    const float denom = sqrtf(v) * a.bc2_sqrt_inv + a.eps;
    p = p - a.step_size * (m / denom);
}

__global__ void __launch_bounds__(512) adam_kernel(AdamArgs a) {
    const std::int64_t total = a.seg_start[a.nseg];
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    int seg = 0;
    for (std::int64_t u = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < total; u += stride) {
        while (u >= a.seg_start[seg + 1]) ++seg;
        const AdamSeg S = a.segs[seg];
        // unit k covers elements [4k - h, 4k - h + 4) of the shard, where h
        // is the shard's element offset mod 4 (all fp32 arrays co-aligned)
        const int h = static_cast<int>((reinterpret_cast<uintptr_t>(S.master) >> 2) & 3);
        const std::int64_t k = u - a.seg_start[seg];
        const std::int64_t e0 = 4 * k - h;
        if (e0 >= 0 && e0 + 4 <= S.n) {
            float4 p = *reinterpret_cast<float4*>(S.master + e0);
            float4 m = *reinterpret_cast<float4*>(S.m + e0);
            float4 v = *reinterpret_cast<float4*>(S.v + e0);
            float4 g = *reinterpret_cast<float4*>(S.grad + e0);
            adam_one(p.x, m.x, v.x, g.x, a);
            adam_one(p.y, m.y, v.y, g.y, a);
            adam_one(p.z, m.z, v.z, g.z, a);
            adam_one(p.w, m.w, v.w, g.w, a);
            *reinterpret_cast<float4*>(S.master + e0) = p;
            *reinterpret_cast<float4*>(S.m + e0) = m;
            *reinterpret_cast<float4*>(S.v + e0) = v;
            *reinterpret_cast<float4*>(S.grad + e0) = make_float4(0.f, 0.f, 0.f, 0.f);
            uint2 pb;
            pb.x = static_cast<unsigned>(f32_to_bf16(p.x)) | (static_cast<unsigned>(f32_to_bf16(p.y)) << 16);
            pb.y = static_cast<unsigned>(f32_to_bf16(p.z)) | (static_cast<unsigned>(f32_to_bf16(p.w)) << 16);
            *reinterpret_cast<uint2*>(S.param + e0) = pb;
        } else {
            for (std::int64_t e = e0 < 0 ? 0 : e0; e < e0 + 4 && e < S.n; ++e) {
                float p = S.master[e], m = S.m[e], v = S.v[e];
                adam_one(p, m, v, S.grad[e], a);
                S.master[e] = p;
                S.m[e] = m;
                S.v[e] = v;
                S.grad[e] = 0.f;
                S.param[e] = f32_to_bf16(p);
            }
        }
    }
}

cudaError_t launch_adam(const AdamArgs& a, std::int64_t total_units, int ctas, cudaStream_t s) {
    if (total_units <= 0) return cudaSuccess;
    if (ctas <= 0) ctas = 148 * 4;
    count_launch();
    adam_kernel<<<ctas, 512, 0, s>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------ L2 flush
__global__ void l2_flush_kernel(uint4* p, std::int64_t n) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        p[i] = make_uint4(static_cast<unsigned>(i), 0u, 0u, 0u);
}

cudaError_t launch_l2_flush(void* scratch, std::int64_t bytes, cudaStream_t s) {
    count_launch();
    l2_flush_kernel<<<148 * 2, 512, 0, s>>>(reinterpret_cast<uint4*>(scratch), bytes / 16);
    return cudaGetLastError();
}

__global__ void init_shard_kernel(float* master, unsigned short* param, const float* src, std::int64_t n) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const float x = src[i];
        master[i] = x;
        param[i] = f32_to_bf16(x);
    }
}

// Loads every kernel of the ODC protocol into the context up front. With CUDA's
// lazy module loading, the FIRST launch of a kernel may wait for the device's
// running work; when that work is a barrier spinning on a peer whose kernels
// this host thread has yet to launch (several ranks driven from one thread,
// odc_ctx_import_ctx), the host would block inside the launch and the barrier
// would only end by its watchdog. Also keeps first-launch latency out of timed steps.
cudaError_t preload_kernels() {
    const void* fns[] = {
        reinterpret_cast<const void*>(copy_segments_kernel), reinterpret_cast<const void*>(fetch_tma_kernel),
        reinterpret_cast<const void*>(push_red_kernel<true>), reinterpret_cast<const void*>(push_red_kernel<false>),
        reinterpret_cast<const void*>(push_bulk_kernel<true, true>),
        reinterpret_cast<const void*>(push_bulk_kernel<true, false>),
        reinterpret_cast<const void*>(push_bulk_kernel<false, true>),
        reinterpret_cast<const void*>(push_bulk_kernel<false, false>), reinterpret_cast<const void*>(slot_reduce_kernel),
        reinterpret_cast<const void*>(fixed_finalize_kernel), reinterpret_cast<const void*>(barrier_kernel),
        reinterpret_cast<const void*>(publish_kernel), reinterpret_cast<const void*>(gated_zero_kernel),
        reinterpret_cast<const void*>(adam_kernel), reinterpret_cast<const void*>(init_shard_kernel)};
    for (const void* f : fns) {
        cudaFuncAttributes a;
        const cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_init_shard(float* master, unsigned short* param, const float* src, std::int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    count_launch();
    init_shard_kernel<<<296, 512, 0, s>>>(master, param, src, n);
    return cudaGetLastError();
}

}  // namespace odc
