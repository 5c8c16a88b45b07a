// p2p_probe.cu — NVLink ceiling probe for the fetch/push kernel design
// (single process, 2+ GPUs with peer access). Measures, GPU0 <-> GPU1:
//   ldg   : SM-driven 16B peer loads (fetch design), varying CTAs / unroll
//   stg   : SM-driven 16B peer stores
//   red   : red.relaxed.sys.global.add.v4.f32 to peer (push design)
//   tma   : cp.async.bulk global(peer)->smem->global(local), one thread/CTA
//   ce    : cudaMemcpyPeerAsync (copy engines)
// one direction and both directions at once. Prints GB/s per direction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe p2p_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
            std::exit(1);                                                                      \
        }                                                                                      \
    } while (0)

template <int U>
__global__ void ldg_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, long n) {
    long i = (long)blockIdx.x * blockDim.x * U + threadIdx.x;
    const long stride = (long)gridDim.x * blockDim.x * U;
    for (; i + (U - 1) * (long)blockDim.x < n; i += stride) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w)
                         : "l"(src + i + u * blockDim.x));
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * blockDim.x] = r[u];
    }
}

__global__ void stg_fill(uint4* dst, long n) {
    long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (long)gridDim.x * blockDim.x) dst[i] = make_uint4(1, 2, 3, (unsigned)i);
}

template <int U>
__global__ void red_push(const float4* __restrict__ src, float* dst, long n4) {
    long i = (long)blockIdx.x * blockDim.x * U + threadIdx.x;
    const long stride = (long)gridDim.x * blockDim.x * U;
    for (; i + (U - 1) * (long)blockDim.x < n4; i += stride) {
        float4 g[U];
#pragma unroll
        for (int u = 0; u < U; ++u) g[u] = src[i + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + 4 * (i + u * blockDim.x)),
                         "f"(g[u].x), "f"(g[u].y), "f"(g[u].z), "f"(g[u].w)
                         : "memory");
    }
}

// TMA bulk: each CTA moves chunks of CH bytes: peer gmem -> smem -> local gmem
template <int CH, int STAGES>
__global__ void tma_copy(const char* src, char* dst, long bytes) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) unsigned long long bar[STAGES];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    const long nch = bytes / CH;
    unsigned phase[STAGES] = {};
    long issued = 0, done = 0;
    long c0 = blockIdx.x;
    auto issue = [&](long c, int s) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * CH);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                     "l"(src + c * CH), "r"(CH), "r"(a)
                     : "memory");
    };
    long cs[STAGES];
    for (int s = 0; s < STAGES && c0 + issued * gridDim.x < nch; ++s, ++issued) {
        cs[s] = c0 + issued * gridDim.x;
        issue(cs[s], s);
    }
    while (done < issued) {
        int s = done % STAGES;
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
        asm volatile(
            "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(a), "r"(phase[s]));
        phase[s] ^= 1;
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * CH);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + cs[s] * CH), "r"(d),
                     "r"(CH)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        ++done;
        long nxt = c0 + issued * gridDim.x;
        if (nxt < nch) {
            cs[s] = nxt;
            issue(nxt, s);
            ++issued;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA bulk reduce push: local grad chunk -> smem (TMA load) -> peer += smem (cp.reduce.async.bulk .add.f32)
template <int CH, int STAGES>
__global__ void tma_red_push(const char* src_local, char* dst_peer, long bytes) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) unsigned long long bar[STAGES];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    const long nch = bytes / CH;
    unsigned phase[STAGES] = {};
    long issued = 0, done = 0;
    long c0 = blockIdx.x;
    long cs[STAGES];
    auto issue = [&](long c, int s) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * CH);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                     "l"(src_local + c * CH), "r"(CH), "r"(a)
                     : "memory");
    };
    for (int s = 0; s < STAGES && c0 + issued * gridDim.x < nch; ++s, ++issued) {
        cs[s] = c0 + issued * gridDim.x;
        issue(cs[s], s);
    }
    while (done < issued) {
        int s = done % STAGES;
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
        asm volatile(
            "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(a), "r"(phase[s]));
        phase[s] ^= 1;
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * CH);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst_peer + cs[s] * CH),
                     "r"(d), "r"(CH)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        ++done;
        long nxt = c0 + issued * gridDim.x;
        if (nxt < nch) {
            cs[s] = nxt;
            issue(nxt, s);
            ++issued;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

struct Pair {
    int dev;
    char* local;   // on dev
    char* remote;  // on the other device
    cudaStream_t s, s2;
    cudaEvent_t a, b, j;
};

int main(int argc, char** argv) {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) {
        std::printf("need 2 GPUs\n");
        return 0;
    }
    const long bytes = 256L << 20;
    Pair P[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&P[d].local, bytes));
        CK(cudaMemset(P[d].local, 1, bytes));
        CK(cudaStreamCreateWithFlags(&P[d].s, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&P[d].s2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&P[d].j, cudaEventDisableTiming));
        CK(cudaEventCreate(&P[d].a));
        CK(cudaEventCreate(&P[d].b));
        P[d].dev = d;
    }
    char* dstbuf[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMalloc(&dstbuf[d], bytes));
    }
    P[0].remote = P[1].local;
    P[1].remote = P[0].local;
    auto cfgtma = [](auto k, int smem) { CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); };
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        cfgtma(tma_copy<32768, 4>, 32768 * 4);
        cfgtma(tma_copy<16384, 8>, 16384 * 8);
        cfgtma(tma_red_push<32768, 4>, 32768 * 4);
    }
    // op(d): run on device d against device 1-d
    auto run = [&](const char* name, auto op, bool both) {
        const int reps = 5;
        for (int warm = 0; warm < 2; ++warm) {
            for (int d = 0; d < (both ? 2 : 1); ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventRecord(P[d].a, P[d].s));
                CK(cudaEventRecord(P[d].j, P[d].s));
                CK(cudaStreamWaitEvent(P[d].s2, P[d].j, 0));
                for (int r = 0; r < (warm ? reps : 1); ++r) op(d);
                CK(cudaEventRecord(P[d].j, P[d].s2));
                CK(cudaStreamWaitEvent(P[d].s, P[d].j, 0));
                CK(cudaEventRecord(P[d].b, P[d].s));
            }
            for (int d = 0; d < (both ? 2 : 1); ++d) {
                CK(cudaSetDevice(d));
                CK(cudaStreamSynchronize(P[d].s));
            }
        }
        float ms = 0;
        for (int d = 0; d < (both ? 2 : 1); ++d) {
            float t;
            CK(cudaEventElapsedTime(&t, P[d].a, P[d].b));
            ms = t > ms ? t : ms;
        }
        std::printf("%-34s %s  %7.1f GB/s per direction\n", name, both ? "bidir" : "1-dir", bytes * reps / (ms / 1e3) / 1e9);
    };
    for (int both = 0; both < 2; ++both) {
        for (int ctas : {32, 74, 148, 296, 592}) {
            char nm[64];
            std::snprintf(nm, 64, "ldg peer read u8 ctas=%d", ctas);
            run(nm, [&](int d) { ldg_copy<8><<<ctas, 512, 0, P[d].s>>>((const uint4*)P[d].remote, (uint4*)dstbuf[d], bytes / 16); }, both);
        }
        run("ldg peer read u4 ctas=296", [&](int d) { ldg_copy<4><<<296, 512, 0, P[d].s>>>((const uint4*)P[d].remote, (uint4*)dstbuf[d], bytes / 16); }, both);
        run("ldg peer read u16 ctas=148", [&](int d) { ldg_copy<16><<<148, 256, 0, P[d].s>>>((const uint4*)P[d].remote, (uint4*)dstbuf[d], bytes / 16); }, both);
        run("ldg local copy u8 ctas=296", [&](int d) { ldg_copy<8><<<296, 512, 0, P[d].s>>>((const uint4*)P[d].local, (uint4*)dstbuf[d], bytes / 16); }, both);
        for (int ctas : {74, 148, 296})  {
            char nm[64];
            std::snprintf(nm, 64, "stg peer write ctas=%d", ctas);
            run(nm, [&](int d) { stg_fill<<<ctas, 512, 0, P[d].s>>>((uint4*)P[d].remote, bytes / 16); }, both);
        }
        for (int ctas : {74, 148, 296}) {
            char nm[64];
            std::snprintf(nm, 64, "red.v4 peer push u4 ctas=%d", ctas);
            run(nm, [&](int d) { red_push<4><<<ctas, 512, 0, P[d].s>>>((const float4*)dstbuf[d], (float*)P[d].remote, bytes / 16); }, both);
        }
        for (int ctas : {16, 32, 74, 148}) {
            char nm[64];
            std::snprintf(nm, 64, "tma bulk 32K x4 ctas=%d", ctas);
            run(nm, [&](int d) { tma_copy<32768, 4><<<ctas, 32, 32768 * 4, P[d].s>>>(P[d].remote, dstbuf[d], bytes); }, both);
            std::snprintf(nm, 64, "tma bulk 16K x8 ctas=%d", ctas);
            run(nm, [&](int d) { tma_copy<16384, 8><<<ctas, 32, 16384 * 8, P[d].s>>>(P[d].remote, dstbuf[d], bytes); }, both);
        }
        for (int ctas : {32, 74, 148}) {
            char nm[64];
            std::snprintf(nm, 64, "tma bulk-reduce push 32Kx4 ctas=%d", ctas);
            run(nm, [&](int d) { tma_red_push<32768, 4><<<ctas, 32, 32768 * 4, P[d].s>>>(dstbuf[d], P[d].remote, bytes); }, both);
        }
        // combined: each GPU fetches from the peer AND pushes to it at the same time (two streams)
        run("fetch(tma64)+push(red148) concurrent", [&](int d) {
            tma_copy<32768, 4><<<64, 32, 32768 * 4, P[d].s>>>(P[d].remote, dstbuf[d], bytes);
            red_push<4><<<148, 512, 0, P[d].s2>>>((const float4*)dstbuf[d], (float*)(P[d].remote), bytes / 16);
        }, both);
        run("fetch(tma64)+push(tmared74) concurrent", [&](int d) {
            tma_copy<32768, 4><<<64, 32, 32768 * 4, P[d].s>>>(P[d].remote, dstbuf[d], bytes);
            tma_red_push<32768, 4><<<74, 32, 32768 * 4, P[d].s2>>>(dstbuf[d], P[d].remote, bytes);
        }, both);
        run("cudaMemcpyPeerAsync pull", [&](int d) { CK(cudaMemcpyPeerAsync(dstbuf[d], d, P[d].remote, 1 - d, bytes, P[d].s)); }, both);
        run("cudaMemcpyAsync D2D pull", [&](int d) { CK(cudaMemcpyAsync(dstbuf[d], P[d].remote, bytes, cudaMemcpyDeviceToDevice, P[d].s)); }, both);
    }
    return 0;
}
