// tmem_probe.cu — microbenchmarks for the attention-backward design (B200):
//   1. tcgen05.ld throughput (TMEM -> registers) vs the number of warps
//   2. tcgen05.mma issue rate: SS (A, B in smem) at N = 128 / 256 and
//      TS (A in TMEM) at N = 128, M = 128, K = 16 per instruction, bf16
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

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

// each warp w loads rows of lane quadrant w%4, columns (w/4)*32 + k*stride ...
__global__ void ld_probe(int iters, unsigned long long* cyc, unsigned* sink) {
    __shared__ unsigned tbase;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned t = tbase;
    const int nw = blockDim.x / 32;
    const unsigned lane_base = static_cast<unsigned>((warp % 4) * 32) << 16;
    const int colgroups = nw / 4;  // warps sharing a lane quadrant split the 512 columns
    const int my_cols = 512 / colgroups;
    const unsigned col0 = static_cast<unsigned>((warp / 4) * my_cols);
    unsigned acc = 0;
    __syncthreads();
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        for (int c = 0; c < my_cols; c += 64) {
            unsigned a[32], b[32];
            TM_LD32(t + lane_base + col0 + c, a);
            TM_LD32(t + lane_base + col0 + c + 32, b);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += a[k] ^ b[k];
        }
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
    }
}

__device__ __forceinline__ std::uint64_t sdesc(unsigned addr, unsigned lbo, unsigned sbo) {
    std::uint64_t d = static_cast<std::uint64_t>((addr & 0x3FFFF) >> 4);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
__host__ __device__ constexpr unsigned instr(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((static_cast<unsigned>(n) >> 3) << 17) | ((128u >> 4) << 24);
}

// mode 0: SS N=128, 1: SS N=256, 2: TS N=128 (A from TMEM cols [256, 320));
// modes 3-5: the same three, alternating between two independent accumulators
// (D at cols 0 and 128 for N=128, 0 and 256 for N=256) instruction by instruction
__global__ void mma_probe(int iters, int mode, unsigned long long* cyc) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ unsigned tbase;
    __shared__ __align__(8) unsigned long long done;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&done)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<unsigned*>(smem)[i] = 0x3f803f80u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned t = tbase;
    if (threadIdx.x == 0) {
        const unsigned a = su32(smem), b = su32(smem + 32768);
        const int base_mode = mode % 3;
        const bool alt = mode >= 3;
        const int n = base_mode == 1 ? 256 : 128;
        const unsigned id = instr(n);
        const unsigned long long c0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const unsigned off = (kk >> 2) * 16384 + (kk & 3) * 32;
                const std::uint64_t bd = sdesc(b + off, 16, 1024);
                const unsigned acc = (i | kk) ? 1u : 0u;
                const unsigned d = t + ((alt && (kk & 1)) ? static_cast<unsigned>(n) : 0u);
                if (base_mode == 2) {
                    asm volatile(
                        "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(d),
                        "r"(t + 384 + kk * 8), "l"(bd), "r"(id), "r"(acc)
                        : "memory");
                } else {
                    const std::uint64_t ad = sdesc(a + off, 16, 1024);
                    asm volatile(
                        "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(id), "r"(acc)
                        : "memory");
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&done))
                     : "memory");
        asm volatile(
            "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], 0; @!p bra WAIT_%=; }" ::"r"(
                su32(&done))
            : "memory");
        const unsigned long long c1 = clock64();
        cyc[blockIdx.x] = c1 - c0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
    }
}

int main() {
    unsigned long long* cyc;
    unsigned* sink;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&sink, 148 * 1024 * 4);
    const int iters = 200;
    for (int threads : {128, 256, 512}) {
        ld_probe<<<148, threads>>>(iters, cyc, sink);
        cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        double bytes = 128.0 * 512 * 4 * iters;  // the whole TMEM per iteration
        printf("tcgen05.ld x32 pairs: %3d threads: %.1f cycles/iter, %.1f B/clk/SM (err %s)\n", threads,
               double(h[0]) / iters, bytes / double(h[0]), cudaGetErrorString(cudaGetLastError()));
    }
    cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const char* names[] = {"SS M128 N128 K16", "SS M128 N256 K16", "TS M128 N128 K16",
                           "SS M128 N128 K16, 2 accumulators alternating", "SS M128 N256 K16, 2 accumulators alternating",
                           "TS M128 N128 K16, 2 accumulators alternating"};
    for (int mode = 0; mode < 6; ++mode) {
        const int it = 2000;
        mma_probe<<<148, 128, 100 * 1024>>>(it, mode, cyc);
        cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        const double n = mode % 3 == 1 ? 256 : 128;
        const double per = double(h[0]) / (it * 8.0);
        printf("%s: %.1f cycles/instr, %.0f MAC/clk/SM (err %s)\n", names[mode], per, 128.0 * n * 16 / per,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
