// Per-SM throughput of the elementwise instructions of the attention backward's
// softmax/dS phase: ex2.approx.ftz.f32 (MUFU), cvt.rn.bf16x2.f32 (pack), fma.rn.f32x2,
// tcgen05-free. One CTA per SM, W warps, 8 independent chains per thread; prints
// lanes per clock per SM for each op and warp count.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_probe tools/pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void probe(float* out, long long* clk, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = 0.001f * (threadIdx.x + k);
    unsigned acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 0) {
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
            } else if (OP == 1) {
                unsigned r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[k]), "f"(a[(k + 1) & 7]));
                acc ^= r;
                a[k] = __int_as_float(__float_as_int(a[k]) ^ (r & 1));
            } else {
                float b = a[(k + 1) & 7];
                asm volatile("{\n.reg .b64 x, y;\nmov.b64 x, {%0, %1};\nfma.rn.f32x2 y, x, x, x;\nmov.b64 {%0, %1}, y;\n}"
                             : "+f"(a[k]), "+f"(b));
                a[(k + 1) & 7] = b;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* clk;
    cudaMalloc(&out, sms * 1024 * 4);
    cudaMalloc(&clk, sms * 8);
    const char* names[3] = {"ex2.approx.f32", "cvt.rn.bf16x2.f32", "fma.rn.f32x2"};
    for (int op = 0; op < 3; ++op)
        for (int w : {4, 8, 16}) {
            const int iters = 2048;
            auto k = op == 0 ? probe<0> : op == 1 ? probe<1> : probe<2>;
            k<<<sms, w * 32>>>(out, clk, iters);
            k<<<sms, w * 32>>>(out, clk, iters);
            cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
            const double ops = double(w) * 32 * iters * 8 * (op == 2 ? 2 : 1);  // lanes (f32x2 = 2 lanes)
            printf("%-20s warps/SM %2d : %.1f lanes/clk/SM (%lld clk)\n", names[op], w, ops / c, c);
        }
    return 0;
}
