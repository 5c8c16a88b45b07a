// kernels.cuh — launch interface of the ODC sm_100a kernels (odc_kernels.cu).
// Every launcher is stream-ordered and bumps the process launch counter.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace odc {

constexpr int kMaxSeg = 16;  // max ranks on one NVSwitch box we size tables for

// Byte segments (fetch / set_params / read-back). src ≡ dst (mod 16) takes
// the 16-byte vector path; any other pair falls back to 4/2/1-byte moves.
struct SegTable {
    int n = 0;
    const char* src[kMaxSeg];
    char* dst[kMaxSeg];
    std::int64_t bytes[kMaxSeg];
    // optional per-segment readiness gate: wait until *gate[i] >= need (sys scope)
    const unsigned long long* gate[kMaxSeg];
    unsigned long long need = 0;
    unsigned long long* err = nullptr;  // device error word (watchdog)
    long long timeout_ns = 0;
};

// fp32 reduction segments for push: dst[i] += w * src[i]
struct RedTable {
    int n = 0;
    const void* src[kMaxSeg];  // grad slice (fp32 or bf16)
    float* dst[kMaxSeg];       // owner's fp32 grad shard (peer memory)
    std::int64_t elems[kMaxSeg];
    const unsigned long long* gate[kMaxSeg];
    unsigned long long need = 0;
    unsigned long long* err = nullptr;
    long long timeout_ns = 0;
};

// bulk-reduction push segments: FIXED dst[i] += rn(w * src[i] * 2^S) in
// int64, F32 dst[i] += w * src[i] in fp32 (TMA bulk reduce into peer memory)
struct BulkTable {
    int n = 0;
    const void* src[kMaxSeg];  // grad slice (fp32 or bf16)
    void* dst[kMaxSeg];        // owner's int64 accumulator / fp32 grad shard / fp32 slot (peer memory)
    std::int64_t elems[kMaxSeg];
    const unsigned long long* gate[kMaxSeg];
    unsigned long long need = 0;
    unsigned long long* err = nullptr;
    long long timeout_ns = 0;
    bool assign[kMaxSeg] = {};                 // F32: store w*g instead of adding it (SLOT first push)
    unsigned long long* mark[kMaxSeg] = {};    // optional: *mark[i] = mark_value (st.relaxed.sys, block 0)
    unsigned long long mark_value = 0;
};
constexpr int kMaxFinal = 64;
struct FixFinal {
    int n = 0;
    float* grad[kMaxFinal];
    long long* acc[kMaxFinal];
    std::int64_t elems[kMaxFinal];
};

// device error word: a bit mask (sticky until the context is recreated)
enum : unsigned long long {
    kErrNone = 0,
    kErrTimeout = 1,          // watchdog: a peer never reached a barrier / never published an epoch
    kErrFixedRange = 2,       // FIXED push: a contribution saturated the int64 range or was NaN/Inf
    kWarnFixedUnderflow = 4   // FIXED push: a nonzero contribution rounded to 0 (resolution, not an error)
};

std::uint64_t launches();
void count_launch();

cudaError_t launch_copy_segments(const SegTable& t, int ctas, cudaStream_t s);
// fetch engine: TMA bulk peer->smem->local pipeline, every CTA round-robins a
// slice of every segment (all owners served concurrently)
cudaError_t launch_fetch_tma(const SegTable& t, int ctas, cudaStream_t s);
// push, RED mode: remote red.relaxed.sys.global.add(.v4).f32 into owner shards
cudaError_t launch_push_red(const RedTable& t, float w, bool src_bf16, int ctas, cudaStream_t s);
// push through TMA bulk reductions (cp.reduce.async.bulk): FIXED mode
// (deterministic, bounded memory) adds rn(w*g*scale) into every owner's int64
// accumulator; otherwise (RED mode) w*g into the owner's fp32 grad shard
cudaError_t launch_push_bulk(const BulkTable& t, bool fixed, float w, float scale, bool src_bf16, int ctas,
                             cudaStream_t s);
// SLOT mode owner reduce (after the barrier): for every unit u,
// dst[u][i] = sum over clients c (rank order) with marks[u][c] == epoch of
// slot0[u][c * slot_stride[u] + i]; 0 if no client pushed the unit
constexpr int kMaxReduceUnits = 48;
struct SlotReduce {
    int n = 0;
    int nsrc = 0;
    unsigned long long epoch = 0;
    float* dst[kMaxReduceUnits];
    const float* slot0[kMaxReduceUnits];
    std::int64_t slot_stride[kMaxReduceUnits];
    std::int64_t elems[kMaxReduceUnits];
    const unsigned long long* marks[kMaxReduceUnits];
};
cudaError_t launch_slot_reduce(const SlotReduce& r, cudaStream_t s);
// owner, after the barrier: grad[i] = fl(acc[i]) * inv_scale; acc[i] = 0
cudaError_t launch_fixed_finalize(const FixFinal& f, float inv_scale, cudaStream_t s);

// ---- the generic typed kernels behind the reference-semantics fabric ----
// dst[i] = dst[i] + w * src[i]   (one multiply, one add, each rounded; no FMA)
template <typename T>
cudaError_t launch_accumulate(T* dst, const T* src, std::int64_t n, T w, cudaStream_t s);
// dst[i] atomically += w * src[i]  (red.global.add: u64 / f64 / f32)
template <typename T>
cudaError_t launch_red_accumulate(T* dst, const T* src, std::int64_t n, T w, cudaStream_t s);

// ---- barrier / flags ----
// thread t < world: st.release.sys peer_done[t][my_slot] = epoch;
// then thread t < world spins ld.acquire.sys my_done[t] >= epoch.
struct BarrierArgs {
    int world = 1;
    int rank = 0;
    unsigned long long* peer_done[kMaxSeg];  // owner t's done array base
    const unsigned long long* my_done = nullptr;
    unsigned long long epoch = 0;
    unsigned long long* err = nullptr;
    long long timeout_ns = 0;
};
cudaError_t launch_barrier(const BarrierArgs& a, cudaStream_t s);
// st.release.sys *flag = value (after everything earlier on the stream);
// optionally a second flag in the same launch
cudaError_t launch_publish(unsigned long long* flag, unsigned long long value, cudaStream_t s,
                           unsigned long long* flag2 = nullptr, unsigned long long value2 = 0);
// wait for every gate >= need, then zero `n` floats at each of `ptrs`
cudaError_t launch_gated_zero(float* const* ptrs, const std::int64_t* n, int count,
                              const unsigned long long* const* gates, int ngates, unsigned long long need,
                              unsigned long long* err, long long timeout_ns, cudaStream_t s);

// ---- fused AdamW over owned shards ----
struct AdamSeg {
    float* master;
    float* m;
    float* v;
    float* grad;              // fp32 grad shard (zeroed after use)
    unsigned short* param;    // bf16 shard out
    std::int64_t n;
};
struct AdamArgs {
    const AdamSeg* segs = nullptr;  // device array
    int nseg = 0;
    const std::int64_t* seg_start = nullptr;  // device prefix of 4-element vector counts (nseg+1)
    float lr, beta1, beta2, eps, wd;
    float step_size;     // lr / (1 - beta1^t)
    float bc2_sqrt_inv;  // 1 / sqrt(1 - beta2^t)
};
cudaError_t launch_adam(const AdamArgs& a, std::int64_t total_vec_units, int ctas, cudaStream_t s);

cudaError_t launch_l2_flush(void* scratch, std::int64_t bytes, cudaStream_t s);
// force-load every protocol kernel into the current context (see odc_kernels.cu)
cudaError_t preload_kernels();
// owner init: master[i] = src[i]; param[i] = bf16_rn(src[i])
cudaError_t launch_init_shard(float* master, unsigned short* param, const float* src, std::int64_t n, cudaStream_t s);

}  // namespace odc
