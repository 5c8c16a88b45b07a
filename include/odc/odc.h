/*
 * odc.h — C ABI of the B200-native On-Demand Communication (ODC) hot path.
 *
 * Two object kinds share the same sm_100a kernels:
 *
 *  odc_fabric_t  The reference's ShardFabric<T>/ShardState<T> (one FSDP unit,
 *                all simulated ranks in this process, shards resident in HBM
 *                on one device). Host-buffer I/O, synchronous, exactly the
 *                reference's by-value semantics. Backs the drop-in C++ façade
 *                include/odcsim/primitives.hpp.
 *                  replaces inc/primitives.hpp:35-207 (ShardState, ShardFabric)
 *
 *  odc_ctx_t     The production engine: one rank per process (or host thread)
 *                per GPU, every FSDP unit (layer) of a model, owner shards in
 *                one HBM arena exported to peers with CUDA IPC handles.
 *                Device pointers, stream-ordered, asynchronous; cross-rank
 *                synchronisation is device-side only (sys-scope flags).
 *
 * Status codes map 1:1 onto the reference exception taxonomy
 * (inc/types.hpp:14-48); the façade rethrows them. No C++ exception ever
 * crosses this boundary. odc_last_error() returns a thread-local message.
 *
 * Reference paths: inc/ = /root/reference/proj/include/odcsim/,
 *                  src/ = /root/reference/proj/src/.
 */
#ifndef ODC_ODC_H
#define ODC_ODC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ODC_ABI_VERSION 5

typedef enum {
    ODC_OK = 0,
    ODC_ERR_PARAM = 2,      /* ParamError / FormatError      inc/types.hpp:14-21 */
    ODC_ERR_INFEASIBLE = 3, /* InfeasibleError                inc/types.hpp:23-27 */
    ODC_ERR_INVARIANT = 4,  /* InvariantError                 inc/types.hpp:45-48 */
    ODC_ERR_PROTOCOL = 5,   /* ProtocolError                  inc/types.hpp:35-38 */
    ODC_ERR_STATE = 6,      /* StateError                     inc/types.hpp:40-43 */
    ODC_ERR_MODE = 7,       /* ModeError                      inc/types.hpp:29-33 */
    ODC_ERR_CUDA = 8,       /* CUDA runtime failure (no reference counterpart) */
    ODC_ERR_TIMEOUT = 9,    /* device barrier watchdog fired (no reference counterpart) */
    ODC_ERR_RANGE = 10      /* FIXED push: a contribution saturated the int64 fixed-point range (no reference counterpart) */
} odc_status;

typedef enum { ODC_I64 = 0, ODC_F64 = 1, ODC_F32 = 2, ODC_BF16 = 3 } odc_dtype;

typedef enum {
    /* remote red.global.add.v4.f32 straight into the owner's fp32 gradient
     * shard over NVLink; order across clients is not fixed */
    ODC_PUSH_RED = 0,
    /* deterministic: every client owns one slot per unit AT EACH OWNER
     * (capacity = block, the reference's per-(server, client) slot,
     * inc/primitives.hpp:99-136); a push stores w*g into it over NVLink (the
     * unit's first push of the minibatch) or adds it (later pushes: single
     * writer, stream order); at the minibatch barrier the owner sums the
     * slots of the clients that pushed, in fixed rank order 0..N-1 (local
     * HBM). Memory: N * block per unit per rank. */
    ODC_PUSH_SLOT = 1,
    /* deterministic in bounded memory: each pushed w*g is rounded once to an
     * int64 fixed-point value (2^-fixed_frac_bits resolution) and added into
     * the owner's int64 accumulator with TMA bulk .add.u64 reductions over
     * NVLink; integer sums are bit-identical for any arrival order and any
     * world size; 8 B per owned element. Range |sum| < 2^(63-frac_bits). */
    ODC_PUSH_FIXED = 2
} odc_push_mode;

#define ODC_FIXED_FRAC_BITS_DEFAULT 40

int odc_abi_version(void);
const char* odc_last_error(void);
/* number of sm_100a kernel launches issued by this process so far */
uint64_t odc_kernel_launches(void);

/* ---------------------------------------------------------------------------
 * (a1) block shard layout.  inc/primitives.hpp:38-56
 *   block = ceil(elems / ranks); begin = min(elems, r*block);
 *   len = min(elems, (r+1)*block) - begin   (trailing ranks may own 0)
 * ------------------------------------------------------------------------- */
odc_status odc_shard_range(int64_t elems, int ranks, int rank, int64_t* begin, int64_t* len);

/* ---------------------------------------------------------------------------
 * Fabric: ShardFabric<T> / ShardState<T>.   inc/primitives.hpp:35-207
 * dtype in {ODC_I64, ODC_F64, ODC_F32}. `weight` points at one T.
 * ------------------------------------------------------------------------- */
typedef struct odc_fabric* odc_fabric_t;

/* ShardState(ranks, elems) :38-48 — ParamError if ranks < 1 or elems < 1 */
odc_status odc_fabric_create(int ranks, int64_t elems, odc_dtype dtype, int device, odc_fabric_t* out);
/* single-process multi-GPU: simulated rank r's shards, accumulator and server
 * slots on devices[r % ndev]; staging and kernels on devices[0], which reads
 * and writes the others' HBM through peer access over NVLink */
odc_status odc_fabric_create_multi(int ranks, int64_t elems, odc_dtype dtype, const int* devices, int ndev,
                                   odc_fabric_t* out);
odc_status odc_fabric_destroy(odc_fabric_t f);
/* scatter_accumulate strategy: ODC_PUSH_SLOT (default) = the reference's
 * staged protocol (stage into the (owner, client) slot, the owner consumes the
 * previous occupant first) — bit-exact in every dtype; ODC_PUSH_RED = remote
 * red.add straight into the owner shard (bit-exact for I64). */
odc_status odc_fabric_set_push_mode(odc_fabric_t f, odc_push_mode mode);
/* set_params :58-67 (ParamError on length mismatch); host_full has `elems` T */
odc_status odc_fabric_set_params(odc_fabric_t f, const char* id, const void* host_full, int64_t n);
/* gather :70-77 — fetch kernel concatenates the owners' shards; StateError if unset */
odc_status odc_fabric_gather(odc_fabric_t f, int client, const char* id, void* host_out);
/* scatter_accumulate :181-188 — ParamError on length mismatch */
odc_status odc_fabric_scatter_accumulate(odc_fabric_t f, int client, const void* host_grad, int64_t n,
                                         const void* weight);
/* push_slice :191-195 — ProtocolError if n > block or the slice overruns the target shard */
odc_status odc_fabric_push_slice(odc_fabric_t f, int client, int target, int64_t offset,
                                 const void* host_payload, int64_t n, const void* weight);
/* finalize_minibatch :199-203 — drains every slot in (server, client) order,
 * writes the N shards concatenated (= elems T) and zeroes them */
odc_status odc_fabric_finalize(odc_fabric_t f, void* host_out);

/* ShardState protocol steps (drivers run_schedule / run_threaded :242-359) */
odc_status odc_fabric_split_stage(odc_fabric_t f, int from, int target, int64_t offset,
                                  const void* host_payload, int64_t n, const void* weight, int* staged);
odc_status odc_fabric_slot_free(odc_fabric_t f, int server, int client, int* is_free);
odc_status odc_fabric_consume(odc_fabric_t f, int server, int client, int* did);
odc_status odc_fabric_any_staged(odc_fabric_t f, int server, int* any);
odc_status odc_fabric_take_grads(odc_fabric_t f, void* host_out);
odc_status odc_fabric_max_staged(odc_fabric_t f, int server, int64_t* peak);

/* ---------------------------------------------------------------------------
 * Engine (one rank per GPU).
 * ------------------------------------------------------------------------- */
typedef struct odc_ctx* odc_ctx_t;

typedef struct {
    int rank;
    int world;
    int device;
    int n_layers;               /* FSDP units */
    const int64_t* layer_elems; /* elements per unit, n_layers entries */
    int push_mode;              /* odc_push_mode */
    int fetch_ctas;             /* CTAs for fetch (0 = default): non-intrusive SM budget */
    int push_ctas;              /* CTAs for push  (0 = default) */
    double timeout_s;           /* device barrier watchdog (<= 0: 60 s) */
    int fetch_engine;           /* odc_fetch_engine */
    int fixed_frac_bits;        /* ODC_PUSH_FIXED resolution 2^-bits (0 = default 40; 8..60) */
} odc_config;

typedef enum {
    ODC_FETCH_TMA = 0, /* sm_100a kernel: cp.async.bulk peer->smem->local pipeline (default) */
    ODC_FETCH_LDG = 1, /* sm_100a kernel: 16-byte vector peer loads, chunked */
    ODC_FETCH_CE = 2   /* copy engines (cudaMemcpyAsync per owner) after a device gate kernel */
} odc_fetch_engine;

odc_status odc_ctx_create(const odc_config* cfg, odc_ctx_t* out);
odc_status odc_ctx_destroy(odc_ctx_t ctx);
/* IPC blob describing this rank's HBM arena (cudaIpcMemHandle + layout hash) */
odc_status odc_ctx_export(odc_ctx_t ctx, void* blob, size_t cap, size_t* len);
odc_status odc_ctx_import(odc_ctx_t ctx, int peer, const void* blob, size_t len);
/* single-process mode: map peer `peer`'s arena from its context living in
 * this process (same device: several ranks on one GPU, for protocol tests;
 * another device: direct peer access over NVLink, enabled here). Same layout
 * checks as odc_ctx_import. */
odc_status odc_ctx_import_ctx(odc_ctx_t ctx, int peer, odc_ctx_t peer_ctx);
/* after every peer was imported: builds the device pointer tables */
odc_status odc_ctx_ready(odc_ctx_t ctx);
/* bytes of HBM the arena holds on this rank */
odc_status odc_ctx_arena_bytes(odc_ctx_t ctx, int64_t* bytes);

/* set_params: copy this rank's owned slice [begin, begin+len) of the full
 * fp32 unit `src_full` (device) into the owner's fp32 master + bf16 shard. */
odc_status odc_set_params(odc_ctx_t ctx, int layer, const float* src_full, void* stream);
/* (a3) fetch: dst_full (bf16, elems) = concat of all owners' bf16 shards;
 * waits (device-side) for each owner's current parameter epoch. */
odc_status odc_fetch(odc_ctx_t ctx, int layer, void* dst_full_bf16, void* stream);
/* fetch variant returning fp32 masters (parity / debugging) */
odc_status odc_fetch_master(odc_ctx_t ctx, int layer, float* dst_full, void* stream);
/* (a6) push: owner_grad += weight * grad_full[owner range] for every owner.
 * grad dtype ODC_F32 or ODC_BF16. */
odc_status odc_push(odc_ctx_t ctx, int layer, const void* grad_full, int grad_dtype, float weight,
                    void* stream);
/* (a7) push_slice: ProtocolError if n > block or offset+n > shard_len(target) */
odc_status odc_push_slice(odc_ctx_t ctx, int layer, int target, int64_t offset, const float* payload,
                          int64_t n, float weight, void* stream);
/* (a8) minibatch barrier: signal every owner, wait for every client, then
 * (slot mode) reduce the per-source slots in rank order into the grad shard,
 * (fixed mode) convert the int64 sums into it. The grad shards then hold the
 * minibatch's sums until the next AdamW step or the rank's next fetch / push /
 * minibatch_end, which consume (zero) them like take_grads (:144-148): read
 * them with odc_read_grad_shard before (stream-ordered) that next call.
 * Peers' pushes of the next minibatch wait device-side for that drain. */
odc_status odc_minibatch_end(odc_ctx_t ctx, void* stream);
/* read this rank's accumulated fp32 grad shard of `layer` (len = shard_len) */
odc_status odc_read_grad_shard(odc_ctx_t ctx, int layer, float* dst, void* stream);
odc_status odc_read_master_shard(odc_ctx_t ctx, int layer, float* dst, void* stream);

typedef struct {
    float lr, beta1, beta2, eps, weight_decay;
    int step; /* 1-based, for bias correction */
} odc_adam_cfg;
/* (a19) fused AdamW over every owned shard (fp32 master/m/v, bf16 shard out),
 * zeroes the grad shards, then publishes the new parameter epoch. (The slot
 * mode's rank-order reduce already ran in odc_minibatch_end.) */
odc_status odc_adam_step(odc_ctx_t ctx, const odc_adam_cfg* cfg, void* stream);
/* host check of the device error word; blocks on `stream`. ODC_ERR_TIMEOUT
 * (watchdog) or ODC_ERR_RANGE (FIXED push saturation / NaN) */
odc_status odc_ctx_check(odc_ctx_t ctx, void* stream);
/* raw sticky device flags: bit0 timeout, bit1 FIXED range error,
 * bit2 FIXED underflow warning (a nonzero w*g rounded to 0); blocks on `stream` */
odc_status odc_ctx_flags(odc_ctx_t ctx, uint64_t* flags, void* stream);
/* current minibatch epoch (number of completed odc_minibatch_end calls) */
int64_t odc_ctx_epoch(odc_ctx_t ctx);

/* ---------------------------------------------------------------------------
 * Raw kernels on caller-owned device memory (bench / FSDP comparison path).
 * ------------------------------------------------------------------------- */
/* multi-segment copy (16B vector path when src ≡ dst mod 16) */
odc_status odc_copy_segments(int nseg, const void* const* srcs, void* const* dsts, const int64_t* bytes,
                             int ctas, void* stream);
/* L2 flush helper for timing hygiene: writes `bytes` of scratch */
odc_status odc_l2_flush(void* scratch, int64_t bytes, void* stream);

/* ---------------------------------------------------------------------------
 * bf16 GEMM on tcgen05 tensor cores (worker dense layers; no reference
 * counterpart — the reference only models their cost, src/cost_model.cpp).
 *   D[M,N] (+)= A · B^T with fp32 accumulation in TMEM
 *   A stored [M][K] (a_mn_major = 0) or [K][M] (a_mn_major = 1), pitch lda
 *   B stored [N][K] (b_mn_major = 0) or [K][N] (b_mn_major = 1), pitch ldb
 *   D row-major [M][ldd], d_dtype ODC_BF16 or ODC_F32; accumulate: D += A·B^T;
 *   C (optional, bf16 output only): D = A·B^T + C, C with D's shape and ldd (fused residual)
 * fwd  X·W^T : a=X [T][in] K-major,  b=W [out][in] K-major
 * dgrad dY·W : a=dY [T][out] K-major, b=W [out][in] N-major
 * wgrad dY^T·X: a=dY [T][out] M-major, b=X [T][in] N-major
 * ------------------------------------------------------------------------- */
odc_status odc_gemm_bf16(const void* A, const void* B, void* D, const void* C, int64_t M, int64_t N, int64_t K,
                         int64_t lda, int64_t ldb, int64_t ldd, int a_mn_major, int b_mn_major, int d_dtype,
                         int accumulate, void* stream);

/* GEMM tile raster (L2 reuse; tuning / A-B only): group = M-tiles per raster
 * group (0 = automatic from the L2 budget), l2_budget_mb (0 = keep). */
odc_status odc_gemm_set_raster(int group, int l2_budget_mb);

/* gate/up projection with SwiGLU fused into the epilogue (2-CTA tcgen05 GEMM):
 * gu [T][2*ffn] = X [T][d] · W^T with W = [gate; up] [2*ffn][d] (as odc_gemm_bf16),
 * and m [T][ffn] = silu(gate) * up computed from the bf16-rounded gu values
 * (bit-identical to odc_w_swiglu_fwd). Output tile n pairs gate rows
 * [128n, 128n+128) with up rows ffn + [128n, 128n+128). ffn % 128 == 0. */
odc_status odc_gemm_gate_up_swiglu(const void* X, const void* W, void* gu, void* m, int64_t T, int64_t ffn, int64_t d,
                                   void* stream);

/* Causal varlen flash-attention forward on tcgen05 (head_dim 128, GQA).
 * q [T][H][128], k/v [T][KV][128] bf16; out [T][H][128]; lse [H][T] fp32 (natural log).
 * items: n_items x {seq_start, seq_len, q_tile, head} (int32 x4), one CTA each;
 * order heaviest (most KV tiles) first. */
odc_status odc_attn_fwd(const void* q, const void* k, const void* v, void* out, float* lse, const void* items,
                        int n_items, int64_t T, int H, int KV, int head_dim, float scale, void* stream);
/* Backward: dq [T][H][128], dk / dv [T][KV][128] bf16 from q, k, v, o, dout and the forward's lse.
 * items: int32 x8 {seq_start, seq_len, kv_tile, kv_head, it_begin, it_end, 0, 0} (one CTA each,
 * heaviest first; iterations n in [it_begin, it_end) of (head-in-group = n / tiles, q tile = kv_tile + n % tiles));
 * workspace: fp32, roundup(H*T, 64) + T*H*128 + 2*T*KV*128 elements, 16-byte aligned. */
odc_status odc_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                        const float* lse, void* dq, void* dk, void* dv, void* workspace, const void* items,
                        int n_items, int64_t T, int H, int KV, int head_dim, float scale, void* stream);

/* The backward straight to the packed qkv gradient: dqkv [T][(H+2KV)*128] bf16 = (dq, dk, dv)
 * with the inverse RoPE (table / pos as odc_w_qkv_rope_bwd) applied to the q and k heads;
 * bit-identical to odc_attn_bwd followed by odc_w_qkv_rope_bwd, one pass instead of four. */
odc_status odc_attn_bwd_qkv(const void* q, const void* k, const void* v, const void* o, const void* dout,
                            const float* lse, const void* table, const int64_t* pos, void* dqkv, void* workspace,
                            const void* items, int n_items, int64_t T, int H, int KV, int head_dim, float scale,
                            void* stream);

/* ---------------------------------------------------------------------------
 * Fused elementwise kernels of the SFT worker (csrc/worker_kernels.cu).
 * bf16 tensors row-major and 16-byte aligned; fp32 for rstd / dw / loss.
 * ------------------------------------------------------------------------- */
odc_status odc_w_rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, int64_t T, int d, float eps,
                             void* stream);
/* out = resid (optional) + dx; dw += sum over rows of dy * x * rstd */
odc_status odc_w_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd, const void* resid,
                             void* out, float* dw, int64_t T, int d, void* stream);
/* packed qkv [T][(H+2KV)hd] (+bias) -> q [T][H][hd], k, v [T][KV][hd], RoPE on q,k;
 * table = float2 {cos, sin} [max_pos][hd/2] */
odc_status odc_w_qkv_rope_fwd(const void* qkv, const void* bias, const void* table, const int64_t* pos, void* q,
                              void* k, void* v, int64_t T, int H, int KV, int hd, void* stream);
odc_status odc_w_qkv_rope_bwd(const void* dq, const void* dk, const void* dv, const void* table, const int64_t* pos,
                              void* dqkv, int64_t T, int H, int KV, int hd, void* stream);
/* out[j] += sum_t m[t][j] (fp32) */
odc_status odc_w_col_sum(const void* m, float* out, int64_t T, int n, void* stream);
odc_status odc_w_swiglu_fwd(const void* gu, void* m, int64_t T, int ffn, void* stream);
odc_status odc_w_swiglu_bwd(const void* dm, const void* gu, void* dgu, int64_t T, int ffn, void* stream);
/* logits [rows][vocab] bf16 overwritten by (softmax - onehot) * scale (0 for label < 0);
 * *loss += sum over labelled rows of (logsumexp - logit[label]) */
odc_status odc_w_ce_fwd_bwd(void* logits, const int64_t* labels, int64_t rows, int64_t vocab, float scale,
                            float* loss, void* stream);

/* ---------------------------------------------------------------------------
 * Load balancer (host C++, bit-exact restatement).  src/partition.cpp
 * strategy: 0 local-sort, 1 lb-micro, 2 lb-mini, 3 verl-native, 4 verl-optimized
 * ------------------------------------------------------------------------- */
/* plan() :490-580 serialised as solutions_to_json() (src/experiment.cpp:215-233),
 * byte-identical to nlohmann::json::dump(). *needed = bytes incl. NUL. */
odc_status odc_plan_json(int strategy, const int64_t* lens, int64_t n, int devices, int minibs,
                         int64_t budget, double alpha, double beta, int layers, uint64_t seed, char* out,
                         int64_t cap, int64_t* needed);
/* flat plan: for each step s, device d, microbatch m: the sample ids.
 * Layout (int64): [n_steps, then per step: n_dev, per dev: n_mb, per mb: n_ids, ids...]
 * *needed = int64 words required. */
odc_status odc_plan_flat(int strategy, const int64_t* lens, int64_t n, int devices, int minibs,
                         int64_t budget, double alpha, double beta, uint64_t seed, int64_t* out, int64_t cap,
                         int64_t* needed);
/* kk_partition :84-128 as JSON {"parts":..,"sums":..,"spread":..} */
odc_status odc_kk_partition_json(const double* costs, int n, int k, int equal_size, char* out, int64_t cap,
                                 int64_t* needed);
/* generate_synthetic + scale_lengths (src/workload.cpp:218-271);
 * dist 0 lognormal(p1=mu,p2=sigma) 1 pareto(scale,shape) 2 uniform(lo,hi) */
odc_status odc_generate_synthetic(int dist, double p1, double p2, int64_t n, int64_t cap, uint64_t seed,
                                  double scale, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* ODC_ODC_H */
