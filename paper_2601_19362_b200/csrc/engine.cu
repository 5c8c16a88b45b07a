// engine.cu — odc_ctx_t: the production ODC engine, one rank per GPU.
//
// HBM arena (one cudaMalloc per rank, exported once with cudaIpcGetMemHandle,
// identical layout on every rank so peers can address each other's shards):
//
//   [flags page 4 KB]  done[r] u64 (written by client r at the barrier),
//                      param_epoch u64 (owner publishes after AdamW), err u64
//                      (bit mask), drain_epoch u64 (push-target reuse gate)
//   per FSDP unit l, this rank's owned shard (block_l = ceil(M_l / N)):
//     param  bf16 [block+8]  stored at pad = begin % 8   (co-aligned with the
//     grad   f32  [block+4]  stored at pad = begin % 4    caller's full-layer
//     master f32  [block+4]                               buffers, so fetch
//     m, v   f32  [block+4]                               and push run the
//     slot   f32  [N][block+4] (SLOT push mode only)      16-byte vector path)
//                            owner-side slot of every client, same padding
//     acc    i64  [block+2]  (FIXED push mode only) stored at pad = begin % 2
//
// Mapping onto the reference (inc/ = /root/reference/proj/include/odcsim/):
//   layout          ShardState ctor/shard_begin/shard_len     inc/primitives.hpp:38-56
//   odc_set_params  ShardState::set_params                    :58-67
//   odc_fetch       ShardState::gather                        :70-77
//   odc_push        ShardFabric::scatter_accumulate           :181-188
//   odc_push_slice  ShardFabric::push_slice (ProtocolError)   :191-195, :105-112
//   odc_minibatch_end + odc_read_grad_shard
//                   ShardFabric::finalize_minibatch/take_grads :199-203, :144-148
//   odc_adam_step   (no reference counterpart: the reference only accumulates)
//
// Ordering protocol (all device-side, sys scope). The waits run in one small
// gate kernel per stream and epoch (odc_ctx::gate), never inside the data-path
// kernels, so a waiting rank holds no SMs a peer on the same GPU may need:
//   * fetch of owner r's shard waits param_epoch[r] >= adams completed here;
//   * every push into owner r waits drain_epoch[r] >= minibatches completed
//     here: the owner has consumed what the previous minibatch left in its
//     push target and published that with st.release.sys:
//       RED    grad shard zeroed — by AdamW, or (no AdamW in between) by the
//              owner's first ODC call of the next minibatch, after the caller
//              read the shard (finalize_minibatch returns + zeroes, :144-148);
//       SLOT   the owner's rank-order reduce of every client's slot finished
//              (a client's first push of a unit overwrites its slot);
//       FIXED  int64 sums converted to the fp32 grad shard and zeroed, right
//              after the barrier;
//     so correctness never depends on an AdamW step between minibatches;
//   * minibatch_end: fence.acq_rel.sys, st.release.sys done[rank] into every
//     owner, then waits ld.acquire.sys done[c] >= epoch for every client c;
//   * AdamW then st.release.sys param_epoch = ++adams.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"

namespace odc {
namespace {
thread_local std::string t_last_error;
}
void set_last_error(const std::string& msg) { t_last_error = msg; }
}  // namespace odc

namespace {

using odcsim::ParamError;
using odcsim::ProtocolError;
using odcsim::StateError;

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Makes `d` the current device for one API call and restores the caller's device on return, so a
// call on one rank's context never leaves another device current behind the caller (e.g. torch).
class DeviceGuard {
  public:
    explicit DeviceGuard(int d) {
        if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
        if (prev_ != d) cuda_ok(cudaSetDevice(d), "cudaSetDevice");
    }
    ~DeviceGuard() {
        if (prev_ >= 0) cudaSetDevice(prev_);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;

  private:
    int prev_ = -1;
};

constexpr std::int64_t kFlagsBytes = 4096;
constexpr std::int64_t kDoneOff = 0;
constexpr std::int64_t kEpochOff = 1024;
constexpr std::int64_t kErrOff = 2048;
constexpr std::int64_t kDrainOff = 3072;  // last minibatch whose push target the owner has consumed
constexpr std::uint64_t kBlobMagic = 0x4f44433142323030ULL;  // "ODC1B200"

std::int64_t round256(std::int64_t x) { return (x + 255) / 256 * 256; }

struct Unit {
    std::int64_t elems = 0, block = 0;
    std::int64_t off_param = 0, off_grad = 0, off_master = 0, off_m = 0, off_v = 0, off_slot = -1, off_acc = -1;
    std::int64_t slot_stride = 0;  // bytes between two clients' slots (SLOT mode)
    std::int64_t begin(int r) const { return std::min<std::int64_t>(elems, static_cast<std::int64_t>(r) * block); }
    std::int64_t len(int r) const { return std::min<std::int64_t>(elems, static_cast<std::int64_t>(r + 1) * block) - begin(r); }
};

struct Blob {
    std::uint64_t magic;
    std::int32_t rank, world;
    std::int64_t arena_bytes;
    std::uint64_t layout_hash;
    cudaIpcMemHandle_t handle;
};

}  // namespace

struct odc_ctx {
    odc_config cfg{};
    std::vector<Unit> units;
    std::int64_t arena_bytes = 0;
    std::uint64_t layout_hash = 0;
    char* arena = nullptr;
    std::vector<char*> peer;  // peer[r] = r's arena mapped here (peer[rank] = arena)
    std::vector<bool> imported;
    std::vector<bool> local_peer;  // mapped from a context of this process (odc_ctx_import_ctx): not an IPC mapping
    bool ready = false;
    long long timeout_ns = 60LL * 1000 * 1000 * 1000;
    std::uint64_t mb_epoch = 0;  // completed minibatch_end calls
    std::uint64_t adams = 0;     // completed adam steps (published param epochs)
    std::vector<char> touched;   // SLOT: [unit][owner] this client wrote its slot at the owner this minibatch
    std::int64_t off_marks = -1;  // SLOT: [unit][client] u64 "pushed in minibatch" marks (owner side)
    bool grads_pending = false;  // RED: the grad shards hold a finished minibatch not yet consumed
    // The waits live in one tiny gate kernel instead of the data-path kernels, so a waiting rank
    // never holds SMs that the rank it waits for needs (several ranks per GPU in one process).
    // Per kind (0 parameter epoch, 1 drain epoch): the epoch the last gate kernel waited for and
    // an event recorded right after it; a later call for the same epoch on any stream just waits
    // on that event (no kernel, and correct for streams created after the gate).
    std::uint64_t gate_need[2] = {0, 0};
    bool gate_issued[2] = {false, false};
    cudaEvent_t gate_ev[2] = {nullptr, nullptr};
    odc::AdamSeg* d_segs = nullptr;
    std::int64_t* d_seg_start = nullptr;
    std::int64_t adam_units = 0;

    int world() const { return cfg.world; }
    int rank() const { return cfg.rank; }
    bool slot_mode() const { return cfg.push_mode == ODC_PUSH_SLOT; }
    bool fixed_mode() const { return cfg.push_mode == ODC_PUSH_FIXED; }
    float fixed_scale() const { return std::ldexp(1.0f, cfg.fixed_frac_bits); }

    char* at(int r, std::int64_t off) const { return peer[static_cast<std::size_t>(r)] + off; }
    unsigned long long* done_of(int r) const { return reinterpret_cast<unsigned long long*>(at(r, kDoneOff)); }
    unsigned long long* epoch_of(int r) const { return reinterpret_cast<unsigned long long*>(at(r, kEpochOff)); }
    unsigned long long* drain_of(int r) const { return reinterpret_cast<unsigned long long*>(at(r, kDrainOff)); }
    unsigned long long* err() const { return reinterpret_cast<unsigned long long*>(arena + kErrOff); }
    // element 0 of owner r's shard of unit u in each array
    unsigned short* param_of(int r, const Unit& u) const {
        return reinterpret_cast<unsigned short*>(at(r, u.off_param)) + u.begin(r) % 8;
    }
    float* f32_of(int r, std::int64_t off, const Unit& u) const {
        return reinterpret_cast<float*>(at(r, off)) + u.begin(r) % 4;
    }
    // SLOT mode: client c's slot at owner r (co-aligned like the grad shard) and its mark
    float* slot_of(int r, const Unit& u, int client) const {
        return reinterpret_cast<float*>(at(r, u.off_slot + client * u.slot_stride)) + u.begin(r) % 4;
    }
    unsigned long long* mark_of(int r, int layer, int client) const {
        return reinterpret_cast<unsigned long long*>(at(r, off_marks)) + static_cast<std::int64_t>(layer) * world() + client;
    }
    char& touched_at(int layer, int owner) {
        return touched[static_cast<std::size_t>(layer) * static_cast<std::size_t>(world()) + static_cast<std::size_t>(owner)];
    }
    // FIXED mode int64 accumulator: element parity == global index parity
    long long* acc_of(int r, const Unit& u) const {
        return reinterpret_cast<long long*>(at(r, u.off_acc)) + u.begin(r) % 2;
    }
    const Unit& unit(int l) const {
        if (l < 0 || l >= static_cast<int>(units.size())) throw ParamError("layer index out of range");
        return units[static_cast<std::size_t>(l)];
    }
    void need_ready() const {
        if (!ready) throw StateError("odc context used before odc_ctx_ready()");
    }
    int dev_id() const { return cfg.device; }
    bool red_mode() const { return cfg.push_mode == ODC_PUSH_RED; }
    // RED: the caller is done with last minibatch's grad shards (this is the
    // next ODC call after odc_minibatch_end without an AdamW step): zero them
    // and let peers push again
    void drain_pending(cudaStream_t s) {
        if (!grads_pending) return;
        std::vector<float*> ptrs;
        std::vector<std::int64_t> cnt;
        for (const Unit& u : units)
            if (u.len(rank()) > 0) {
                ptrs.push_back(f32_of(rank(), u.off_grad, u));
                cnt.push_back(u.len(rank()));
            }
        if (!ptrs.empty())
            cuda_ok(odc::launch_gated_zero(ptrs.data(), cnt.data(), static_cast<int>(ptrs.size()), nullptr, 0, 0, err(),
                                           timeout_ns, s),
                    "zero grad shards");
        cuda_ok(odc::launch_publish(drain_of(rank()), mb_epoch, s), "publish drain epoch");
        grads_pending = false;
    }
    // Wait (device-side, one 32-thread block) until every owner's parameter epoch
    // >= adams (param = true: fetch) or drain epoch >= mb_epoch (push), once per
    // stream and epoch.
    void gate(bool param, cudaStream_t s) {
        const int k = param ? 0 : 1;
        const std::uint64_t need = param ? adams : mb_epoch;
        if (need == 0) return;  // epoch 0 is every flag's initial value
        if (gate_issued[k] && gate_need[k] >= need) {
            cuda_ok(cudaStreamWaitEvent(s, gate_ev[k], 0), "wait gate");
            return;
        }
        const unsigned long long* g[odc::kMaxSeg];
        for (int r = 0; r < world(); ++r) g[r] = param ? epoch_of(r) : drain_of(r);
        cuda_ok(odc::launch_gated_zero(nullptr, nullptr, 0, g, world(), need, err(), timeout_ns, s), "gate");
        if (!gate_ev[k]) cuda_ok(cudaEventCreateWithFlags(&gate_ev[k], cudaEventDisableTiming), "gate event");
        cuda_ok(cudaEventRecord(gate_ev[k], s), "record gate");
        gate_need[k] = need;
        gate_issued[k] = true;
    }
    // rotation: rank r visits owners r+1, r+2, ..., r so that concurrent
    // fetches/pushes from all ranks spread over all owners' links
    int owner_at(int i) const { return (rank() + 1 + i) % world(); }
};

namespace {

odc_ctx* C(odc_ctx_t c) {
    if (!c) throw ParamError("null odc context");
    return c;
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// fetch engine dispatch (odc_fetch_engine)
void launch_fetch(const odc_ctx* c, const odc::SegTable& t, cudaStream_t s) {
    switch (c->cfg.fetch_engine) {
        case ODC_FETCH_LDG: cuda_ok(odc::launch_copy_segments(t, c->cfg.fetch_ctas, s), "fetch (ldg)"); return;
        case ODC_FETCH_CE: {  // the owners' epochs were awaited by the stream's gate kernel (odc_ctx::gate)
            for (int i = 0; i < t.n; ++i)
                if (t.bytes[i] > 0)
                    cuda_ok(cudaMemcpyAsync(t.dst[i], t.src[i], static_cast<std::size_t>(t.bytes[i]),
                                            cudaMemcpyDeviceToDevice, s),
                            "fetch (ce)");
            return;
        }
        default: {
            // all-local fetch (N=1) is HBM-bound: give it the whole GPU; over
            // NVLink 64 CTAs already saturate the link (profiles/r01/p2p_*)
            const int ctas = c->cfg.fetch_ctas > 0 ? c->cfg.fetch_ctas : (c->world() == 1 ? 148 : 64);
            cuda_ok(odc::launch_fetch_tma(t, ctas, s), "fetch (tma)");
        }
    }
}

}  // namespace

extern "C" {

int odc_abi_version(void) { return ODC_ABI_VERSION; }
const char* odc_last_error(void) { return odc::t_last_error.c_str(); }
std::uint64_t odc_kernel_launches(void) { return odc::launches(); }

odc_status odc_shard_range(std::int64_t elems, int ranks, int rank, std::int64_t* begin, std::int64_t* len) {
    return odc::guard([&] {
        if (ranks < 1 || elems < 1) throw ParamError("need ranks >= 1 and elems >= 1");
        if (rank < 0 || rank >= ranks) throw ParamError("rank out of range");
        const std::int64_t block = (elems + ranks - 1) / ranks;
        const std::int64_t b = std::min<std::int64_t>(elems, static_cast<std::int64_t>(rank) * block);
        *begin = b;
        *len = std::min<std::int64_t>(elems, static_cast<std::int64_t>(rank + 1) * block) - b;
    });
}

odc_status odc_ctx_create(const odc_config* cfg, odc_ctx_t* out) {
    return odc::guard([&] {
        if (!cfg || !out) throw ParamError("null config");
        if (cfg->world < 1 || cfg->world > odc::kMaxSeg) throw ParamError("world must be 1..16");
        if (cfg->rank < 0 || cfg->rank >= cfg->world) throw ParamError("rank out of range");
        if (cfg->n_layers < 1 || !cfg->layer_elems) throw ParamError("need at least one FSDP unit");
        if (cfg->push_mode != ODC_PUSH_RED && cfg->push_mode != ODC_PUSH_SLOT && cfg->push_mode != ODC_PUSH_FIXED)
            throw ParamError("bad push mode");
        if (cfg->fixed_frac_bits != 0 && (cfg->fixed_frac_bits < 8 || cfg->fixed_frac_bits > 60))
            throw ParamError("fixed_frac_bits must be 0 (default) or 8..60");
        if (cfg->fetch_engine < ODC_FETCH_TMA || cfg->fetch_engine > ODC_FETCH_CE) throw ParamError("bad fetch engine");
        auto* c = new odc_ctx();
        try {
            c->cfg = *cfg;
            c->cfg.layer_elems = nullptr;
            if (c->cfg.fixed_frac_bits == 0) c->cfg.fixed_frac_bits = ODC_FIXED_FRAC_BITS_DEFAULT;
            if (cfg->timeout_s > 0) c->timeout_ns = static_cast<long long>(cfg->timeout_s * 1e9);
            std::int64_t off = kFlagsBytes;
            std::uint64_t h = 1469598103934665603ULL;
            auto mix = [&](std::uint64_t v) { h = (h ^ v) * 1099511628211ULL; };
            mix(static_cast<std::uint64_t>(cfg->world));
            mix(static_cast<std::uint64_t>(cfg->push_mode));
            mix(static_cast<std::uint64_t>(c->cfg.fixed_frac_bits));
            for (int l = 0; l < cfg->n_layers; ++l) {
                Unit u;
                u.elems = cfg->layer_elems[l];
                if (u.elems < 1) throw ParamError("every FSDP unit needs elems >= 1");
                u.block = (u.elems + cfg->world - 1) / cfg->world;
                mix(static_cast<std::uint64_t>(u.elems));
                u.off_param = off;
                off += round256((u.block + 8) * 2);
                const std::int64_t f32 = round256((u.block + 4) * 4);
                u.off_grad = off;
                off += f32;
                u.off_master = off;
                off += f32;
                u.off_m = off;
                off += f32;
                u.off_v = off;
                off += f32;
                if (cfg->push_mode == ODC_PUSH_SLOT) {
                    u.off_slot = off;
                    u.slot_stride = f32;
                    off += f32 * cfg->world;
                }
                if (cfg->push_mode == ODC_PUSH_FIXED) {
                    u.off_acc = off;
                    off += round256((u.block + 2) * 8);
                }
                c->units.push_back(u);
            }
            if (cfg->push_mode == ODC_PUSH_SLOT) {
                c->off_marks = off;
                off += round256(static_cast<std::int64_t>(cfg->n_layers) * cfg->world * 8);
            }
            c->arena_bytes = off;
            c->layout_hash = h;
            DeviceGuard dg(c->dev_id());
            cuda_ok(odc::preload_kernels(), "preload kernels");
            cuda_ok(cudaMalloc(&c->arena, static_cast<std::size_t>(off)), "cudaMalloc arena");
            cuda_ok(cudaMemset(c->arena, 0, static_cast<std::size_t>(off)), "memset arena");
            // the zeroed flags page must be visible before the arena is exported: peers poll it over NVLink
            // (cudaMemset on device memory may return before it completes; a freshly malloc'd arena can hold a
            // previous process's epochs)
            cuda_ok(cudaDeviceSynchronize(), "memset arena sync");
            c->peer.assign(static_cast<std::size_t>(cfg->world), nullptr);
            c->imported.assign(static_cast<std::size_t>(cfg->world), false);
            c->local_peer.assign(static_cast<std::size_t>(cfg->world), false);
            c->peer[static_cast<std::size_t>(cfg->rank)] = c->arena;
            c->imported[static_cast<std::size_t>(cfg->rank)] = true;
            c->touched.assign(c->units.size() * static_cast<std::size_t>(cfg->world), 0);
        } catch (...) {
            odc_ctx_destroy(c);
            throw;
        }
        *out = c;
    });
}

odc_status odc_ctx_destroy(odc_ctx_t c) {
    if (!c) return ODC_OK;
    DeviceGuard dg(c->cfg.device);
    cudaDeviceSynchronize();
    for (int r = 0; r < static_cast<int>(c->peer.size()); ++r)
        if (r != c->cfg.rank && c->peer[static_cast<std::size_t>(r)] &&
            !(r < static_cast<int>(c->local_peer.size()) && c->local_peer[static_cast<std::size_t>(r)]))
            cudaIpcCloseMemHandle(c->peer[static_cast<std::size_t>(r)]);
    if (c->arena) cudaFree(c->arena);
    if (c->d_segs) cudaFree(c->d_segs);
    for (cudaEvent_t e : c->gate_ev)
        if (e) cudaEventDestroy(e);
    if (c->d_seg_start) cudaFree(c->d_seg_start);
    delete c;
    return ODC_OK;
}

odc_status odc_ctx_export(odc_ctx_t ch, void* blob, std::size_t cap, std::size_t* len) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        if (len) *len = sizeof(Blob);
        if (!blob || cap < sizeof(Blob)) throw ParamError("export buffer too small");
        DeviceGuard dg(c->dev_id());
        Blob b{};
        b.magic = kBlobMagic;
        b.rank = c->rank();
        b.world = c->world();
        b.arena_bytes = c->arena_bytes;
        b.layout_hash = c->layout_hash;
        cuda_ok(cudaIpcGetMemHandle(&b.handle, c->arena), "cudaIpcGetMemHandle");
        std::memcpy(blob, &b, sizeof b);
    });
}

odc_status odc_ctx_import(odc_ctx_t ch, int peer, const void* blob, std::size_t len) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        if (peer < 0 || peer >= c->world()) throw ParamError("peer out of range");
        if (peer == c->rank()) return;  // own arena is already mapped
        if (!blob || len < sizeof(Blob)) throw ParamError("bad IPC blob");
        Blob b;
        std::memcpy(&b, blob, sizeof b);
        if (b.magic != kBlobMagic || b.rank != peer || b.world != c->world())
            throw ParamError("IPC blob does not belong to this peer/world");
        if (b.layout_hash != c->layout_hash || b.arena_bytes != c->arena_bytes)
            throw ParamError("peer arena layout differs (different layer sizes or push mode)");
        DeviceGuard dg(c->dev_id());
        void* p = nullptr;
        cuda_ok(cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        c->peer[static_cast<std::size_t>(peer)] = static_cast<char*>(p);
        c->imported[static_cast<std::size_t>(peer)] = true;
    });
}

odc_status odc_ctx_import_ctx(odc_ctx_t ch, int peer, odc_ctx_t peer_ctx) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        odc_ctx* p = C(peer_ctx);
        if (peer < 0 || peer >= c->world()) throw ParamError("peer out of range");
        if (peer == c->rank()) return;
        if (p->rank() != peer || p->world() != c->world()) throw ParamError("context does not belong to this peer/world");
        if (p->layout_hash != c->layout_hash || p->arena_bytes != c->arena_bytes)
            throw ParamError("peer arena layout differs (different layer sizes or push mode)");
        DeviceGuard dg(c->dev_id());
        if (p->cfg.device != c->cfg.device) {  // another GPU of this process: direct peer access over NVLink
            int ok = 0;
            cuda_ok(cudaDeviceCanAccessPeer(&ok, c->cfg.device, p->cfg.device), "cudaDeviceCanAccessPeer");
            if (!ok) throw ParamError("no peer access between the two devices");
            const cudaError_t e = cudaDeviceEnablePeerAccess(p->cfg.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else cuda_ok(e, "cudaDeviceEnablePeerAccess");
        }
        c->peer[static_cast<std::size_t>(peer)] = p->arena;
        c->imported[static_cast<std::size_t>(peer)] = true;
        c->local_peer[static_cast<std::size_t>(peer)] = true;
    });
}

odc_status odc_ctx_ready(odc_ctx_t ch) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        for (int r = 0; r < c->world(); ++r)
            if (!c->imported[static_cast<std::size_t>(r)]) throw StateError("peer " + std::to_string(r) + " not imported");
        DeviceGuard dg(c->dev_id());
        // AdamW segment table over this rank's owned shards
        std::vector<odc::AdamSeg> segs;
        std::vector<std::int64_t> start{0};
        for (const Unit& u : c->units) {
            const int r = c->rank();
            odc::AdamSeg s{};
            s.master = c->f32_of(r, u.off_master, u);
            s.m = c->f32_of(r, u.off_m, u);
            s.v = c->f32_of(r, u.off_v, u);
            s.grad = c->f32_of(r, u.off_grad, u);
            s.param = c->param_of(r, u);
            s.n = u.len(r);
            segs.push_back(s);
            const std::int64_t h = u.begin(r) % 4;
            start.push_back(start.back() + (s.n > 0 ? (h + s.n + 3) / 4 : 0));
        }
        cuda_ok(cudaMalloc(&c->d_segs, segs.size() * sizeof(odc::AdamSeg)), "malloc segs");
        cuda_ok(cudaMalloc(&c->d_seg_start, start.size() * sizeof(std::int64_t)), "malloc seg_start");
        cuda_ok(cudaMemcpy(c->d_segs, segs.data(), segs.size() * sizeof(odc::AdamSeg), cudaMemcpyHostToDevice), "H2D segs");
        cuda_ok(cudaMemcpy(c->d_seg_start, start.data(), start.size() * 8, cudaMemcpyHostToDevice), "H2D start");
        c->adam_units = start.back();
        c->ready = true;
    });
}

odc_status odc_ctx_arena_bytes(odc_ctx_t ch, std::int64_t* bytes) {
    return odc::guard([&] { *bytes = C(ch)->arena_bytes; });
}

int64_t odc_ctx_epoch(odc_ctx_t ch) { return ch ? static_cast<int64_t>(ch->mb_epoch) : -1; }

odc_status odc_set_params(odc_ctx_t ch, int layer, const float* src_full, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        const Unit& u = c->unit(layer);
        DeviceGuard dg(c->dev_id());
        const int r = c->rank();
        c->drain_pending(S(stream));
        cuda_ok(odc::launch_init_shard(c->f32_of(r, u.off_master, u), c->param_of(r, u), src_full + u.begin(r), u.len(r),
                                       S(stream)),
                "set_params");
    });
}

odc_status odc_fetch(odc_ctx_t ch, int layer, void* dst_full, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        const Unit& u = c->unit(layer);
        DeviceGuard dg(c->dev_id());
        c->drain_pending(S(stream));
        odc::SegTable t{};
        t.n = c->world();
        for (int i = 0; i < c->world(); ++i) {
            const int r = c->owner_at(i);
            t.src[i] = reinterpret_cast<const char*>(c->param_of(r, u));
            t.dst[i] = static_cast<char*>(dst_full) + u.begin(r) * 2;
            t.bytes[i] = u.len(r) * 2;
            t.gate[i] = nullptr;
        }
        c->gate(true, S(stream));
        t.err = c->err();
        t.timeout_ns = c->timeout_ns;
        launch_fetch(c, t, S(stream));
    });
}

odc_status odc_fetch_master(odc_ctx_t ch, int layer, float* dst_full, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        const Unit& u = c->unit(layer);
        DeviceGuard dg(c->dev_id());
        odc::SegTable t{};
        t.n = c->world();
        for (int i = 0; i < c->world(); ++i) {
            const int r = c->owner_at(i);
            t.src[i] = reinterpret_cast<const char*>(c->f32_of(r, u.off_master, u));
            t.dst[i] = reinterpret_cast<char*>(dst_full + u.begin(r));
            t.bytes[i] = u.len(r) * 4;
            t.gate[i] = nullptr;
        }
        c->gate(true, S(stream));
        t.err = c->err();
        t.timeout_ns = c->timeout_ns;
        launch_fetch(c, t, S(stream));
    });
}

odc_status odc_push(odc_ctx_t ch, int layer, const void* grad_full, int grad_dtype, float weight, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        const Unit& u = c->unit(layer);
        if (grad_dtype != ODC_F32 && grad_dtype != ODC_BF16) throw ParamError("grad dtype must be ODC_F32 or ODC_BF16");
        const bool bf16 = grad_dtype == ODC_BF16;
        DeviceGuard dg(c->dev_id());
        c->drain_pending(S(stream));
        if (c->slot_mode()) {
            // w*g for every owner goes straight into this client's slot AT THE OWNER over NVLink:
            // stored by the unit's first push of the minibatch (after the owner's reduce of the
            // previous minibatch released the slot), added (single writer, stream order) by later ones
            odc::BulkTable t{};
            t.n = c->world();
            const int me = c->rank();
            for (int i = 0; i < c->world(); ++i) {
                const int r = c->owner_at(i);
                t.src[i] = static_cast<const char*>(grad_full) + u.begin(r) * (bf16 ? 2 : 4);
                t.dst[i] = c->slot_of(r, u, me);
                t.elems[i] = u.len(r);
                t.gate[i] = nullptr;
                const bool first = !c->touched_at(layer, r);
                t.assign[i] = first;
                t.mark[i] = first ? c->mark_of(r, layer, me) : nullptr;
                c->touched_at(layer, r) = 1;
            }
            t.mark_value = c->mb_epoch + 1;
            c->gate(false, S(stream));
            t.err = c->err();
            t.timeout_ns = c->timeout_ns;
            cuda_ok(odc::launch_push_bulk(t, false, weight, 1.f, bf16, c->cfg.push_ctas, S(stream)), "push (slot)");
            return;
        }
        if (c->fixed_mode()) {
            odc::BulkTable t{};
            t.n = c->world();
            for (int i = 0; i < c->world(); ++i) {
                const int r = c->owner_at(i);
                t.src[i] = static_cast<const char*>(grad_full) + u.begin(r) * (bf16 ? 2 : 4);
                t.dst[i] = c->acc_of(r, u);
                t.elems[i] = u.len(r);
                t.gate[i] = nullptr;
            }
            c->gate(false, S(stream));  // the owners drained (converted + zeroed) the previous minibatch's sums
            t.err = c->err();
            t.timeout_ns = c->timeout_ns;
            cuda_ok(odc::launch_push_bulk(t, true, weight, c->fixed_scale(), bf16, c->cfg.push_ctas, S(stream)),
                    "push (fixed)");
            return;
        }
        // RED engine: TMA bulk reductions (cp.reduce.async.bulk .add.f32, 8 KB per op) beat
        // per-thread red.global.add.v4.f32 by 7-8% over NVLink from 16 MB shards up (N=2: 552 vs
        // 514 GB/s, N=4: 567 vs 527 at 256 MB, profiles/r01/p2p_push_engines.md); red.v4 stays
        // for small shards (< 1 M elements per owner), where its lower launch cost wins.
        // ODC_RED_ENGINE=red|bulk pins one engine (ablation).
        static const int red_engine = [] {
            const char* v = std::getenv("ODC_RED_ENGINE");
            if (!v) return 0;
            return std::string(v) == "bulk" ? 2 : std::string(v) == "red" ? 1 : 0;
        }();
        if (red_engine == 2 || (red_engine == 0 && u.block >= (1 << 20))) {
            odc::BulkTable t{};
            t.n = c->world();
            for (int i = 0; i < c->world(); ++i) {
                const int r = c->owner_at(i);
                t.src[i] = static_cast<const char*>(grad_full) + u.begin(r) * (bf16 ? 2 : 4);
                t.dst[i] = c->f32_of(r, u.off_grad, u);
                t.elems[i] = u.len(r);
                t.gate[i] = nullptr;
            }
            c->gate(false, S(stream));  // the owners consumed (zeroed) last minibatch's shard
            t.err = c->err();
            t.timeout_ns = c->timeout_ns;
            cuda_ok(odc::launch_push_bulk(t, false, weight, 1.f, bf16, c->cfg.push_ctas, S(stream)), "push (bulk)");
            return;
        }
        odc::RedTable t{};
        t.n = c->world();
        for (int i = 0; i < c->world(); ++i) {
            const int r = c->owner_at(i);
            t.src[i] = static_cast<const char*>(grad_full) + u.begin(r) * (bf16 ? 2 : 4);
            t.dst[i] = c->f32_of(r, u.off_grad, u);
            t.elems[i] = u.len(r);
            t.gate[i] = nullptr;
        }
        c->gate(false, S(stream));
        t.err = c->err();
        t.timeout_ns = c->timeout_ns;
        cuda_ok(odc::launch_push_red(t, weight, bf16, c->cfg.push_ctas, S(stream)), "push");
    });
}

odc_status odc_push_slice(odc_ctx_t ch, int layer, int target, std::int64_t offset, const float* payload,
                          std::int64_t n, float weight, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        const Unit& u = c->unit(layer);
        if (target < 0 || target >= c->world()) throw ParamError("target rank out of range");
        if (n < 0) throw ParamError("negative payload length");
        if (n > u.block)
            throw ProtocolError("payload of " + std::to_string(n) + " elements exceeds the per-client buffer slot of " +
                                std::to_string(u.block));
        if (offset < 0 || offset + n > u.len(target)) throw ProtocolError("payload does not fit the target shard");
        if (n == 0) return;
        DeviceGuard dg(c->dev_id());
        c->drain_pending(S(stream));
        if (c->slot_mode()) {
            const int me = c->rank();
            float* slot = c->slot_of(target, u, me);
            const bool first = !c->touched_at(layer, target);
            c->gate(false, S(stream));
            if (first) {  // the slot still holds an older minibatch: zero it (the owner released it)
                float* p = slot;
                std::int64_t cnt = u.len(target);
                cuda_ok(odc::launch_gated_zero(&p, &cnt, 1, nullptr, 0, 0, c->err(), c->timeout_ns, S(stream)),
                        "slot zero");
                c->touched_at(layer, target) = 1;
            }
            odc::BulkTable t{};
            t.n = 1;
            t.src[0] = payload;
            t.dst[0] = slot + offset;
            t.elems[0] = n;
            t.mark[0] = first ? c->mark_of(target, layer, me) : nullptr;
            t.mark_value = c->mb_epoch + 1;
            t.err = c->err();
            t.timeout_ns = c->timeout_ns;
            cuda_ok(odc::launch_push_bulk(t, false, weight, 1.f, false, 8, S(stream)), "push_slice (slot)");
            return;
        }
        if (c->fixed_mode()) {
            odc::BulkTable t{};
            t.n = 1;
            t.src[0] = payload;
            t.dst[0] = c->acc_of(target, u) + offset;
            t.elems[0] = n;
            c->gate(false, S(stream));
            t.err = c->err();
            t.timeout_ns = c->timeout_ns;
            cuda_ok(odc::launch_push_bulk(t, true, weight, c->fixed_scale(), false, 8, S(stream)), "push_slice (fixed)");
            return;
        }
        odc::RedTable t{};
        t.n = 1;
        t.src[0] = payload;
        t.dst[0] = c->f32_of(target, u.off_grad, u) + offset;
        t.elems[0] = n;
        c->gate(false, S(stream));
        t.err = c->err();
        t.timeout_ns = c->timeout_ns;
        cuda_ok(odc::launch_push_red(t, weight, false, 8, S(stream)), "push_slice");
    });
}

odc_status odc_minibatch_end(odc_ctx_t ch, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        DeviceGuard dg(c->dev_id());
        c->drain_pending(S(stream));
        odc::BarrierArgs a{};
        a.world = c->world();
        a.rank = c->rank();
        for (int r = 0; r < c->world(); ++r) a.peer_done[r] = c->done_of(r);
        a.my_done = c->done_of(c->rank());
        a.epoch = c->mb_epoch + 1;
        a.err = c->err();
        a.timeout_ns = c->timeout_ns;
        cuda_ok(odc::launch_barrier(a, S(stream)), "barrier");
        c->mb_epoch += 1;
        if (c->slot_mode()) {  // every client's slot writes landed before its done flag: rank-order reduce
            const int me = c->rank();
            odc::SlotReduce r{};
            r.nsrc = c->world();
            r.epoch = c->mb_epoch;
            for (std::size_t l = 0; l < c->units.size(); ++l) {
                const Unit& u = c->units[l];
                r.dst[r.n] = c->f32_of(me, u.off_grad, u);
                r.slot0[r.n] = c->slot_of(me, u, 0);
                r.slot_stride[r.n] = u.slot_stride / 4;
                r.elems[r.n] = u.len(me);
                r.marks[r.n] = c->mark_of(me, static_cast<int>(l), 0);
                if (++r.n == odc::kMaxReduceUnits) {
                    cuda_ok(odc::launch_slot_reduce(r, S(stream)), "slot reduce");
                    r.n = 0;
                }
            }
            cuda_ok(odc::launch_slot_reduce(r, S(stream)), "slot reduce");
            std::fill(c->touched.begin(), c->touched.end(), 0);
            // the slots of this minibatch are consumed: clients may store into them again
            cuda_ok(odc::launch_publish(c->drain_of(me), c->mb_epoch, S(stream)), "publish drain epoch");
        }
        if (c->red_mode()) c->grads_pending = true;
        if (c->fixed_mode()) {  // every client's reductions landed before its done flag: convert + zero
            const int me = c->rank();
            const float inv = std::ldexp(1.0f, -c->cfg.fixed_frac_bits);
            odc::FixFinal f{};
            for (const Unit& u : c->units) {
                if (u.len(me) <= 0) continue;
                f.grad[f.n] = c->f32_of(me, u.off_grad, u);
                f.acc[f.n] = c->acc_of(me, u);
                f.elems[f.n] = u.len(me);
                if (++f.n == odc::kMaxFinal) {
                    cuda_ok(odc::launch_fixed_finalize(f, inv, S(stream)), "fixed finalize");
                    f.n = 0;
                }
            }
            cuda_ok(odc::launch_fixed_finalize(f, inv, S(stream)), "fixed finalize");
            cuda_ok(odc::launch_publish(c->drain_of(me), c->mb_epoch, S(stream)), "publish drain epoch");
        }
    });
}

odc_status odc_read_grad_shard(odc_ctx_t ch, int layer, float* dst, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        const Unit& u = c->unit(layer);
        DeviceGuard dg(c->dev_id());
        const int r = c->rank();
        if (u.len(r) > 0)
            cuda_ok(cudaMemcpyAsync(dst, c->f32_of(r, u.off_grad, u), static_cast<std::size_t>(u.len(r)) * 4,
                                    cudaMemcpyDeviceToDevice, S(stream)),
                    "read grad");
    });
}

odc_status odc_read_master_shard(odc_ctx_t ch, int layer, float* dst, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        const Unit& u = c->unit(layer);
        DeviceGuard dg(c->dev_id());
        const int r = c->rank();
        if (u.len(r) > 0)
            cuda_ok(cudaMemcpyAsync(dst, c->f32_of(r, u.off_master, u), static_cast<std::size_t>(u.len(r)) * 4,
                                    cudaMemcpyDeviceToDevice, S(stream)),
                    "read master");
    });
}

odc_status odc_adam_step(odc_ctx_t ch, const odc_adam_cfg* cfg, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        c->need_ready();
        if (!cfg || cfg->step < 1) throw ParamError("adam step must be >= 1");
        DeviceGuard dg(c->dev_id());
        odc::AdamArgs a{};
        a.segs = c->d_segs;
        a.nseg = static_cast<int>(c->units.size());
        a.seg_start = c->d_seg_start;
        a.lr = cfg->lr;
        a.beta1 = cfg->beta1;
        a.beta2 = cfg->beta2;
        a.eps = cfg->eps;
        a.wd = cfg->weight_decay;
        const double bc1 = 1.0 - std::pow(static_cast<double>(cfg->beta1), cfg->step);
        const double bc2 = 1.0 - std::pow(static_cast<double>(cfg->beta2), cfg->step);
        a.step_size = static_cast<float>(cfg->lr / bc1);
        a.bc2_sqrt_inv = static_cast<float>(1.0 / std::sqrt(bc2));
        cuda_ok(odc::launch_adam(a, c->adam_units, 0, S(stream)), "adam");  // also zeroes the grad shards
        c->adams += 1;
        // new parameter epoch (fetch gate) and, RED, the consumed grad shards (push gate)
        cuda_ok(odc::launch_publish(c->epoch_of(c->rank()), c->adams, S(stream), c->drain_of(c->rank()), c->mb_epoch),
                "publish epoch");
        c->grads_pending = false;
    });
}

odc_status odc_ctx_check(odc_ctx_t ch, void* stream) {
    unsigned long long e = 0;
    odc_status st = odc::guard([&] {
        odc_ctx* c = C(ch);
        DeviceGuard dg(c->dev_id());
        cuda_ok(cudaStreamSynchronize(S(stream)), "sync");
        cuda_ok(cudaMemcpy(&e, c->err(), 8, cudaMemcpyDeviceToHost), "read err");
    });
    if (st != ODC_OK) return st;
    if (e & odc::kErrTimeout) {
        odc::set_last_error("device barrier watchdog fired: a peer never reached the minibatch barrier "
                            "or never published its parameter epoch");
        return ODC_ERR_TIMEOUT;
    }
    if (e & odc::kErrFixedRange) {
        odc::set_last_error("FIXED push out of range: a contribution |w*g| * 2^frac_bits reached 2^55 "
                            "(int64 accumulator headroom) or was NaN/Inf; lower fixed_frac_bits");
        return ODC_ERR_RANGE;
    }
    return ODC_OK;
}

odc_status odc_ctx_flags(odc_ctx_t ch, uint64_t* flags, void* stream) {
    return odc::guard([&] {
        odc_ctx* c = C(ch);
        if (!flags) throw ParamError("null flags");
        DeviceGuard dg(c->dev_id());
        cuda_ok(cudaStreamSynchronize(S(stream)), "sync");
        unsigned long long e = 0;
        cuda_ok(cudaMemcpy(&e, c->err(), 8, cudaMemcpyDeviceToHost), "read err");
        *flags = e;
    });
}

odc_status odc_copy_segments(int nseg, const void* const* srcs, void* const* dsts, const std::int64_t* bytes, int ctas,
                             void* stream) {
    return odc::guard([&] {
        if (nseg < 0 || nseg > odc::kMaxSeg) throw ParamError("1..16 segments per call");
        odc::SegTable t{};
        t.n = nseg;
        for (int i = 0; i < nseg; ++i) {
            t.src[i] = static_cast<const char*>(srcs[i]);
            t.dst[i] = static_cast<char*>(dsts[i]);
            t.bytes[i] = bytes[i];
        }
        cuda_ok(odc::launch_copy_segments(t, ctas, S(stream)), "copy_segments");
    });
}

odc_status odc_l2_flush(void* scratch, std::int64_t bytes, void* stream) {
    return odc::guard([&] { cuda_ok(odc::launch_l2_flush(scratch, bytes, S(stream)), "l2 flush"); });
}

}  // extern "C"
