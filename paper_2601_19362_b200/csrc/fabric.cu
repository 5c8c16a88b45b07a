// fabric.cu — odc_fabric_t: the reference's ShardFabric<T>/ShardState<T>
// (inc/primitives.hpp:35-207) with every shard, staging slot and gradient
// accumulator resident in HBM and every data movement done by the sm_100a
// kernels of odc_kernels.cu. All simulated ranks live on one device; the
// per-rank storage uses the same co-aligned padding as the multi-GPU engine
// (shard r stored at an offset congruent to begin_r mod 16 bytes) so gather
// runs the 16-byte vector path of the fetch kernel.
//
// Protocol (ODC_PUSH_SLOT, default) follows the reference exactly:
//   scatter_accumulate :181-188  for each owner: consume own occupied slot,
//                                then stage the slice into slot(owner, client)
//   push_slice :191-195          consume first, then bounds-check + stage
//   consume :125-136             owner shard[off+i] += w * payload[i]
//   finalize :199-203            consume (s, c) in order, copy out, zero
// so float/double results are bit-identical to the reference, not just close.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"

namespace {

using odcsim::InvariantError;
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

std::size_t dtype_size(odc_dtype d) {
    switch (d) {
        case ODC_I64: return 8;
        case ODC_F64: return 8;
        case ODC_F32: return 4;
        default: throw ParamError("fabric dtype must be ODC_I64, ODC_F64 or ODC_F32");
    }
}

}  // namespace

struct odc_fabric {
    int ranks = 1;
    std::int64_t elems = 0, block = 0;
    odc_dtype dt = ODC_I64;
    std::size_t es = 8;
    int device = 0;
    odc_push_mode mode = ODC_PUSH_SLOT;
    cudaStream_t stream = nullptr;

    // Single-process multi-GPU mode (odc_fabric_create_multi): simulated rank r's
    // shards, gradient accumulator and server-side slots live on rank_dev[r];
    // the host staging / output buffers and every kernel live on `device`, which
    // reaches the other GPUs' memory through peer access over NVLink.
    std::vector<int> rank_dev;

    // one allocation per (shard set, device); rank r's shard at base_of_its_device + k*stride + pad_r
    struct ShardSet {
        std::vector<char*> bases;  // allocations to free
        std::vector<char*> ptr;
    };
    std::int64_t stride_bytes = 0;
    std::map<std::string, ShardSet> params;
    ShardSet grads;

    std::vector<char*> slots;  // per server s: [client] x block elements, on rank_dev[s]
    std::vector<unsigned char> occ;
    std::vector<std::int64_t> slot_off, slot_len;
    std::vector<std::uint64_t> slot_w;  // weight bits
    std::vector<std::int64_t> staged, peak;

    char* stage = nullptr;  // full-length host->device staging
    char* out = nullptr;    // full-length gather/finalize output

    std::int64_t begin(int r) const { return std::min<std::int64_t>(elems, static_cast<std::int64_t>(r) * block); }
    std::int64_t len(int r) const {
        return std::min<std::int64_t>(elems, static_cast<std::int64_t>(r + 1) * block) - begin(r);
    }
    char* slot_ptr(int s, int c) const {
        return slots[static_cast<std::size_t>(s)] + static_cast<std::int64_t>(c) * block * static_cast<std::int64_t>(es);
    }
    std::size_t sidx(int s, int c) const { return static_cast<std::size_t>(s) * ranks + c; }

    ShardSet alloc_set() {
        ShardSet s;
        s.ptr.assign(static_cast<std::size_t>(ranks), nullptr);
        std::vector<int> devs(rank_dev);
        std::sort(devs.begin(), devs.end());
        devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
        for (int d : devs) {  // the ranks of device d share one allocation there
            std::vector<int> rs;
            for (int r = 0; r < ranks; ++r)
                if (rank_dev[static_cast<std::size_t>(r)] == d) rs.push_back(r);
            char* base = nullptr;
            const std::int64_t total = stride_bytes * static_cast<std::int64_t>(rs.size());
            cuda_ok(cudaSetDevice(d), "cudaSetDevice");
            cuda_ok(cudaMalloc(&base, static_cast<std::size_t>(total)), "cudaMalloc shards");
            cuda_ok(cudaMemset(base, 0, static_cast<std::size_t>(total)), "memset shards");
            s.bases.push_back(base);
            for (std::size_t k = 0; k < rs.size(); ++k) {
                const int r = rs[k];
                const std::int64_t pad = (begin(r) * static_cast<std::int64_t>(es)) % 16;
                s.ptr[static_cast<std::size_t>(r)] = base + static_cast<std::int64_t>(k) * stride_bytes + pad;
            }
        }
        DeviceGuard dg(dev_id());
        return s;
    }
    // zero every rank's accumulator (a kernel on `device`: the shards may be on peer GPUs)
    void zero_set(ShardSet& set) {
        for (int r = 0; r < ranks; ++r) {
            float* p = reinterpret_cast<float*>(set.ptr[static_cast<std::size_t>(r)]);
            std::int64_t n = len(r) * static_cast<std::int64_t>(es) / 4;  // es is 4 or 8: whole fp32 words
            if (n > 0)
                cuda_ok(odc::launch_gated_zero(&p, &n, 1, nullptr, 0, 0, nullptr, 0, stream), "zero grads");
        }
    }

    int dev_id() const { return device; }

    // one copy per simulated rank; the copy kernel's table holds kMaxSeg
    // segments, so any rank count is split into tables of at most kMaxSeg
    template <typename Fn>
    void copy_ranks(Fn&& seg, int ctas, const char* what) {
        for (int base = 0; base < ranks; base += odc::kMaxSeg) {
            odc::SegTable t{};
            t.n = std::min(odc::kMaxSeg, ranks - base);
            for (int i = 0; i < t.n; ++i) seg(base + i, t.src[i], t.dst[i], t.bytes[i]);
            cuda_ok(odc::launch_copy_segments(t, ctas, stream), what);
        }
    }

    template <typename T>
    void consume_t(int s, int c) {
        const std::size_t k = sidx(s, c);
        T w;
        std::memcpy(&w, &slot_w[k], sizeof(T));
        cuda_ok(odc::launch_accumulate<T>(reinterpret_cast<T*>(grads.ptr[s]) + slot_off[k],
                                          reinterpret_cast<const T*>(slot_ptr(s, c)), slot_len[k], w, stream),
                "consume");
    }

    bool consume(int s, int c) {
        const std::size_t k = sidx(s, c);
        if (!occ[k]) return false;
        switch (dt) {
            case ODC_I64: consume_t<long long>(s, c); break;
            case ODC_F64: consume_t<double>(s, c); break;
            default: consume_t<float>(s, c); break;
        }
        staged[static_cast<std::size_t>(s)] -= slot_len[k];
        occ[k] = 0;
        return true;
    }

    // try_stage :105-121 with the payload already on the device at `dev_src`
    bool try_stage(int from, int target, std::int64_t offset, const char* dev_src, std::int64_t n,
                   const void* weight) {
        if (n > block)
            throw ProtocolError("payload of " + std::to_string(n) + " elements exceeds the per-client buffer slot of " +
                                std::to_string(block));
        if (offset < 0 || offset + n > len(target)) throw ProtocolError("payload does not fit the target shard");
        const std::size_t k = sidx(target, from);
        if (occ[k]) return false;
        if (n > 0) {
            odc::SegTable t{};
            t.n = 1;
            t.src[0] = dev_src;
            t.dst[0] = slot_ptr(target, from);
            t.bytes[0] = n * static_cast<std::int64_t>(es);
            cuda_ok(odc::launch_copy_segments(t, 4, stream), "stage copy");
        }
        occ[k] = 1;
        slot_off[k] = offset;
        slot_len[k] = n;
        slot_w[k] = 0;
        std::memcpy(&slot_w[k], weight, es);
        auto& st = staged[static_cast<std::size_t>(target)];
        st += n;
        peak[static_cast<std::size_t>(target)] = std::max(peak[static_cast<std::size_t>(target)], st);
        return true;
    }

    void upload(const void* host, std::int64_t n) {
        cuda_ok(cudaMemcpyAsync(stage, host, static_cast<std::size_t>(n) * es, cudaMemcpyHostToDevice, stream),
                "H2D stage");
    }

    template <typename T>
    void red_push(int client, const void* weight) {
        T w;
        std::memcpy(&w, weight, sizeof(T));
        (void)client;
        for (int r = 0; r < ranks; ++r)
            cuda_ok(odc::launch_red_accumulate<T>(reinterpret_cast<T*>(grads.ptr[r]),
                                                  reinterpret_cast<const T*>(stage) + begin(r), len(r), w, stream),
                    "red push");
    }

    void take_grads(void* host_out) {
        copy_ranks(
            [&](int r, const char*& src, char*& dst, std::int64_t& bytes) {
                src = grads.ptr[r];
                dst = out + begin(r) * static_cast<std::int64_t>(es);
                bytes = len(r) * static_cast<std::int64_t>(es);
            },
            8, "collect grads");
        cuda_ok(cudaMemcpyAsync(host_out, out, static_cast<std::size_t>(elems) * es, cudaMemcpyDeviceToHost, stream),
                "D2H grads");
        zero_set(grads);
        cuda_ok(cudaStreamSynchronize(stream), "sync");
    }
};

namespace {
odc_fabric* F(odc_fabric_t f) {
    if (!f) throw ParamError("null fabric");
    return f;
}
void check_rank(const odc_fabric* f, int r, const char* what) {
    if (r < 0 || r >= f->ranks) throw ParamError(std::string(what) + " rank out of range");
}
}  // namespace

extern "C" {

odc_status odc_fabric_create_multi(int ranks, std::int64_t elems, odc_dtype dtype, const int* devices, int ndev,
                                   odc_fabric_t* out) {
    return odc::guard([&] {
        if (ranks < 1 || elems < 1) throw ParamError("need ranks >= 1 and elems >= 1");
        if (ranks > 4096) throw ParamError("too many ranks");
        if (!devices || ndev < 1) throw ParamError("need at least one device");
        auto* f = new odc_fabric();
        try {
            f->ranks = ranks;
            f->elems = elems;
            f->block = (elems + ranks - 1) / ranks;
            f->dt = dtype;
            f->es = dtype_size(dtype);
            f->device = devices[0];
            for (int r = 0; r < ranks; ++r) f->rank_dev.push_back(devices[r % ndev]);
            DeviceGuard dg(f->dev_id());
            for (int i = 0; i < ndev; ++i) {  // the primary device's kernels reach every shard
                if (devices[i] == f->device) continue;
                int ok = 0;
                cuda_ok(cudaDeviceCanAccessPeer(&ok, f->device, devices[i]), "cudaDeviceCanAccessPeer");
                if (!ok) throw ParamError("no peer access from the primary device to device " + std::to_string(devices[i]));
                const cudaError_t e = cudaDeviceEnablePeerAccess(devices[i], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else cuda_ok(e, "cudaDeviceEnablePeerAccess");
            }
            cuda_ok(cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking), "stream");
            f->stride_bytes = ((f->block * static_cast<std::int64_t>(f->es) + 16 + 255) / 256) * 256;
            f->grads = f->alloc_set();
            const std::int64_t slot_bytes = static_cast<std::int64_t>(ranks) * f->block * f->es;
            for (int sv = 0; sv < ranks; ++sv) {  // server sv's slots live with its shard
                char* p = nullptr;
                cuda_ok(cudaSetDevice(f->rank_dev[static_cast<std::size_t>(sv)]), "cudaSetDevice");
                cuda_ok(cudaMalloc(&p, static_cast<std::size_t>(std::max<std::int64_t>(slot_bytes, 16))), "slots");
                f->slots.push_back(p);
            }
            cuda_ok(cudaSetDevice(f->dev_id()), "cudaSetDevice");  // the guard above restores the caller's
            cuda_ok(cudaMalloc(&f->stage, static_cast<std::size_t>(elems) * f->es + 16), "stage");
            cuda_ok(cudaMalloc(&f->out, static_cast<std::size_t>(elems) * f->es + 16), "out");
            const std::size_t nn = static_cast<std::size_t>(ranks) * ranks;
            f->occ.assign(nn, 0);
            f->slot_off.assign(nn, 0);
            f->slot_len.assign(nn, 0);
            f->slot_w.assign(nn, 0);
            f->staged.assign(static_cast<std::size_t>(ranks), 0);
            f->peak.assign(static_cast<std::size_t>(ranks), 0);
            cuda_ok(cudaStreamSynchronize(f->stream), "sync");
        } catch (...) {
            odc_fabric_destroy(f);
            throw;
        }
        *out = f;
    });
}

odc_status odc_fabric_create(int ranks, std::int64_t elems, odc_dtype dtype, int device, odc_fabric_t* out) {
    return odc_fabric_create_multi(ranks, elems, dtype, &device, 1, out);
}

odc_status odc_fabric_destroy(odc_fabric_t f) {
    if (!f) return ODC_OK;
    DeviceGuard dg(f->device);
    if (f->stream) cudaStreamSynchronize(f->stream);
    for (auto& kv : f->params)
        for (char* b : kv.second.bases) cudaFree(b);
    for (char* b : f->grads.bases) cudaFree(b);
    for (char* b : f->slots) cudaFree(b);
    cudaFree(f->stage);
    cudaFree(f->out);
    if (f->stream) cudaStreamDestroy(f->stream);
    delete f;
    return ODC_OK;
}

odc_status odc_fabric_set_push_mode(odc_fabric_t f, odc_push_mode mode) {
    return odc::guard([&] {
        if (mode != ODC_PUSH_SLOT && mode != ODC_PUSH_RED) throw ParamError("bad push mode");
        F(f)->mode = mode;
    });
}

odc_status odc_fabric_set_params(odc_fabric_t fh, const char* id, const void* host_full, std::int64_t n) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        if (n != f->elems) throw ParamError("parameter vector length mismatch");
        DeviceGuard dg(f->dev_id());
        auto it = f->params.find(id);
        if (it == f->params.end()) it = f->params.emplace(id, f->alloc_set()).first;
        f->upload(host_full, n);
        const auto& dst = it->second.ptr;  // owners take their slices of the full vector
        f->copy_ranks(
            [&](int r, const char*& s, char*& d, std::int64_t& bytes) {
                s = f->stage + f->begin(r) * static_cast<std::int64_t>(f->es);
                d = dst[static_cast<std::size_t>(r)];
                bytes = f->len(r) * static_cast<std::int64_t>(f->es);
            },
            8, "set_params");
        cuda_ok(cudaStreamSynchronize(f->stream), "sync");
    });
}

odc_status odc_fabric_gather(odc_fabric_t fh, int client, const char* id, void* host_out) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        (void)client;  // read-only fetch: the client rank does not matter (:70)
        auto it = f->params.find(id);
        if (it == f->params.end()) throw StateError(std::string("gather of uninitialized params '") + id + "'");
        DeviceGuard dg(f->dev_id());
        const auto& src = it->second.ptr;
        f->copy_ranks(
            [&](int r, const char*& s, char*& d, std::int64_t& bytes) {
                s = src[static_cast<std::size_t>(r)];
                d = f->out + f->begin(r) * static_cast<std::int64_t>(f->es);
                bytes = f->len(r) * static_cast<std::int64_t>(f->es);
            },
            16, "gather");
        cuda_ok(cudaMemcpyAsync(host_out, f->out, static_cast<std::size_t>(f->elems) * f->es, cudaMemcpyDeviceToHost,
                                f->stream),
                "D2H gather");
        cuda_ok(cudaStreamSynchronize(f->stream), "sync");
    });
}

odc_status odc_fabric_scatter_accumulate(odc_fabric_t fh, int client, const void* host_grad, std::int64_t n,
                                         const void* weight) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        check_rank(f, client, "client");
        if (n != f->elems) throw ParamError("gradient vector length mismatch");
        DeviceGuard dg(f->dev_id());
        f->upload(host_grad, n);
        if (f->mode == ODC_PUSH_RED) {
            for (int r = 0; r < f->ranks; ++r)  // keep immediate-mode semantics for any staged slot
                while (f->occ[f->sidx(r, client)]) f->consume(r, client);
            switch (f->dt) {
                case ODC_I64: f->red_push<long long>(client, weight); break;
                case ODC_F64: f->red_push<double>(client, weight); break;
                default: f->red_push<float>(client, weight); break;
            }
        } else {
            for (int r = 0; r < f->ranks; ++r) {
                while (f->occ[f->sidx(r, client)]) f->consume(r, client);
                if (!f->try_stage(client, r, 0, f->stage + f->begin(r) * static_cast<std::int64_t>(f->es), f->len(r),
                                  weight))
                    throw InvariantError("stage into a free slot failed");
            }
        }
        cuda_ok(cudaStreamSynchronize(f->stream), "sync");
    });
}

odc_status odc_fabric_push_slice(odc_fabric_t fh, int client, int target, std::int64_t offset, const void* payload,
                                 std::int64_t n, const void* weight) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        check_rank(f, client, "client");
        check_rank(f, target, "target");
        if (n < 0) throw ParamError("negative payload length");
        DeviceGuard dg(f->dev_id());
        while (f->occ[f->sidx(target, client)]) f->consume(target, client);
        if (n > f->block)
            throw ProtocolError("payload of " + std::to_string(n) + " elements exceeds the per-client buffer slot of " +
                                std::to_string(f->block));
        if (offset < 0 || offset + n > f->len(target)) throw ProtocolError("payload does not fit the target shard");
        if (n > 0) f->upload(payload, n);
        if (f->mode == ODC_PUSH_RED) {
            switch (f->dt) {
                case ODC_I64: {
                    long long w;
                    std::memcpy(&w, weight, 8);
                    cuda_ok(odc::launch_red_accumulate<long long>(reinterpret_cast<long long*>(f->grads.ptr[target]) + offset,
                                                                  reinterpret_cast<const long long*>(f->stage), n, w, f->stream),
                            "red slice");
                    break;
                }
                case ODC_F64: {
                    double w;
                    std::memcpy(&w, weight, 8);
                    cuda_ok(odc::launch_red_accumulate<double>(reinterpret_cast<double*>(f->grads.ptr[target]) + offset,
                                                               reinterpret_cast<const double*>(f->stage), n, w, f->stream),
                            "red slice");
                    break;
                }
                default: {
                    float w;
                    std::memcpy(&w, weight, 4);
                    cuda_ok(odc::launch_red_accumulate<float>(reinterpret_cast<float*>(f->grads.ptr[target]) + offset,
                                                              reinterpret_cast<const float*>(f->stage), n, w, f->stream),
                            "red slice");
                }
            }
        } else {
            f->try_stage(client, target, offset, f->stage, n, weight);
        }
        cuda_ok(cudaStreamSynchronize(f->stream), "sync");
    });
}

odc_status odc_fabric_finalize(odc_fabric_t fh, void* host_out) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        DeviceGuard dg(f->dev_id());
        for (int s = 0; s < f->ranks; ++s)
            for (int c = 0; c < f->ranks; ++c) f->consume(s, c);
        f->take_grads(host_out);
    });
}

odc_status odc_fabric_split_stage(odc_fabric_t fh, int from, int target, std::int64_t offset, const void* payload,
                                  std::int64_t n, const void* weight, int* staged) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        check_rank(f, from, "client");
        check_rank(f, target, "target");
        if (n < 0) throw ParamError("negative payload length");
        DeviceGuard dg(f->dev_id());
        // bounds first (the reference checks before looking at the slot)
        if (n > f->block)
            throw ProtocolError("payload of " + std::to_string(n) + " elements exceeds the per-client buffer slot of " +
                                std::to_string(f->block));
        if (offset < 0 || offset + n > f->len(target)) throw ProtocolError("payload does not fit the target shard");
        if (f->occ[f->sidx(target, from)]) {
            *staged = 0;
            return;
        }
        if (n > 0) f->upload(payload, n);
        *staged = f->try_stage(from, target, offset, f->stage, n, weight) ? 1 : 0;
        cuda_ok(cudaStreamSynchronize(f->stream), "sync");
    });
}

odc_status odc_fabric_slot_free(odc_fabric_t fh, int server, int client, int* is_free) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        check_rank(f, server, "server");
        check_rank(f, client, "client");
        *is_free = f->occ[f->sidx(server, client)] ? 0 : 1;
    });
}

odc_status odc_fabric_consume(odc_fabric_t fh, int server, int client, int* did) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        check_rank(f, server, "server");
        check_rank(f, client, "client");
        DeviceGuard dg(f->dev_id());
        *did = f->consume(server, client) ? 1 : 0;
        cuda_ok(cudaStreamSynchronize(f->stream), "sync");
    });
}

odc_status odc_fabric_any_staged(odc_fabric_t fh, int server, int* any) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        check_rank(f, server, "server");
        int a = 0;
        for (int c = 0; c < f->ranks; ++c) a |= f->occ[f->sidx(server, c)];
        *any = a;
    });
}

odc_status odc_fabric_take_grads(odc_fabric_t fh, void* host_out) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        DeviceGuard dg(f->dev_id());
        f->take_grads(host_out);
    });
}

odc_status odc_fabric_max_staged(odc_fabric_t fh, int server, std::int64_t* pk) {
    return odc::guard([&] {
        odc_fabric* f = F(fh);
        check_rank(f, server, "server");
        *pk = f->peak[static_cast<std::size_t>(server)];
    });
}

}  // extern "C"
