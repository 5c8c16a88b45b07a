// odcsim/primitives.hpp — drop-in façade (B200 build) of the ODC protocol
// objects of /root/reference/proj/include/odcsim/primitives.hpp.
//
// Same class templates, member names and exception behaviour, so code (and
// the reference's own tests) written against the reference compiles
// unchanged — but every shard, staging slot and accumulator lives in HBM and
// every gather / stage / consume is an sm_100a kernel behind the C ABI of
// include/odc/odc.h (odc_fabric_*). T in {std::int64_t, double, float}.
//
//   ShardState<T>    inc/primitives.hpp:35-163   -> odc_fabric_t (owning)
//   ShardFabric<T>   inc/primitives.hpp:167-207  -> odc_fabric_scatter_accumulate / push_slice / finalize
//   run_schedule / run_threaded / verify_primitives (:239-367) are the
//   reference's host protocol drivers; here they drive the GPU-backed state.
//   collective_reduce_reference (:210-220) stays a host-side oracle.
#ifndef ODCSIM_PRIMITIVES_HPP
#define ODCSIM_PRIMITIVES_HPP

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "odc/odc.h"
#include "odcsim/types.hpp"

namespace odcsim {

namespace detail {
template <typename T>
constexpr odc_dtype dtype_of() {
    static_assert(std::is_same_v<T, std::int64_t> || std::is_same_v<T, double> || std::is_same_v<T, float>,
                  "the B200 fabric supports int64_t, double and float");
    if constexpr (std::is_same_v<T, std::int64_t>) return ODC_I64;
    else if constexpr (std::is_same_v<T, double>) return ODC_F64;
    else return ODC_F32;
}
inline int fabric_device() {
    const char* d = std::getenv("ODC_DEVICE");
    return d ? std::atoi(d) : 0;
}
// ODC_DEVICES="0,1,2,3": single-process multi-GPU mode (simulated rank r on the
// r % n-th listed GPU); otherwise every rank on ODC_DEVICE (default 0)
inline std::vector<int> fabric_devices() {
    std::vector<int> out;
    if (const char* d = std::getenv("ODC_DEVICES")) {
        std::string s(d);
        std::size_t pos = 0;
        while (pos < s.size()) {
            const std::size_t comma = s.find(',', pos);
            const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
            if (!tok.empty()) out.push_back(std::atoi(tok.c_str()));
            if (comma == std::string::npos) break;
            pos = comma + 1;
        }
    }
    if (out.empty()) out.push_back(fabric_device());
    return out;
}
}  // namespace detail

// One gradient slice addressed to the owner of that slice.
template <typename T>
struct GradMessage {
    int from_rank = 0;
    int target_rank = 0;
    std::int64_t offset = 0;
    std::vector<T> payload;
    T weight{};
};

template <typename T>
class ShardState {
public:
    ShardState(int ranks, std::int64_t elems) : ranks_(ranks), elems_(elems) {
        if (ranks < 1 || elems < 1) throw ParamError("need ranks >= 1 and elems >= 1");
        block_ = (elems + ranks - 1) / ranks;
        const std::vector<int> devs = detail::fabric_devices();
        detail::check(odc_fabric_create_multi(ranks, elems, detail::dtype_of<T>(), devs.data(),
                                              static_cast<int>(devs.size()), &f_));
    }
    ~ShardState() { odc_fabric_destroy(f_); }
    ShardState(const ShardState&) = delete;
    ShardState& operator=(const ShardState&) = delete;

    int ranks() const { return ranks_; }
    std::int64_t elems() const { return elems_; }
    std::int64_t slot_capacity() const { return block_; }
    std::int64_t shard_begin(int r) const { return std::min<std::int64_t>(elems_, r * block_); }
    std::int64_t shard_len(int r) const { return std::min<std::int64_t>(elems_, (r + 1) * block_) - shard_begin(r); }

    void set_params(const std::string& id, std::vector<T> full) {
        detail::check(odc_fabric_set_params(f_, id.c_str(), full.data(), static_cast<std::int64_t>(full.size())));
    }
    std::vector<T> gather(int client, const std::string& id) const {
        std::vector<T> out(static_cast<std::size_t>(elems_));
        detail::check(odc_fabric_gather(f_, client, id.c_str(), out.data()));
        return out;
    }
    std::vector<GradMessage<T>> split_gradient(int from_rank, const std::vector<T>& grad, T weight) const {
        if (static_cast<std::int64_t>(grad.size()) != elems_) throw ParamError("gradient vector length mismatch");
        std::vector<GradMessage<T>> msgs;
        for (int r = 0; r < ranks_; ++r) {
            auto first = grad.begin() + shard_begin(r);
            msgs.push_back(GradMessage<T>{from_rank, r, 0, std::vector<T>(first, first + shard_len(r)), weight});
        }
        return msgs;
    }
    bool slot_free(int server, int client) const {
        int v = 0;
        detail::check(odc_fabric_slot_free(f_, server, client, &v));
        return v != 0;
    }
    bool try_stage(GradMessage<T> msg) {
        int staged = 0;
        detail::check(odc_fabric_split_stage(f_, msg.from_rank, msg.target_rank, msg.offset, msg.payload.data(),
                                             static_cast<std::int64_t>(msg.payload.size()), &msg.weight, &staged));
        return staged != 0;
    }
    bool consume(int server, int client) {
        int did = 0;
        detail::check(odc_fabric_consume(f_, server, client, &did));
        return did != 0;
    }
    bool any_staged(int server) const {
        int any = 0;
        detail::check(odc_fabric_any_staged(f_, server, &any));
        return any != 0;
    }
    std::vector<std::vector<T>> take_grads() {
        std::vector<T> flat(static_cast<std::size_t>(elems_));
        detail::check(odc_fabric_take_grads(f_, flat.data()));
        return split(flat);
    }
    std::int64_t max_staged_elems(int server) const {
        std::int64_t p = 0;
        detail::check(odc_fabric_max_staged(f_, server, &p));
        return p;
    }

    // B200 extensions used by ShardFabric
    odc_fabric_t handle() const { return f_; }
    std::vector<std::vector<T>> split(const std::vector<T>& flat) const {
        std::vector<std::vector<T>> shards;
        for (int r = 0; r < ranks_; ++r) {
            auto first = flat.begin() + shard_begin(r);
            shards.emplace_back(first, first + shard_len(r));
        }
        return shards;
    }

private:
    int ranks_;
    std::int64_t elems_;
    std::int64_t block_ = 0;
    odc_fabric_t f_ = nullptr;
};

// Immediate-mode fabric (the fully serial schedule), GPU-resident.
template <typename T>
class ShardFabric {
public:
    ShardFabric(int ranks, std::int64_t elems) : state_(ranks, elems) {}

    ShardState<T>& state() { return state_; }

    void set_params(const std::string& id, std::vector<T> full) { state_.set_params(id, std::move(full)); }
    std::vector<T> gather(int client_rank, const std::string& id) const { return state_.gather(client_rank, id); }

    void scatter_accumulate(int client_rank, const std::vector<T>& grad, T weight) {
        detail::check(odc_fabric_scatter_accumulate(state_.handle(), client_rank, grad.data(),
                                                    static_cast<std::int64_t>(grad.size()), &weight));
    }
    void push_slice(int client_rank, int target_rank, std::int64_t offset, std::vector<T> payload, T weight) {
        detail::check(odc_fabric_push_slice(state_.handle(), client_rank, target_rank, offset, payload.data(),
                                            static_cast<std::int64_t>(payload.size()), &weight));
    }
    std::vector<std::vector<T>> finalize_minibatch() {
        std::vector<T> flat(static_cast<std::size_t>(state_.elems()));
        detail::check(odc_fabric_finalize(state_.handle(), flat.data()));
        return state_.split(flat);
    }

private:
    ShardState<T> state_;
};

// Host-side sequential reduce oracle: sum of weight * grad in input order.
template <typename T>
std::vector<T> collective_reduce_reference(const std::vector<std::pair<std::vector<T>, T>>& grads) {
    if (grads.empty()) throw ParamError("collective_reduce_reference needs at least one gradient");
    const std::size_t n = grads.front().first.size();
    std::vector<T> sum(n, T{});
    for (const auto& gw : grads) {
        if (gw.first.size() != n) throw ParamError("gradient length mismatch");
        for (std::size_t i = 0; i < n; ++i) sum[i] += gw.second * gw.first[i];
    }
    return sum;
}

template <typename T>
struct ClientScript {
    std::vector<std::pair<std::vector<T>, T>> pushes;  // (full gradient, weight)
};

template <typename T>
struct ScheduleResult {
    std::vector<std::vector<T>> shards;
    std::int64_t max_staged_elems = 0;
    std::vector<T> concatenated() const {
        std::vector<T> flat;
        for (const auto& s : shards) flat.insert(flat.end(), s.begin(), s.end());
        return flat;
    }
};

// Seeded random interleaving of client stages and owner consumes over the
// GPU-resident state. The enabled-action list is built in the reference's
// order (stages by client, then consumes by (server, client)) and one action
// is drawn with mt19937_64, so a seed replays the same interleaving.
template <typename T>
ScheduleResult<T> run_schedule(int ranks, std::int64_t elems, const std::vector<ClientScript<T>>& clients,
                               std::uint64_t seed) {
    ShardState<T> state(ranks, elems);
    std::vector<std::vector<GradMessage<T>>> queue(clients.size());
    std::vector<std::size_t> head(clients.size(), 0);
    for (std::size_t c = 0; c < clients.size(); ++c)
        for (const auto& gw : clients[c].pushes)
            for (auto& m : state.split_gradient(static_cast<int>(c), gw.first, gw.second)) queue[c].push_back(std::move(m));
    // host mirror of slot occupancy (kept in lock step with the device state)
    std::vector<char> busy(static_cast<std::size_t>(ranks) * ranks, 0);
    auto occ = [&](int s, int c) -> char& { return busy[static_cast<std::size_t>(s) * ranks + c]; };
    std::mt19937_64 rng(seed);
    struct Step {
        bool stage;
        int a, b;
    };
    std::vector<Step> enabled;
    for (;;) {
        enabled.clear();
        for (std::size_t c = 0; c < queue.size(); ++c)
            if (head[c] < queue[c].size() && !occ(queue[c][head[c]].target_rank, static_cast<int>(c)))
                enabled.push_back({true, static_cast<int>(c), 0});
        for (int s = 0; s < ranks; ++s)
            for (int c = 0; c < ranks; ++c)
                if (occ(s, c)) enabled.push_back({false, s, c});
        if (enabled.empty()) break;
        const Step st = enabled[rng() % enabled.size()];
        if (st.stage) {
            GradMessage<T>& m = queue[static_cast<std::size_t>(st.a)][head[static_cast<std::size_t>(st.a)]++];
            const int tgt = m.target_rank;
            if (!state.try_stage(std::move(m))) throw InvariantError("stage of an enabled action failed");
            occ(tgt, st.a) = 1;
        } else {
            state.consume(st.a, st.b);
            occ(st.a, st.b) = 0;
        }
    }
    ScheduleResult<T> res;
    for (int s = 0; s < ranks; ++s) res.max_staged_elems = std::max(res.max_staged_elems, state.max_staged_elems(s));
    res.shards = state.take_grads();
    return res;
}

// One host thread per client and one accumulation daemon per owner over the
// GPU-resident state; a single mutex + condvar serialise state access as in
// the reference. Clients block only on their own slot, daemons never block
// on clients, so every schedule terminates.
template <typename T>
ScheduleResult<T> run_threaded(int ranks, std::int64_t elems, const std::vector<ClientScript<T>>& clients) {
    ShardState<T> state(ranks, elems);
    std::mutex mu;
    std::condition_variable cv;
    bool stop = false;
    std::exception_ptr err;
    auto client = [&](int c) {
        try {
            for (const auto& gw : clients[static_cast<std::size_t>(c)].pushes)
                for (auto& m : state.split_gradient(c, gw.first, gw.second)) {
                    std::unique_lock lk(mu);
                    cv.wait(lk, [&] { return err || state.slot_free(m.target_rank, c); });
                    if (err) return;
                    if (!state.try_stage(std::move(m))) throw InvariantError("stage into a free slot failed");
                    cv.notify_all();
                }
        } catch (...) {
            std::lock_guard lk(mu);
            if (!err) err = std::current_exception();
            cv.notify_all();
        }
    };
    auto daemon = [&](int s) {
        for (;;) {
            std::unique_lock lk(mu);
            cv.wait(lk, [&] { return err || stop || state.any_staged(s); });
            if (err) return;
            bool any = false;
            for (int c = 0; c < ranks; ++c) any = state.consume(s, c) || any;
            if (any) cv.notify_all();
            if (stop && !state.any_staged(s)) return;
        }
    };
    std::vector<std::thread> daemons, workers;
    for (int s = 0; s < ranks; ++s) daemons.emplace_back(daemon, s);
    for (std::size_t c = 0; c < clients.size(); ++c) workers.emplace_back(client, static_cast<int>(c));
    for (auto& t : workers) t.join();
    {
        std::lock_guard lk(mu);
        stop = true;
    }
    cv.notify_all();
    for (auto& t : daemons) t.join();
    if (err) std::rethrow_exception(err);
    ScheduleResult<T> res;
    for (int s = 0; s < ranks; ++s) res.max_staged_elems = std::max(res.max_staged_elems, state.max_staged_elems(s));
    res.shards = state.take_grads();
    return res;
}

struct PrimitivesVerifyReport {
    int passed = 0;
    int failed = 0;
    std::int64_t max_staged_elems = 0;
};

// Randomised equivalence suite (src/primitives.cpp:26-49 draw order): per
// minibatch elems = 8 + rng()%57, 1..8 pushes per client of values in
// [-1000, 1000] with weights in [0, 4]; pass iff the GPU schedule equals the
// sequential oracle and the peak staged volume stays within ceil(M/N)*N.
inline PrimitivesVerifyReport verify_primitives(int clients, int minibatches, std::uint64_t seed) {
    if (clients < 1 || minibatches < 1) throw ParamError("verify-primitives needs clients >= 1 and minibatches >= 1");
    PrimitivesVerifyReport rep;
    std::mt19937_64 rng(seed);
    for (int mb = 0; mb < minibatches; ++mb) {
        const std::int64_t elems = 8 + static_cast<std::int64_t>(rng() % 57);
        std::vector<ClientScript<std::int64_t>> scripts(static_cast<std::size_t>(clients));
        std::vector<std::pair<std::vector<std::int64_t>, std::int64_t>> flat;
        for (auto& sc : scripts) {
            const int pushes = 1 + static_cast<int>(rng() % 8);
            for (int p = 0; p < pushes; ++p) {
                std::vector<std::int64_t> g(static_cast<std::size_t>(elems));
                for (auto& x : g) x = static_cast<std::int64_t>(rng() % 2001) - 1000;
                const auto w = static_cast<std::int64_t>(rng() % 5);
                sc.pushes.emplace_back(g, w);
                flat.emplace_back(std::move(g), w);
            }
        }
        const auto want = collective_reduce_reference(flat);
        const auto got = run_schedule(clients, elems, scripts, rng());
        rep.max_staged_elems = std::max(rep.max_staged_elems, got.max_staged_elems);
        const std::int64_t slot = (elems + clients - 1) / clients;
        if (got.concatenated() == want && got.max_staged_elems <= slot * clients) ++rep.passed;
        else ++rep.failed;
    }
    return rep;
}

}  // namespace odcsim

#endif
