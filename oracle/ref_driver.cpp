// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (oracle side).
//
// A thin extern "C" shim over the UNMODIFIED reference library built from
// /root/reference/proj/src by oracle/Makefile. It lets the Python tests and
// bench.py's cpu_baseline / --impl reference arm call the reference itself:
//   * plan()            src/partition.cpp:490-580   -> solutions_to_json (src/experiment.cpp:215-233)
//   * kk_partition()    src/partition.cpp:84-128
//   * generate_synthetic / scale_lengths  src/workload.cpp:218-230, :263-271
//   * ShardFabric<T>    inc/primitives.hpp:168-207 (scatter_accumulate + finalize scripts)
//   * run_schedule      inc/primitives.hpp:242-294
//   * timing of gather / scatter_accumulate / finalize on host cores
// Nothing in the product (paper_2601_19362_b200/, include/) links this file.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "odcsim/cost_model.hpp"
#include "odcsim/experiment.hpp"
#include "odcsim/partition.hpp"
#include "odcsim/primitives.hpp"
#include "odcsim/runtime.hpp"
#include "odcsim/workload.hpp"

using namespace odcsim;

namespace {

int put_string(const std::string& s, char* out, std::int64_t cap, std::int64_t* out_len) {
    if (out_len) *out_len = static_cast<std::int64_t>(s.size());
    if (!out || cap <= 0) return 0;
    std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
    std::memcpy(out, s.data(), n);
    out[n] = 0;
    return 0;
}

template <typename F>
int guarded(F&& f, char* out, std::int64_t cap, std::int64_t* out_len) {
    try {
        return f();
    } catch (const ParamError& e) {
        put_string(e.what(), out, cap, out_len);
        return 2;
    } catch (const FormatError& e) {
        put_string(e.what(), out, cap, out_len);
        return 2;
    } catch (const InfeasibleError& e) {
        put_string(e.what(), out, cap, out_len);
        return 3;
    } catch (const ProtocolError& e) {
        put_string(e.what(), out, cap, out_len);
        return 5;
    } catch (const StateError& e) {
        put_string(e.what(), out, cap, out_len);
        return 6;
    } catch (const InvariantError& e) {
        put_string(e.what(), out, cap, out_len);
        return 4;
    } catch (const std::exception& e) {
        put_string(e.what(), out, cap, out_len);
        return 9;
    }
}

Workload workload_of(const std::int64_t* lens, std::int64_t n) {
    std::vector<Sample> s;
    s.reserve(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) s.push_back(Sample{i, lens[i]});
    return Workload(std::move(s));
}

template <typename T>
int fabric_script(int ranks, std::int64_t elems, int npush, const int* clients, const T* grads,
                  const T* weights, T* out) {
    ShardFabric<T> fab(ranks, elems);
    for (int p = 0; p < npush; ++p) {
        std::vector<T> g(grads + static_cast<std::int64_t>(p) * elems,
                         grads + static_cast<std::int64_t>(p + 1) * elems);
        fab.scatter_accumulate(clients[p], g, weights[p]);
    }
    auto shards = fab.finalize_minibatch();
    std::int64_t o = 0;
    for (auto& s : shards)
        for (auto v : s) out[o++] = v;
    return 0;
}

}  // namespace

extern "C" {

// strategy: 0 local-sort, 1 lb-micro, 2 lb-mini, 3 verl-native, 4 verl-optimized
int ref_plan_json(int strategy, const std::int64_t* lens, std::int64_t n, int devices, int minibs,
                  std::int64_t budget, double alpha, double beta, int layers, std::uint64_t seed,
                  char* out, std::int64_t cap, std::int64_t* out_len) {
    return guarded(
        [&] {
            static const Strategy kS[] = {Strategy::LocalSort, Strategy::LbMicro, Strategy::LbMini,
                                          Strategy::VerlNative, Strategy::VerlOptimized};
            if (strategy < 0 || strategy > 4) throw ParamError("bad strategy");
            CostModel cm{alpha, beta, layers};
            auto res = plan(kS[strategy], workload_of(lens, n), devices, minibs,
                            MemoryBudget{budget}, cm, seed);
            return put_string(solutions_to_json(res).dump(), out, cap, out_len);
        },
        out, cap, out_len);
}

// Times plan() only (the JSON dump is outside the timed region). Returns seconds.
double ref_plan_seconds(int strategy, const std::int64_t* lens, std::int64_t n, int devices,
                        int minibs, std::int64_t budget, double alpha, double beta, int iters) {
    static const Strategy kS[] = {Strategy::LocalSort, Strategy::LbMicro, Strategy::LbMini,
                                  Strategy::VerlNative, Strategy::VerlOptimized};
    CostModel cm{alpha, beta, 1};
    Workload w = workload_of(lens, n);
    auto t0 = std::chrono::steady_clock::now();
    std::size_t sink = 0;
    for (int i = 0; i < iters; ++i)
        sink += plan(kS[strategy], w, devices, minibs, MemoryBudget{budget}, cm, 0).steps.size();
    auto t1 = std::chrono::steady_clock::now();
    return sink ? std::chrono::duration<double>(t1 - t0).count() : -1.0;
}

int ref_kk_partition_json(const double* costs, int n, int k, int equal_size, int brute, char* out,
                          std::int64_t cap, std::int64_t* out_len) {
    return guarded(
        [&] {
            std::span<const double> c(costs, static_cast<std::size_t>(n));
            PartitionResult r = brute ? brute_force_partition(c, k, equal_size != 0)
                                      : kk_partition(c, k, equal_size != 0);
            nlohmann::json j{{"parts", r.parts}, {"sums", r.sums}, {"spread", r.spread}};
            return put_string(j.dump(), out, cap, out_len);
        },
        out, cap, out_len);
}

// dist: 0 lognormal(p1=mu,p2=sigma) 1 pareto(p1=scale,p2=shape) 2 uniform(p1=lo,p2=hi)
int ref_generate_synthetic(int dist, double p1, double p2, std::int64_t n, std::int64_t cap_len,
                           std::uint64_t seed, double scale, std::int64_t* out) {
    return guarded(
        [&] {
            DistSpec d;
            if (dist == 0) d = LognormalDist{p1, p2};
            else if (dist == 1) d = ParetoDist{p1, p2};
            else d = UniformDist{static_cast<Tokens>(p1), static_cast<Tokens>(p2)};
            Workload w = generate_synthetic(d, n, cap_len, seed);
            if (scale != 1.0) w = scale_lengths(w, scale);
            for (std::int64_t i = 0; i < n; ++i) out[i] = w.samples()[static_cast<std::size_t>(i)].length;
            return 0;
        },
        nullptr, 0, nullptr);
}

int ref_fabric_script_i64(int ranks, std::int64_t elems, int npush, const int* clients,
                          const std::int64_t* grads, const std::int64_t* weights, std::int64_t* out) {
    return guarded([&] { return fabric_script(ranks, elems, npush, clients, grads, weights, out); },
                   nullptr, 0, nullptr);
}
int ref_fabric_script_f64(int ranks, std::int64_t elems, int npush, const int* clients,
                          const double* grads, const double* weights, double* out) {
    return guarded([&] { return fabric_script(ranks, elems, npush, clients, grads, weights, out); },
                   nullptr, 0, nullptr);
}
int ref_fabric_script_f32(int ranks, std::int64_t elems, int npush, const int* clients,
                          const float* grads, const float* weights, float* out) {
    return guarded([&] { return fabric_script(ranks, elems, npush, clients, grads, weights, out); },
                   nullptr, 0, nullptr);
}

// push_slice error surface: returns the status code (0 ok, 5 ProtocolError).
int ref_push_slice_status(int ranks, std::int64_t elems, int client, int target,
                          std::int64_t offset, std::int64_t len) {
    return guarded(
        [&] {
            ShardFabric<std::int64_t> fab(ranks, elems);
            fab.push_slice(client, target, offset, std::vector<std::int64_t>(static_cast<std::size_t>(len), 1), 1);
            return 0;
        },
        nullptr, 0, nullptr);
}

// run_schedule over integer scripts: pushes given as (client, weight, grad) in
// per-client order. Writes the concatenated shards; returns max staged elems.
std::int64_t ref_run_schedule_i64(int ranks, std::int64_t elems, int npush, const int* clients,
                                  const std::int64_t* grads, const std::int64_t* weights,
                                  std::uint64_t seed, std::int64_t* out) {
    std::vector<ClientScript<std::int64_t>> scripts(static_cast<std::size_t>(ranks));
    for (int p = 0; p < npush; ++p) {
        std::vector<std::int64_t> g(grads + static_cast<std::int64_t>(p) * elems,
                                    grads + static_cast<std::int64_t>(p + 1) * elems);
        scripts[static_cast<std::size_t>(clients[p])].pushes.emplace_back(std::move(g), weights[p]);
    }
    auto r = run_schedule(ranks, elems, scripts, seed);
    auto cat = r.concatenated();
    for (std::size_t i = 0; i < cat.size(); ++i) out[i] = cat[i];
    return r.max_staged_elems;
}

// Host-core timing of the reference fabric for one FSDP unit of `elems`
// fp32 elements over `ranks` simulated ranks: every client gathers
// `gathers_per_client` times and scatter_accumulates `pushes_per_client`
// times, then one finalize_minibatch. Returns seconds for `iters` rounds.
double ref_fabric_seconds_f32(int ranks, std::int64_t elems, int gathers_per_client,
                              int pushes_per_client, int iters) {
    ShardFabric<float> fab(ranks, elems);
    std::vector<float> params(static_cast<std::size_t>(elems), 0.5f);
    fab.set_params("layer", params);
    std::vector<float> grad(static_cast<std::size_t>(elems), 0.25f);
    double sink = 0.0;
    auto t0 = std::chrono::steady_clock::now();
    for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < ranks; ++c) {
            for (int g = 0; g < gathers_per_client; ++g) sink += fab.gather(c, "layer").back();
            for (int p = 0; p < pushes_per_client; ++p) fab.scatter_accumulate(c, grad, 1.0f / ranks);
        }
        auto shards = fab.finalize_minibatch();
        sink += shards.back().empty() ? 0.0 : shards.back().back();
    }
    auto t1 = std::chrono::steady_clock::now();
    return sink >= 0.0 ? std::chrono::duration<double>(t1 - t0).count() : -1.0;
}

// The same sample on `threads` host threads, each moving its own FSDP unit
// through its own ShardFabric<float> (units are independent fabrics; one
// fabric is not thread-safe, and the reference's threaded driver serialises
// every client under one mutex, inc/primitives.hpp:296-303). Returns the wall
// time for all `threads` units; per-unit time = wall / threads.
double ref_fabric_seconds_f32_mt(int ranks, std::int64_t elems, int gathers_per_client,
                                 int pushes_per_client, int iters, int threads) {
    if (threads <= 1) return ref_fabric_seconds_f32(ranks, elems, gathers_per_client, pushes_per_client, iters);
    std::vector<std::thread> pool;
    std::vector<double> sec(static_cast<std::size_t>(threads), 0.0);
    auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            sec[static_cast<std::size_t>(t)] =
                ref_fabric_seconds_f32(ranks, elems, gathers_per_client, pushes_per_client, iters);
        });
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    for (double v : sec)
        if (v < 0.0) return -1.0;
    return std::chrono::duration<double>(t1 - t0).count();
}

// ---------------------------------------------------------------------------
// One ODC minibatch step of the reference's CPU path, measured (bench.py
// --impl reference and the GPU arm's cpu_baseline): every FSDP unit at its
// true size is one ShardFabric<float> (one fabric = one unit's gradient
// space, inc/primitives.hpp:158-159) with `ranks` simulated ranks. For every
// microbatch of client c in the step (the LB-Mini plan): gather the unit
// twice (forward + backward re-fetch, inc/primitives.hpp:177-179) and
// scatter_accumulate its gradient once (:181-188); then finalize_minibatch
// (:199-203) once per unit. Units are independent fabrics, so `threads` host
// threads take units off a shared queue (largest first); one fabric is only
// ever touched by one thread (it is not thread-safe).
struct RefStep {
    int ranks = 1;
    std::vector<std::int64_t> elems;
    std::vector<ShardFabric<float>*> fabs;
    std::vector<std::vector<float>> grads;  // one read-only gradient per unit size
    std::vector<int> grad_of;
};

void* ref_step_new(int ranks, int n_units, const std::int64_t* elems) {
    try {
        auto* h = new RefStep();
        h->ranks = ranks;
        for (int u = 0; u < n_units; ++u) {
            h->elems.push_back(elems[u]);
            auto* f = new ShardFabric<float>(ranks, elems[u]);
            f->set_params("unit", std::vector<float>(static_cast<std::size_t>(elems[u]), 0.01f));
            h->fabs.push_back(f);
            int g = -1;
            for (std::size_t k = 0; k < h->grads.size(); ++k)
                if (static_cast<std::int64_t>(h->grads[k].size()) == elems[u]) g = static_cast<int>(k);
            if (g < 0) {
                h->grads.emplace_back(static_cast<std::size_t>(elems[u]), 1e-3f);
                g = static_cast<int>(h->grads.size()) - 1;
            }
            h->grad_of.push_back(g);
        }
        return h;
    } catch (...) {
        return nullptr;
    }
}

void ref_step_free(void* hv) {
    auto* h = static_cast<RefStep*>(hv);
    if (!h) return;
    for (auto* f : h->fabs) delete f;
    delete h;
}

// micro[c] = microbatches of client c in this step. Returns wall seconds
// (negative on failure).
double ref_step_run(void* hv, const int* micro, int threads) {
    auto* h = static_cast<RefStep*>(hv);
    if (!h) return -1.0;
    const int n = static_cast<int>(h->fabs.size());
    std::vector<int> order(static_cast<std::size_t>(n));
    for (int u = 0; u < n; ++u) order[static_cast<std::size_t>(u)] = u;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return h->elems[static_cast<std::size_t>(a)] > h->elems[static_cast<std::size_t>(b)];
    });
    std::atomic<int> next{0};
    std::atomic<bool> failed{false};
    std::vector<double> sink(static_cast<std::size_t>(std::max(1, threads)), 0.0);
    auto work = [&](int t) {
        try {
            for (int i = next++; i < n; i = next++) {
                const int u = order[static_cast<std::size_t>(i)];
                ShardFabric<float>& f = *h->fabs[static_cast<std::size_t>(u)];
                const std::vector<float>& g = h->grads[static_cast<std::size_t>(h->grad_of[static_cast<std::size_t>(u)])];
                const float w = 1.0f / static_cast<float>(h->ranks);
                for (int c = 0; c < h->ranks; ++c)
                    for (int m = 0; m < micro[c]; ++m) {
                        sink[static_cast<std::size_t>(t)] += f.gather(c, "unit").back();  // forward fetch
                        sink[static_cast<std::size_t>(t)] += f.gather(c, "unit").back();  // backward re-fetch
                        f.scatter_accumulate(c, g, w);                                     // gradient push
                    }
                auto shards = f.finalize_minibatch();
                sink[static_cast<std::size_t>(t)] += shards.front().empty() ? 0.0 : shards.front().front();
            }
        } catch (...) {
            failed = true;
        }
    };
    auto t0 = std::chrono::steady_clock::now();
    if (threads <= 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    auto t1 = std::chrono::steady_clock::now();
    double s = 0.0;
    for (double v : sink) s += v;
    return (failed || s < 0.0) ? -1.0 : std::chrono::duration<double>(t1 - t0).count();
}

// Analytic compute-only runtimes (src/runtime.cpp:52-79) of a plan, for the
// predicted-speedup / bubble columns. Returns 0 ok.
int ref_runtime(int strategy, const std::int64_t* lens, std::int64_t n, int devices, int minibs,
                std::int64_t budget, double alpha, double beta, int layers, double* total_out,
                double* bubble_out) {
    return guarded(
        [&] {
            static const Strategy kS[] = {Strategy::LocalSort, Strategy::LbMicro, Strategy::LbMini,
                                          Strategy::VerlNative, Strategy::VerlOptimized};
            CostModel cm{alpha, beta, layers};
            auto res = plan(kS[strategy], workload_of(lens, n), devices, minibs, MemoryBudget{budget}, cm, 0);
            std::vector<RuntimeReport> reps;
            for (const auto& sol : res.steps)
                reps.push_back(strategy == 2 ? runtime_odc(sol, cm) : runtime_collective(sol, cm));
            auto agg = aggregate_reports(reps);
            *total_out = agg.total_time;
            *bubble_out = agg.bubble_rate;
            return 0;
        },
        nullptr, 0, nullptr);
}

}  // extern "C"
