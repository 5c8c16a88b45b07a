// lb.cpp — host C++ load balancer of the ODC path (LB-Mini for ODC, LB-Micro
// for the FSDP comparison path), plus the cost model and the seeded workload
// generator it consumes.
//
// A bit-exact restatement of the reference (src/ = /root/reference/proj/src):
//   * KK largest differencing          src/partition.cpp:84-128
//       heap top = widest spread, tie -> lowest min index (:33-39); merge pairs
//       a.parts[i] with b.parts[k-1-i] and re-sorts (sum desc, min asc) (:41-53)
//   * microbatch k loop                src/partition.cpp:266-276
//   * joint loop / split_to_k          src/partition.cpp:284-348
//   * plan() strategies                src/partition.cpp:423-580
//   * cost model                       src/cost_model.cpp:8-38
//   * generate_synthetic/scale_lengths src/workload.cpp:120-271
// Compiled with -ffp-contract=off so alpha*d*d + beta*d rounds like the reference.
//
// B200-build differences (all output-preserving):
//   * the heap moves states instead of copying heap.top() (:121);
//   * microbatch_partition starts its k loop at ceil(token_sum / budget):
//     any smaller k has a part above the budget by pigeonhole, so the first
//     fitting k — the reference's answer — is unchanged.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <fstream>
#include <istream>
#include <sstream>
#include <type_traits>
#include <variant>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numbers>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "common.hpp"
#include "odcsim/cost_model.hpp"
#include "odcsim/experiment.hpp"
#include "odcsim/partition.hpp"
#include "odcsim/runtime.hpp"
#include "odcsim/workload.hpp"

namespace odcsim {

// ---------------------------------------------------------------- logging
namespace {
std::atomic<int> g_log{static_cast<int>(LogLevel::Warn)};
}
LogLevel log_level() { return static_cast<LogLevel>(g_log.load(std::memory_order_relaxed)); }
void set_log_level(LogLevel level) { g_log.store(static_cast<int>(level), std::memory_order_relaxed); }
void set_log_level_from_env() {
    const char* v = std::getenv("ODC_SIM_LOG");
    if (!v) return;
    static const char* names[] = {"quiet", "warn", "info", "debug"};
    for (int i = 0; i < 4; ++i)
        if (!std::strcmp(v, names[i]) || (v[0] == '0' + i && v[1] == 0)) set_log_level(static_cast<LogLevel>(i));
}
void log_warn(const std::string& m) {
    if (log_level() >= LogLevel::Warn) std::fprintf(stderr, "[warn] %s\n", m.c_str());
}
void log_info(const std::string& m) {
    if (log_level() >= LogLevel::Info) std::fprintf(stderr, "[info] %s\n", m.c_str());
}
void log_debug(const std::string& m) {
    if (log_level() >= LogLevel::Debug) std::fprintf(stderr, "[debug] %s\n", m.c_str());
}

// ------------------------------------------------------------- cost model
void CostModel::validate() const {
    const bool ok = alpha >= 0.0 && beta >= 0.0 && alpha + beta > 0.0;
    if (!ok) throw ParamError("cost model requires alpha >= 0, beta >= 0, alpha + beta > 0");
    if (layers < 1) throw ParamError("cost model requires layers >= 1");
}

double compute_cost(const CostModel& m, Tokens s) {
    if (s < 1) throw ParamError("compute_cost requires length >= 1");
    const double d = static_cast<double>(s);
    const double quad = m.alpha * d * d;  // (alpha*d)*d, then + beta*d: reference order
    return quad + m.beta * d;
}

double microbatch_cost(const CostModel& m, std::span<const Tokens> lengths) {
    if (lengths.empty()) throw ParamError("microbatch_cost requires a non-empty microbatch");
    double acc = 0.0;
    for (Tokens s : lengths) acc += compute_cost(m, s);
    return acc;
}

Tokens token_budget(Tokens max_len, double ratio) {
    if (max_len < 1) throw ParamError("token_budget requires max_len >= 1");
    if (!(ratio >= 1.0)) throw ParamError("packing ratio must be >= 1 so a single max-length sample fits");
    return static_cast<Tokens>(std::floor(static_cast<double>(max_len) * ratio));
}

bool check_oom(std::span<const Tokens> lengths, const MemoryBudget& b) {
    Tokens total = 0;
    for (Tokens s : lengths) total += s;
    return total > b.max_tokens_per_microbatch;
}

// --------------------------------------------------------------- workload
Workload::Workload(std::vector<Sample> samples) : samples_(std::move(samples)) {
    if (samples_.empty()) throw ParamError("workload must contain at least one sample");
    for (const Sample& s : samples_) {
        if (s.length < 1)
            throw ParamError("sample " + std::to_string(s.id) + " has non-positive length " +
                             std::to_string(s.length));
        if (s.length > max_length_) max_length_ = s.length;
    }
}

std::vector<Tokens> Workload::lengths() const {
    std::vector<Tokens> v;
    v.reserve(samples_.size());
    for (const Sample& s : samples_) v.push_back(s.length);
    return v;
}

namespace {
double top53_uniform(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

Tokens to_length(double raw, Tokens cap) {
    if (!std::isfinite(raw)) return cap;
    const double r = std::round(raw);
    if (r < 1.0) return 1;
    if (r >= static_cast<double>(cap)) return cap;
    return static_cast<Tokens>(r);
}

void check_dist(const DistSpec& d) {
    if (auto* ln = std::get_if<LognormalDist>(&d)) {
        if (!(ln->sigma > 0.0) || !std::isfinite(ln->mu) || !std::isfinite(ln->sigma))
            throw ParamError("lognormal requires finite mu and sigma > 0");
    } else if (auto* pa = std::get_if<ParetoDist>(&d)) {
        if (!(pa->scale > 0.0) || !(pa->shape > 0.0)) throw ParamError("pareto requires scale > 0 and shape > 0");
    } else if (auto* un = std::get_if<UniformDist>(&d)) {
        if (un->lo < 1 || un->hi < un->lo) throw ParamError("uniform requires 1 <= lo <= hi");
    }
}

double kv(const std::string& args, const std::string& key) {
    auto p = args.find(key + "=");
    if (p == std::string::npos) throw FormatError("distribution spec missing '" + key + "='");
    p += key.size() + 1;
    auto e = args.find(',', p);
    std::string v = args.substr(p, e == std::string::npos ? std::string::npos : e - p);
    try {
        std::size_t used = 0;
        double x = std::stod(v, &used);
        if (used == v.size()) return x;
    } catch (...) {
    }
    throw FormatError("bad value for '" + key + "' in distribution spec: '" + v + "'");
}
}  // namespace

DistSpec parse_dist_spec(const std::string& text) {
    auto c = text.find(':');
    std::string name = text.substr(0, c), args = c == std::string::npos ? "" : text.substr(c + 1);
    DistSpec d;
    if (name == "lognormal") d = LognormalDist{kv(args, "mu"), kv(args, "sigma")};
    else if (name == "pareto") d = ParetoDist{kv(args, "scale"), kv(args, "shape")};
    else if (name == "uniform") d = UniformDist{static_cast<Tokens>(kv(args, "lo")), static_cast<Tokens>(kv(args, "hi"))};
    else throw FormatError("unknown distribution '" + name + "' (expected lognormal|pareto|uniform)");
    check_dist(d);
    return d;
}

Workload generate_synthetic(const DistSpec& dist, std::int64_t n, Tokens cap, std::uint64_t seed) {
    if (n < 1) throw ParamError("sample count must be >= 1");
    if (cap < 1) throw ParamError("length cap must be >= 1");
    check_dist(dist);
    std::mt19937_64 g(seed);
    std::vector<Sample> out;
    out.reserve(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) {
        Tokens len;
        if (auto* ln = std::get_if<LognormalDist>(&dist)) {
            const double u1 = top53_uniform(g);
            const double u2 = top53_uniform(g);
            const double z = std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(2.0 * std::numbers::pi * u2);
            len = to_length(std::exp(ln->mu + ln->sigma * z), cap);
        } else if (auto* pa = std::get_if<ParetoDist>(&dist)) {
            const double u = top53_uniform(g);
            len = to_length(pa->scale * std::pow(1.0 - u, -1.0 / pa->shape), cap);
        } else {
            const auto& un = std::get<UniformDist>(dist);
            len = un.lo + static_cast<Tokens>(g() % (static_cast<std::uint64_t>(un.hi - un.lo) + 1));
        }
        out.push_back(Sample{i, len});
    }
    return Workload(std::move(out));
}

Workload scale_lengths(const Workload& w, double ratio) {
    if (!(ratio > 0.0)) throw ParamError("scale ratio must be > 0");
    std::vector<Sample> s = w.samples();
    for (Sample& x : s) x.length = std::max<Tokens>(1, std::llround(static_cast<double>(x.length) * ratio));
    return Workload(std::move(s));
}

// "lognormal:mu=8,sigma=1.5" — the inverse of parse_dist_spec, numbers in the
// stream's default (6 significant digits) format (src/workload.cpp:120-131)
std::string format_dist_spec(const DistSpec& dist) {
    std::ostringstream os;
    std::visit(
        [&](const auto& d) {
            using D = std::decay_t<decltype(d)>;
            if constexpr (std::is_same_v<D, LognormalDist>) os << "lognormal:mu=" << d.mu << ",sigma=" << d.sigma;
            else if constexpr (std::is_same_v<D, ParetoDist>) os << "pareto:scale=" << d.scale << ",shape=" << d.shape;
            else os << "uniform:lo=" << d.lo << ",hi=" << d.hi;
        },
        dist);
    return os.str();
}

// one positive integer per line; whitespace-only lines skipped; anything else
// is a FormatError naming its 1-based line (src/workload.cpp:145-169)
Workload load_lengths(std::istream& in) {
    std::vector<Sample> out;
    std::string line;
    for (std::int64_t no = 1; std::getline(in, line); ++no) {
        const auto first = line.find_first_not_of(" \t\r");
        if (first == std::string::npos) continue;
        const auto last = line.find_last_not_of(" \t\r");
        const char* b = line.data() + first;
        const char* e = line.data() + last + 1;
        Tokens v = 0;
        const auto r = std::from_chars(b, e, v);
        if (r.ec != std::errc() || r.ptr != e)
            throw FormatError("line " + std::to_string(no) + ": not an integer: '" + std::string(b, e) + "'");
        if (v < 1) throw FormatError("line " + std::to_string(no) + ": length must be positive, got " + std::to_string(v));
        out.push_back(Sample{static_cast<std::int64_t>(out.size()), v});
    }
    if (out.empty()) throw FormatError("no lengths found in input");
    return Workload(std::move(out));
}

Workload load_lengths_file(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw FormatError("cannot open length file: " + path);
    return load_lengths(f);
}

// count / min / max / exact total / mean and nearest-rank p50, p90, p99: the
// smallest length with at least fraction p of the samples at or below it
// (src/workload.cpp:187-214)
WorkloadStats summarize(const Workload& w) {
    std::vector<Tokens> v = w.lengths();
    std::sort(v.begin(), v.end());
    const auto n = static_cast<std::int64_t>(v.size());
    auto rank = [&](double p) {
        std::int64_t k = static_cast<std::int64_t>(std::ceil(p * static_cast<double>(n)));
        return v[static_cast<std::size_t>(std::clamp<std::int64_t>(k, 1, n) - 1)];
    };
    WorkloadStats st;
    st.count = n;
    st.min = v.front();
    st.max = v.back();
    st.total = std::accumulate(v.begin(), v.end(), std::int64_t{0});
    st.mean = static_cast<double>(st.total) / static_cast<double>(n);
    st.p50 = rank(0.50);
    st.p90 = rank(0.90);
    st.p99 = rank(0.99);
    return st;
}

// -------------------------------------------------------------- KK engine
namespace {

constexpr int kNoIndex = std::numeric_limits<int>::max();

struct Bin {
    double sum = 0.0;
    int lo = kNoIndex;  // smallest original index in the bin
    std::vector<int> items;
};

// ordering of bins inside a tuple: heavier first, then lower index
inline bool heavier(const Bin& a, const Bin& b) { return a.sum != b.sum ? a.sum > b.sum : a.lo < b.lo; }

struct Tuple {
    std::vector<Bin> bins;
    int lo = kNoIndex;
    double spread = 0.0;
    void refresh() { spread = bins.front().sum - bins.back().sum; }
};

// max-heap order: wider spread on top, ties to the lower index
inline bool heap_less(const Tuple& a, const Tuple& b) { return a.spread != b.spread ? a.spread < b.spread : a.lo > b.lo; }

PartitionResult to_result(Tuple& t) {
    PartitionResult r;
    double lo = std::numeric_limits<double>::infinity(), hi = -lo;
    for (Bin& b : t.bins) {
        std::sort(b.items.begin(), b.items.end());
        lo = std::min(lo, b.sum);
        hi = std::max(hi, b.sum);
        r.sums.push_back(b.sum);
        r.parts.push_back(std::move(b.items));
    }
    r.spread = t.bins.empty() ? 0.0 : hi - lo;
    return r;
}

std::vector<int> order_by_cost_desc(std::span<const double> c) {
    std::vector<int> o(c.size());
    std::iota(o.begin(), o.end(), 0);
    std::sort(o.begin(), o.end(), [&](int a, int b) { return c[a] != c[b] ? c[a] > c[b] : a < b; });
    return o;
}

}  // namespace

PartitionResult kk_partition(std::span<const double> costs, int k, bool equal_size) {
    if (k < 1) throw ParamError("kk_partition requires k >= 1");
    const int n = static_cast<int>(costs.size());
    if (equal_size && n % k != 0)
        throw ParamError("equal_size requires k to divide the input size (" + std::to_string(k) +
                         " does not divide " + std::to_string(n) + ")");
    std::vector<Tuple> heap;
    heap.reserve(static_cast<std::size_t>(equal_size ? n / k : n));
    if (equal_size) {
        const std::vector<int> ord = order_by_cost_desc(costs);
        for (int g = 0; g < n / k; ++g) {
            Tuple t;
            t.bins.resize(static_cast<std::size_t>(k));
            for (int i = 0; i < k; ++i) {
                const int idx = ord[static_cast<std::size_t>(g * k + i)];
                t.bins[static_cast<std::size_t>(i)] = Bin{costs[idx], idx, {idx}};
                t.lo = std::min(t.lo, idx);
            }
            t.refresh();
            heap.push_back(std::move(t));
        }
    } else {
        for (int idx = 0; idx < n; ++idx) {
            Tuple t;
            t.bins.resize(static_cast<std::size_t>(k));
            t.bins[0] = Bin{costs[idx], idx, {idx}};
            t.lo = idx;
            t.refresh();
            heap.push_back(std::move(t));
        }
    }
    if (heap.empty()) {
        Tuple t;
        t.bins.resize(static_cast<std::size_t>(k));
        return to_result(t);
    }
    std::make_heap(heap.begin(), heap.end(), heap_less);
    while (heap.size() > 1) {
        std::pop_heap(heap.begin(), heap.end(), heap_less);
        Tuple a = std::move(heap.back());
        heap.pop_back();
        std::pop_heap(heap.begin(), heap.end(), heap_less);
        Tuple& b = heap.back();
        for (int i = 0; i < k; ++i) {
            Bin& dst = a.bins[static_cast<std::size_t>(i)];
            Bin& src = b.bins[static_cast<std::size_t>(k - 1 - i)];
            dst.sum += src.sum;
            dst.lo = std::min(dst.lo, src.lo);
            dst.items.insert(dst.items.end(), src.items.begin(), src.items.end());
        }
        std::sort(a.bins.begin(), a.bins.end(), heavier);
        a.lo = std::min(a.lo, b.lo);
        a.refresh();
        heap.back() = std::move(a);
        std::push_heap(heap.begin(), heap.end(), heap_less);
    }
    return to_result(heap.front());
}

PartitionResult brute_force_partition(std::span<const double> costs, int k, bool equal_size) {
    if (k < 1) throw ParamError("brute_force_partition requires k >= 1");
    const int n = static_cast<int>(costs.size());
    if (n > 14) throw ParamError("brute_force_partition is limited to 14 items, got " + std::to_string(n));
    if (equal_size && n % k != 0) throw ParamError("equal_size requires k to divide the input size");
    const std::vector<int> ord = order_by_cost_desc(costs);
    const int cap = equal_size ? n / k : n;
    std::vector<double> rest(static_cast<std::size_t>(n) + 1, 0.0);
    for (int i = n - 1; i >= 0; --i) rest[static_cast<std::size_t>(i)] = rest[static_cast<std::size_t>(i) + 1] + costs[ord[static_cast<std::size_t>(i)]];
    std::vector<double> sum(static_cast<std::size_t>(k), 0.0);
    std::vector<int> cnt(static_cast<std::size_t>(k), 0), pick(static_cast<std::size_t>(n), 0), best_pick;
    double best = std::numeric_limits<double>::infinity();
    // depth-first over canonical labelings (a new bin may only be opened in
    // order), pruned by the best spread found so far
    auto dfs = [&](auto&& self, int pos, int opened) -> void {
        auto [mn, mx] = std::minmax_element(sum.begin(), sum.end());
        if (pos == n) {
            if (*mx - *mn < best) {
                best = *mx - *mn;
                best_pick = pick;
            }
            return;
        }
        if (*mx - (*mn + rest[static_cast<std::size_t>(pos)]) >= best) return;
        const double c = costs[ord[static_cast<std::size_t>(pos)]];
        for (int b = 0; b < std::min(opened + 1, k); ++b) {
            if (cnt[static_cast<std::size_t>(b)] >= cap) continue;
            sum[static_cast<std::size_t>(b)] += c;
            ++cnt[static_cast<std::size_t>(b)];
            pick[static_cast<std::size_t>(pos)] = b;
            self(self, pos + 1, std::max(opened, b + 1));
            sum[static_cast<std::size_t>(b)] -= c;
            --cnt[static_cast<std::size_t>(b)];
        }
    };
    dfs(dfs, 0, 0);
    PartitionResult r;
    r.parts.assign(static_cast<std::size_t>(k), {});
    r.sums.assign(static_cast<std::size_t>(k), 0.0);
    for (int pos = 0; pos < n; ++pos) {
        const int b = best_pick[static_cast<std::size_t>(pos)], idx = ord[static_cast<std::size_t>(pos)];
        r.parts[static_cast<std::size_t>(b)].push_back(idx);
        r.sums[static_cast<std::size_t>(b)] += costs[idx];
    }
    for (auto& p : r.parts) std::sort(p.begin(), p.end());
    if (n > 0) {
        auto [lo, hi] = std::minmax_element(r.sums.begin(), r.sums.end());
        r.spread = *hi - *lo;
    }
    return r;
}

PartitionResult minibatch_partition(std::span<const Tokens> seqlens, int world_size, bool equal_size,
                                    const CostModel& cost) {
    if (world_size < 1) throw ParamError("world_size must be >= 1");
    cost.validate();
    std::vector<double> c;
    c.reserve(seqlens.size());
    for (Tokens s : seqlens) c.push_back(compute_cost(cost, s));
    return kk_partition(c, world_size, equal_size);
}

namespace {

bool fits(const std::vector<std::vector<int>>& parts, std::span<const Sample> s, const MemoryBudget& b) {
    for (const auto& p : parts) {
        if (p.empty()) continue;
        Tokens t = 0;
        for (int i : p) t += s[static_cast<std::size_t>(i)].length;
        if (t > b.max_tokens_per_microbatch) return false;
    }
    return true;
}

std::vector<double> costs_of(std::span<const Sample> s, const CostModel& cost) {
    std::vector<double> c;
    c.reserve(s.size());
    for (const Sample& x : s) c.push_back(compute_cost(cost, x.length));
    return c;
}

std::vector<std::vector<int>> split_to_k(std::vector<std::vector<int>> parts, int k, std::span<const Sample> s,
                                         const CostModel& cost) {
    while (static_cast<int>(parts.size()) < k) {
        int best = -1;
        Tokens best_tok = -1;
        int best_lo = kNoIndex;
        for (std::size_t p = 0; p < parts.size(); ++p) {
            if (parts[p].size() < 2) continue;
            Tokens t = 0;
            int lo = kNoIndex;
            for (int i : parts[p]) {
                t += s[static_cast<std::size_t>(i)].length;
                lo = std::min(lo, i);
            }
            if (t > best_tok || (t == best_tok && lo < best_lo)) {
                best = static_cast<int>(p);
                best_tok = t;
                best_lo = lo;
            }
        }
        if (best < 0) {
            parts.emplace_back();
            continue;
        }
        std::vector<int> whole = std::move(parts[static_cast<std::size_t>(best)]);
        std::vector<double> c;
        for (int i : whole) c.push_back(compute_cost(cost, s[static_cast<std::size_t>(i)].length));
        auto halves = kk_partition(c, 2, false).parts;
        for (auto& h : halves)
            for (int& i : h) i = whole[static_cast<std::size_t>(i)];
        parts[static_cast<std::size_t>(best)] = std::move(halves[0]);
        parts.push_back(std::move(halves[1]));
    }
    return parts;
}

}  // namespace

std::vector<std::vector<int>> microbatch_partition(std::span<const Sample> samples, const MemoryBudget& budget,
                                                   const CostModel& cost) {
    Tokens total = 0;
    for (const Sample& s : samples) {
        if (s.length > budget.max_tokens_per_microbatch)
            throw InfeasibleError("sample " + std::to_string(s.id) + " has length " + std::to_string(s.length) +
                                  " exceeding the microbatch budget of " +
                                  std::to_string(budget.max_tokens_per_microbatch) + " tokens");
        total += s.length;
    }
    const int n = static_cast<int>(samples.size());
    const std::vector<double> c = costs_of(samples, cost);
    // pigeonhole lower bound (see file header); budget >= every length >= 1 here
    int k = 1;
    if (budget.max_tokens_per_microbatch > 0 && total > 0)
        k = static_cast<int>(std::max<Tokens>(1, (total + budget.max_tokens_per_microbatch - 1) /
                                                      budget.max_tokens_per_microbatch));
    for (;; ++k) {
        auto parts = kk_partition(c, k, false).parts;
        if (fits(parts, samples, budget)) return parts;
        if (k >= n) throw InvariantError("microbatch partition failed at k == n");
    }
}

std::vector<std::vector<std::vector<int>>> microbatch_partition_joint(
    const std::vector<std::vector<Sample>>& per_device, const MemoryBudget& budget, const CostModel& cost) {
    std::vector<std::vector<std::vector<int>>> own;
    own.reserve(per_device.size());
    int k_star = 1;
    for (const auto& dev : per_device) {
        own.push_back(microbatch_partition(dev, budget, cost));
        k_star = std::max(k_star, static_cast<int>(own.back().size()));
    }
    std::vector<std::vector<std::vector<int>>> out;
    out.reserve(per_device.size());
    for (std::size_t d = 0; d < per_device.size(); ++d) {
        auto parts = kk_partition(costs_of(per_device[d], cost), k_star, false).parts;
        if (!fits(parts, per_device[d], budget)) parts = split_to_k(std::move(own[d]), k_star, per_device[d], cost);
        out.push_back(std::move(parts));
    }
    return out;
}

std::int64_t BatchingSolution::sample_count() const {
    std::int64_t n = 0;
    for (const auto& d : per_device)
        for (const auto& mb : d) n += static_cast<std::int64_t>(mb.sample_ids.size());
    return n;
}

Strategy parse_strategy(const std::string& name) {
    static const char* names[] = {"local-sort", "lb-micro", "lb-mini", "verl-native", "verl-optimized"};
    for (int i = 0; i < 5; ++i)
        if (name == names[i]) return static_cast<Strategy>(i);
    throw ParamError("unknown strategy '" + name + "' (expected local-sort|lb-micro|lb-mini|verl-native|verl-optimized)");
}

std::string strategy_name(Strategy s) {
    switch (s) {
        case Strategy::LocalSort: return "local-sort";
        case Strategy::LbMicro: return "lb-micro";
        case Strategy::LbMini: return "lb-mini";
        case Strategy::VerlNative: return "verl-native";
        case Strategy::VerlOptimized: return "verl-optimized";
    }
    throw InvariantError("unreachable strategy");
}

namespace {

template <typename T>
void fisher_yates(std::vector<T>& v, std::mt19937_64& g) {
    for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[g() % i]);
}

Microbatch build_mb(std::span<const Sample> pool, const std::vector<int>& idx) {
    Microbatch mb;
    mb.sample_ids.reserve(idx.size());
    mb.lengths.reserve(idx.size());
    for (int i : idx) {
        const Sample& s = pool[static_cast<std::size_t>(i)];
        mb.sample_ids.push_back(s.id);
        mb.lengths.push_back(s.length);
        mb.token_sum += s.length;
    }
    return mb;
}

std::vector<Sample> pick(std::span<const Sample> pool, const std::vector<int>& idx) {
    std::vector<Sample> v;
    v.reserve(idx.size());
    for (int i : idx) v.push_back(pool[static_cast<std::size_t>(i)]);
    return v;
}

BatchingSolution equal_micro(const std::vector<std::vector<Sample>>& pools,
                             const std::vector<std::vector<std::vector<int>>>& joint, int mbs, int step,
                             bool partial) {
    BatchingSolution sol;
    sol.mode = BatchingMode::EqualMicro;
    sol.minibatch_size_per_device = mbs;
    sol.step_index = step;
    sol.partial = partial;
    for (std::size_t d = 0; d < pools.size(); ++d) {
        std::vector<Microbatch> v;
        for (const auto& p : joint[d]) v.push_back(build_mb(pools[d], p));
        sol.per_device.push_back(std::move(v));
    }
    return sol;
}

BatchingSolution local_sort_step(std::span<const Sample> pool, int devices, int mbs, int step, bool partial) {
    std::vector<Sample> srt(pool.begin(), pool.end());
    std::sort(srt.begin(), srt.end(),
              [](const Sample& a, const Sample& b) { return a.length != b.length ? a.length > b.length : a.id < b.id; });
    BatchingSolution sol;
    sol.mode = BatchingMode::EqualMicro;
    sol.minibatch_size_per_device = mbs;
    sol.step_index = step;
    sol.partial = partial;
    sol.per_device.assign(static_cast<std::size_t>(devices), {});
    for (std::size_t i = 0; i < srt.size(); ++i) {
        Microbatch mb;
        mb.sample_ids.push_back(srt[i].id);
        mb.lengths.push_back(srt[i].length);
        mb.token_sum = srt[i].length;
        sol.per_device[i % static_cast<std::size_t>(devices)].push_back(std::move(mb));
    }
    std::size_t most = 0;
    for (const auto& d : sol.per_device) most = std::max(most, d.size());
    for (auto& d : sol.per_device) d.resize(most);
    return sol;
}

BatchingSolution balanced_step(std::span<const Sample> pool, int devices, int mbs, const MemoryBudget& budget,
                               const CostModel& cost, bool lb_mini, int step, bool partial) {
    const bool equal = !lb_mini && pool.size() % static_cast<std::size_t>(devices) == 0;
    if (!lb_mini && !equal)
        log_warn("step " + std::to_string(step) + ": pool not divisible by devices, dropping the equal-size constraint");
    std::vector<Tokens> lens;
    lens.reserve(pool.size());
    for (const Sample& s : pool) lens.push_back(s.length);
    const PartitionResult split = minibatch_partition(lens, devices, equal, cost);
    std::vector<std::vector<Sample>> pools;
    for (const auto& p : split.parts) pools.push_back(pick(pool, p));
    if (!lb_mini)
        return equal_micro(pools, microbatch_partition_joint(pools, budget, cost), mbs, step, partial);
    BatchingSolution sol;
    sol.mode = BatchingMode::VariableMicro;
    sol.minibatch_size_per_device = mbs;
    sol.step_index = step;
    sol.partial = partial;
    for (const auto& dev : pools) {
        std::vector<Microbatch> v;
        if (!dev.empty())
            for (const auto& p : microbatch_partition(dev, budget, cost)) v.push_back(build_mb(dev, p));
        sol.per_device.push_back(std::move(v));  // a rank may get zero microbatches
    }
    return sol;
}

}  // namespace

PlanResult plan(Strategy strategy, const Workload& w, int devices, int mbs, const MemoryBudget& budget,
                const CostModel& cost, std::uint64_t seed) {
    if (devices < 1) throw ParamError("devices must be >= 1");
    if (mbs < 1) throw ParamError("minibatch_size must be >= 1");
    cost.validate();
    if (budget.max_tokens_per_microbatch < w.max_length())
        throw InfeasibleError("microbatch budget " + std::to_string(budget.max_tokens_per_microbatch) +
                              " is below the max sample length " + std::to_string(w.max_length()));
    const std::vector<Sample>& all = w.samples();
    PlanResult out;
    const std::size_t D = static_cast<std::size_t>(devices), B = static_cast<std::size_t>(mbs);

    if (strategy == Strategy::VerlNative) {
        const std::size_t keep = all.size() - all.size() % D;
        for (std::size_t i = keep; i < all.size(); ++i) out.dropped_ids.push_back(all[i].id);
        if (!out.dropped_ids.empty())
            log_warn("verl-native: dropping " + std::to_string(out.dropped_ids.size()) +
                     " trailing samples to make the pool divisible by " + std::to_string(devices));
        if (keep == 0) throw ParamError("workload smaller than the device count");
        std::span<const Sample> kept(all.data(), keep);
        std::vector<Tokens> lens;
        for (const Sample& s : kept) lens.push_back(s.length);
        const PartitionResult split = minibatch_partition(lens, devices, true, cost);
        std::vector<std::vector<Sample>> rank_pool;
        for (int d = 0; d < devices; ++d) {
            auto p = pick(kept, split.parts[static_cast<std::size_t>(d)]);
            std::mt19937_64 g(seed + 0x9e3779b97f4a7c15ULL * static_cast<std::uint64_t>(d + 1));
            fisher_yates(p, g);
            rank_pool.push_back(std::move(p));
        }
        const std::size_t per_rank = rank_pool.front().size();
        for (std::size_t m = 0; m * B < per_rank; ++m) {  // ceil(per_rank / B) steps
            std::vector<std::vector<Sample>> step_pools;
            bool partial = false;
            for (std::size_t d = 0; d < D; ++d) {
                const std::size_t b = m * B, e = std::min(per_rank, b + B);
                partial = partial || (e - b) < B;
                step_pools.emplace_back(rank_pool[d].begin() + static_cast<std::ptrdiff_t>(b),
                                        rank_pool[d].begin() + static_cast<std::ptrdiff_t>(e));
            }
            out.steps.push_back(equal_micro(step_pools, microbatch_partition_joint(step_pools, budget, cost), mbs,
                                            static_cast<int>(m), partial));
        }
        return out;
    }

    std::vector<Sample> ordered = all;
    if (strategy == Strategy::VerlOptimized) {
        std::mt19937_64 g(seed);
        fisher_yates(ordered, g);
    }
    int step = 0;
    for (std::size_t b = 0; b < ordered.size(); b += D * B, ++step) {
        const std::size_t e = std::min(ordered.size(), b + D * B);
        std::span<const Sample> pool(ordered.data() + b, e - b);
        const bool partial = pool.size() < D * B;
        if (strategy == Strategy::LocalSort) out.steps.push_back(local_sort_step(pool, devices, mbs, step, partial));
        else out.steps.push_back(balanced_step(pool, devices, mbs, budget, cost, strategy == Strategy::LbMini, step, partial));
    }
    if (out.steps.empty()) throw ParamError("workload produced no steps");
    return out;
}

// ---------------------------------------------------------------- runtime
Scheme parse_scheme(const std::string& name) {
    if (name == "collective") return Scheme::Collective;
    if (name == "odc") return Scheme::Odc;
    throw ParamError("unknown scheme '" + name + "' (expected collective|odc)");
}
std::string scheme_name(Scheme s) { return s == Scheme::Collective ? "collective" : "odc"; }

namespace {
double mb_cost(const CostModel& c, const Microbatch& mb) { return mb.empty() ? 0.0 : microbatch_cost(c, mb.lengths); }

std::vector<double> busy_of(const BatchingSolution& sol, const CostModel& c) {
    std::vector<double> busy;
    for (const auto& d : sol.per_device) {
        double s = 0.0;
        for (const Microbatch& mb : d) s += mb_cost(c, mb);
        busy.push_back(s * static_cast<double>(c.layers));
    }
    return busy;
}

double idle_fraction(const std::vector<double>& busy, double total) {
    double s = 0.0;
    for (double b : busy) s += b;
    return 1.0 - s / (static_cast<double>(busy.size()) * total);
}

RuntimeReport report(Scheme scheme, const BatchingSolution& sol, double total, std::vector<double> busy) {
    if (!(total > 0.0)) throw ParamError("degenerate solution: zero total runtime");
    RuntimeReport r;
    r.scheme = scheme;
    r.total_time = total;
    r.per_device_busy = std::move(busy);
    r.bubble_rate = idle_fraction(r.per_device_busy, total);
    r.sample_count = sol.sample_count();
    r.samples_per_time = static_cast<double>(r.sample_count) / total;
    return r;
}
}  // namespace

RuntimeReport runtime_collective(const BatchingSolution& sol, const CostModel& cost) {
    cost.validate();
    if (sol.mode != BatchingMode::EqualMicro)
        throw ModeError("per-layer collectives require a uniform microbatch count; "
                        "minibatch-level balancing applies only to ODC");
    if (sol.per_device.empty()) throw ParamError("empty solution");
    const std::size_t m = sol.per_device.front().size();
    for (const auto& d : sol.per_device)
        if (d.size() != m) throw ModeError("EqualMicro solution has differing per-device microbatch counts");
    double total = 0.0;
    for (std::size_t i = 0; i < m; ++i) {
        double worst = 0.0;
        for (const auto& d : sol.per_device) worst = std::max(worst, mb_cost(cost, d[i]));
        total += worst;
    }
    total *= static_cast<double>(cost.layers);
    return report(Scheme::Collective, sol, total, busy_of(sol, cost));
}

RuntimeReport runtime_odc(const BatchingSolution& sol, const CostModel& cost) {
    cost.validate();
    if (sol.per_device.empty()) throw ParamError("empty solution");
    auto busy = busy_of(sol, cost);
    const double total = *std::max_element(busy.begin(), busy.end());
    return report(Scheme::Odc, sol, total, std::move(busy));
}

double bubble_rate(const RuntimeReport& r) {
    if (!(r.total_time > 0.0)) throw ParamError("bubble rate undefined for zero total time");
    return idle_fraction(r.per_device_busy, r.total_time);
}

double acceleration_ratio(const RuntimeReport& coll, const RuntimeReport& odc) {
    if (!(odc.total_time > 0.0)) throw ParamError("acceleration ratio undefined for zero ODC time");
    return coll.total_time / odc.total_time;
}

RuntimeReport aggregate_reports(std::span<const RuntimeReport> reps) {
    if (reps.empty()) throw ParamError("nothing to aggregate");
    RuntimeReport agg;
    agg.scheme = reps.front().scheme;
    agg.per_device_busy.assign(reps.front().per_device_busy.size(), 0.0);
    agg.steps = 0;
    for (const RuntimeReport& r : reps) {
        if (r.per_device_busy.size() != agg.per_device_busy.size())
            throw ParamError("cannot aggregate reports over differing device counts");
        agg.total_time += r.total_time;
        for (std::size_t d = 0; d < agg.per_device_busy.size(); ++d) agg.per_device_busy[d] += r.per_device_busy[d];
        agg.sample_count += r.sample_count;
        agg.steps += r.steps;
    }
    agg.bubble_rate = idle_fraction(agg.per_device_busy, agg.total_time);
    agg.samples_per_time = static_cast<double>(agg.sample_count) / agg.total_time;
    return agg;
}

// ------------------------------------------------------------ serialiser
namespace {
void put_ints(std::string& s, const std::vector<std::int64_t>& v) {
    s += '[';
    for (std::size_t i = 0; i < v.size(); ++i) {
        if (i) s += ',';
        s += std::to_string(v[i]);
    }
    s += ']';
}
}  // namespace

std::string solutions_to_json_string(const PlanResult& pr) {
    // keys in lexicographic order, compact: what nlohmann::json::dump() emits
    std::string s = "{\"dropped_ids\":";
    put_ints(s, pr.dropped_ids);
    s += ",\"steps\":[";
    for (std::size_t i = 0; i < pr.steps.size(); ++i) {
        const BatchingSolution& sol = pr.steps[i];
        if (i) s += ',';
        s += "{\"minibatch_size_per_device\":" + std::to_string(sol.minibatch_size_per_device);
        s += ",\"mode\":\"";
        s += sol.mode == BatchingMode::EqualMicro ? "equal-micro" : "variable-micro";
        s += "\",\"partial\":";
        s += sol.partial ? "true" : "false";
        s += ",\"per_device\":[";
        for (std::size_t d = 0; d < sol.per_device.size(); ++d) {
            if (d) s += ',';
            s += '[';
            for (std::size_t m = 0; m < sol.per_device[d].size(); ++m) {
                if (m) s += ',';
                s += "{\"sample_ids\":";
                put_ints(s, sol.per_device[d][m].sample_ids);
                s += ",\"token_sum\":" + std::to_string(sol.per_device[d][m].token_sum) + '}';
            }
            s += ']';
        }
        s += "],\"step\":" + std::to_string(sol.step_index) + '}';
    }
    s += "]}";
    return s;
}

}  // namespace odcsim

// ---------------------------------------------------------------- C ABI
namespace {
odcsim::Workload workload_from(const std::int64_t* lens, std::int64_t n) {
    if (n < 0 || (n > 0 && !lens)) throw odcsim::ParamError("bad length array");
    std::vector<odcsim::Sample> v;
    v.reserve(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) v.push_back({i, lens[i]});
    return odcsim::Workload(std::move(v));
}

odcsim::Strategy strategy_of(int s) {
    if (s < 0 || s > 4) throw odcsim::ParamError("strategy code must be 0..4");
    return static_cast<odcsim::Strategy>(s);
}

void emit(const std::string& s, char* out, std::int64_t cap, std::int64_t* needed) {
    if (needed) *needed = static_cast<std::int64_t>(s.size()) + 1;
    if (out && cap > 0) {
        const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
}
}  // namespace

extern "C" {

odc_status odc_plan_json(int strategy, const std::int64_t* lens, std::int64_t n, int devices, int minibs,
                         std::int64_t budget, double alpha, double beta, int layers, std::uint64_t seed, char* out,
                         std::int64_t cap, std::int64_t* needed) {
    return odc::guard([&] {
        auto pr = odcsim::plan(strategy_of(strategy), workload_from(lens, n), devices, minibs,
                               odcsim::MemoryBudget{budget}, odcsim::CostModel{alpha, beta, layers}, seed);
        emit(odcsim::solutions_to_json_string(pr), out, cap, needed);
    });
}

odc_status odc_plan_flat(int strategy, const std::int64_t* lens, std::int64_t n, int devices, int minibs,
                         std::int64_t budget, double alpha, double beta, std::uint64_t seed, std::int64_t* out,
                         std::int64_t cap, std::int64_t* needed) {
    return odc::guard([&] {
        auto pr = odcsim::plan(strategy_of(strategy), workload_from(lens, n), devices, minibs,
                               odcsim::MemoryBudget{budget}, odcsim::CostModel{alpha, beta, 1}, seed);
        std::vector<std::int64_t> f;
        f.push_back(static_cast<std::int64_t>(pr.steps.size()));
        for (const auto& sol : pr.steps) {
            f.push_back(static_cast<std::int64_t>(sol.per_device.size()));
            for (const auto& d : sol.per_device) {
                f.push_back(static_cast<std::int64_t>(d.size()));
                for (const auto& mb : d) {
                    f.push_back(static_cast<std::int64_t>(mb.sample_ids.size()));
                    f.insert(f.end(), mb.sample_ids.begin(), mb.sample_ids.end());
                }
            }
        }
        if (needed) *needed = static_cast<std::int64_t>(f.size());
        if (out && cap >= static_cast<std::int64_t>(f.size())) std::memcpy(out, f.data(), f.size() * 8);
    });
}

odc_status odc_kk_partition_json(const double* costs, int n, int k, int equal_size, char* out, std::int64_t cap,
                                 std::int64_t* needed) {
    return odc::guard([&] {
        auto r = odcsim::kk_partition(std::span<const double>(costs, static_cast<std::size_t>(n)), k, equal_size != 0);
        std::string s = "{\"parts\":[";
        for (std::size_t p = 0; p < r.parts.size(); ++p) {
            if (p) s += ',';
            s += '[';
            for (std::size_t i = 0; i < r.parts[p].size(); ++i) {
                if (i) s += ',';
                s += std::to_string(r.parts[p][i]);
            }
            s += ']';
        }
        char buf[64];
        s += "],\"spread\":";
        std::snprintf(buf, sizeof buf, "%.17g", r.spread);
        s += buf;
        s += ",\"sums\":[";
        for (std::size_t p = 0; p < r.sums.size(); ++p) {
            if (p) s += ',';
            std::snprintf(buf, sizeof buf, "%.17g", r.sums[p]);
            s += buf;
        }
        s += "]}";
        emit(s, out, cap, needed);
    });
}

odc_status odc_generate_synthetic(int dist, double p1, double p2, std::int64_t n, std::int64_t cap, std::uint64_t seed,
                                  double scale, std::int64_t* out) {
    return odc::guard([&] {
        odcsim::DistSpec d;
        if (dist == 0) d = odcsim::LognormalDist{p1, p2};
        else if (dist == 1) d = odcsim::ParetoDist{p1, p2};
        else if (dist == 2) d = odcsim::UniformDist{static_cast<odcsim::Tokens>(p1), static_cast<odcsim::Tokens>(p2)};
        else throw odcsim::ParamError("dist code must be 0..2");
        auto w = odcsim::generate_synthetic(d, n, cap, seed);
        if (scale != 1.0) w = odcsim::scale_lengths(w, scale);
        for (std::int64_t i = 0; i < n; ++i) out[i] = w.samples()[static_cast<std::size_t>(i)].length;
    });
}

}  // extern "C"
