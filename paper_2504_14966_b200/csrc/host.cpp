// Host side of the B200 scheduler: the reference-shaped C++ API of
// include/slosched_b200.hpp. Everything O(N) or O(N log N) that the reference runs once
// per anneal() call (candidates, shortcut, tables, final evaluation) stays on the host;
// the O(proposals x N) annealing loop runs on the GPU through include/slosched_gpu.h.
// There is no CPU fallback: an engine failure throws EngineError.
// P: = /root/reference/proj/.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <exception>
#include <future>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <thread>

#include "slosched_b200.hpp"
#include "slosched_gpu.h"
#include "internal.hpp"

namespace slosched {

// ================================================================ domain validation
// (semantics of P:src/core.cpp:8-170)
SloSpec SloSpec::e2e(double ms) {
    SloSpec s;
    s.kind = SloKind::E2E;
    s.e2e_ms = ms;
    return s;
}

SloSpec SloSpec::ttft_tpot(double ttft, double tpot) {
    SloSpec s;
    s.kind = SloKind::TTFT_TPOT;
    s.ttft_ms = ttft;
    s.tpot_ms = tpot;
    return s;
}

void SloSpec::validate() const {
    if (kind == SloKind::E2E) {
        if (!e2e_ms || !(*e2e_ms > 0.0)) throw DataError("SloSpec: E2E kind requires e2e_ms > 0");
        return;
    }
    if (!ttft_ms || !(*ttft_ms > 0.0) || !tpot_ms || !(*tpot_ms > 0.0))
        throw DataError("SloSpec: TTFT_TPOT kind requires ttft_ms > 0 and tpot_ms > 0");
}

void TaskClass::validate() const {
    slo.validate();
    if (auto g = std::get_if<GaussianPrior>(&output_prior)) {
        if (!(g->std_tokens >= 0.0) || !std::isfinite(g->mean_tokens) || !std::isfinite(g->std_tokens))
            throw DataError("TaskClass '" + name + "': Gaussian prior requires finite mean and std >= 0");
    } else if (auto r = std::get_if<RangePrior>(&output_prior)) {
        if (r->low < 1 || r->low > r->high)
            throw DataError("TaskClass '" + name + "': range prior requires 1 <= low <= high");
    }
}

void Request::validate() const {
    const std::string who = "request " + std::to_string(id);
    if (input_len < 1 || true_output_len < 1 || (predicted_output_len && *predicted_output_len < 1))
        throw DataError(who + ": non-positive length");
    if (!std::isfinite(arrival_time_ms) || arrival_time_ms < 0.0) throw DataError(who + ": invalid arrival time");
}

void LatencyCoefficients::validate() const {
    for (double v : {alpha_p, beta_p, gamma_p, delta_p, alpha_d, beta_d, gamma_d, delta_d})
        if (!std::isfinite(v)) throw DataError("LatencyCoefficients: non-finite value");
    if (alpha_p < 0.0 || alpha_d < 0.0) throw DataError("LatencyCoefficients: alpha_p and alpha_d must be >= 0");
}

std::size_t Schedule::request_count() const {
    std::size_t n = 0;
    for (const auto& b : batches) n += b.size();
    return n;
}

std::vector<int> Schedule::flatten() const {
    std::vector<int> out;
    out.reserve(request_count());
    for (const auto& b : batches) out.insert(out.end(), b.begin(), b.end());
    return out;
}

std::unordered_map<int, std::pair<int, int>> Schedule::positions() const {
    std::unordered_map<int, std::pair<int, int>> out;
    int pos = 0;
    for (int k = 0; k < static_cast<int>(batches.size()); ++k)
        for (int id : batches[k]) out[id] = {pos++, k};
    return out;
}

bool Schedule::is_partition_of(const std::vector<int>& ids, int max_batch) const {
    std::vector<int> got;
    for (const auto& b : batches) {
        if (b.empty() || (max_batch > 0 && static_cast<int>(b.size()) > max_batch)) return false;
        got.insert(got.end(), b.begin(), b.end());
    }
    std::vector<int> want = ids;
    if (got.size() != want.size()) return false;
    std::sort(got.begin(), got.end());
    std::sort(want.begin(), want.end());
    return std::adjacent_find(got.begin(), got.end()) == got.end() && got == want;
}

void InstanceState::validate() const {
    const std::string who = "instance " + std::to_string(id);
    if (remaining_mem > total_mem) throw DataError(who + ": remaining_mem > total_mem");
    if (!(mem_utility > 0.0) || mem_utility > 1.0) throw DataError(who + ": mem_utility must be in (0,1]");
    if (!(bytes_per_token > 0.0)) throw DataError(who + ": bytes_per_token must be > 0");
    if (max_batch_size < 1) throw DataError(who + ": max_batch_size must be >= 1");
}

const TaskClass& Workload::class_of(const Request& r) const {
    const TaskClass* t = find_class(r.task_class_id);
    if (!t) throw DataError("request " + std::to_string(r.id) + ": unknown task_class_id " + std::to_string(r.task_class_id));
    return *t;
}

const TaskClass* Workload::find_class(int class_id) const {
    if (classes.size() <= 8) {  // a handful of classes: a scan beats hashing
        for (const auto& t : classes)
            if (t.id == class_id) return &t;
        return nullptr;
    }
    auto it = class_index_.find(class_id);
    return it == class_index_.end() ? nullptr : &classes[it->second];
}

const Request* Workload::find_request(int request_id) const {
    if (!dense_.empty()) {
        const long long k = (long long)request_id - dense_lo_;
        if (k < 0 || k >= (long long)dense_.size() || !dense_[k]) return nullptr;
        return &requests[dense_[k] - 1];
    }
    auto it = request_index_.find(request_id);
    return it == request_index_.end() ? nullptr : &requests[it->second];
}

Workload validate_workload(std::vector<Request> requests, std::vector<TaskClass> classes) {
    Workload w;
    w.classes = std::move(classes);
    w.requests = std::move(requests);
    w.class_index_.reserve(w.classes.size());
    for (std::size_t i = 0; i < w.classes.size(); ++i) {
        w.classes[i].validate();
        if (!w.class_index_.emplace(w.classes[i].id, i).second)
            throw DataError("duplicate task class id " + std::to_string(w.classes[i].id));
    }
    const std::size_t n = w.requests.size();
    long long lo = 0, hi = -1;
    for (std::size_t i = 0; i < n; ++i) {
        const long long id = w.requests[i].id;
        lo = i ? std::min(lo, id) : id, hi = i ? std::max(hi, id) : id;
    }
    const bool dense = n > 0 && hi - lo < 4 * (long long)n + 64;
    if (dense) w.dense_lo_ = lo, w.dense_.assign((std::size_t)(hi - lo + 1), 0u);
    else w.request_index_.reserve(n);
    for (std::size_t i = 0; i < n; ++i) {
        const Request& r = w.requests[i];
        r.validate();
        bool fresh;
        if (dense) {
            std::uint32_t& slot = w.dense_[(std::size_t)(r.id - lo)];
            fresh = slot == 0;
            if (fresh) slot = (std::uint32_t)(i + 1);
        } else {
            fresh = w.request_index_.emplace(r.id, i).second;
        }
        if (!fresh) throw DataError("duplicate request id " + std::to_string(r.id));
        if (!w.find_class(r.task_class_id))
            throw DataError("request " + std::to_string(r.id) + ": unknown task_class_id " + std::to_string(r.task_class_id));
    }
    return w;
}

// ================================================================ rng (P:include/slosched/rng.hpp)
namespace {
std::uint64_t splitmix_finalize(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
}  // namespace

Rng::Rng(std::uint64_t seed) {
    std::uint64_t z = seed;
    for (auto& s : s_) s = splitmix_finalize(z += 0x9e3779b97f4a7c15ULL);
}

std::uint64_t Rng::next_u64() {
    const std::uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
    const std::uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return out;
}

double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

std::uint64_t Rng::uniform_index(std::uint64_t n) {
    unsigned __int128 m = static_cast<unsigned __int128>(next_u64()) * n;
    if (static_cast<std::uint64_t>(m) < n) {
        const std::uint64_t floor = (0 - n) % n;
        while (static_cast<std::uint64_t>(m) < floor) m = static_cast<unsigned __int128>(next_u64()) * n;
    }
    return static_cast<std::uint64_t>(m >> 64);
}

double Rng::normal() {
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

std::uint64_t Rng::derive(std::uint64_t seed, std::uint64_t stream) {
    return splitmix_finalize(seed + 0x9e3779b97f4a7c15ULL * (stream + 1));
}

// ================================================================ latency model
// Eq. 14-19; operand order as P:src/latency_model.cpp:86-113 so the
// tables are bit-identical to the reference's.
double predict_prefill(const LatencyCoefficients& c, int b, int input_len) {
    const double bd = b, ld = input_len;
    return c.alpha_p * bd * ld + c.beta_p * bd + c.gamma_p * ld + c.delta_p;
}

double predict_per_token_decode(const LatencyCoefficients& c, int b, int accumulated_len) {
    const double bd = b, ld = accumulated_len;
    return c.alpha_d * bd * ld + c.beta_d * bd + c.gamma_d * ld + c.delta_d;
}

double predict_decode_total(const LatencyCoefficients& c, int b, int input_len, int output_len) {
    const double bd = b, li = input_len, lo = output_len;
    const double per_token_slope = c.alpha_d * bd + c.gamma_d;
    const double summed_len = lo * li + lo * (lo + 1.0) / 2.0;
    return per_token_slope * summed_len + lo * (c.beta_d * bd + c.delta_d);
}

double predict_exec(const LatencyCoefficients& c, int b, int input_len, int output_len) {
    return predict_prefill(c, b, input_len) + predict_decode_total(c, b, input_len, output_len);
}

double predict_tpot(const LatencyCoefficients& c, int b, int input_len, int output_len) {
    if (output_len <= 0) throw std::invalid_argument("predict_tpot: TPOT undefined for zero output");
    return predict_decode_total(c, b, input_len, output_len) / static_cast<double>(output_len);
}

LatencyCoefficients table_coefficients() { return {0.1, 5.7, 0.01, 43.67, 0.0002, 0.275, 0.00088, 15.85}; }

// ================================================================ objective
// (P:src/objective.cpp:7-82)
namespace {
const Request& require_predicted(const Workload& w, int id, const char* what) {
    const Request* r = w.find_request(id);
    if (!r) throw DataError(std::string(what) + " references unknown request " + std::to_string(id));
    if (!r->predicted_output_len) throw DataError("request " + std::to_string(id) + " missing predicted length");
    return *r;
}
double max_of(double a, double b) { return a < b ? b : a; }  // std::max semantics

// Positions 0..n-1 in ascending (key[i], tie[i], i) order (tie: optional secondary key) -- the
// order of a stable sort -- by an LSD radix sort of order-preserving bit patterns (8-bit digits,
// constant digits skipped): a comparison sort of a few thousand doubles is dominated by branch
// mispredictions. Keys are never NaN (execs, latest starts and arrival times).
std::vector<int> order_by_key(const std::vector<double>& key, const std::vector<int>* tie = nullptr) {
    const int n = static_cast<int>(key.size());
    std::vector<uint64_t> k(n), k2(n);
    std::vector<int> idx(n), idx2(n);
    for (int i = 0; i < n; ++i) idx[i] = i;
    auto passes = [&](int bits, auto&& digit_key) {
        uint64_t all_or = 0, all_and = ~0ull;
        for (int i = 0; i < n; ++i) {
            k[i] = digit_key(idx[i]);
            all_or |= k[i], all_and &= k[i];
        }
        for (int shift = 0; shift < bits; shift += 8) {
            if ((((all_or ^ all_and) >> shift) & 0xffu) == 0) continue;  // every key has this digit
            int cnt[257] = {};
            for (int i = 0; i < n; ++i) ++cnt[((k[i] >> shift) & 0xffu) + 1];
            for (int d = 0; d < 256; ++d) cnt[d + 1] += cnt[d];
            for (int i = 0; i < n; ++i) {
                const int at = cnt[(k[i] >> shift) & 0xffu]++;
                k2[at] = k[i], idx2[at] = idx[i];
            }
            k.swap(k2), idx.swap(idx2);
        }
    };
    if (tie) passes(32, [&](int i) { return (uint64_t)((uint32_t)(*tie)[i] ^ 0x80000000u); });
    passes(64, [&](int i) {
        const double d = key[i] == 0.0 ? 0.0 : key[i];  // -0 ties +0, as under <
        uint64_t b;
        std::memcpy(&b, &d, sizeof b);
        return (b >> 63) ? ~b : (b | (1ull << 63));
    });
    return idx;
}
}  // namespace

std::vector<ExecProfile> batch_exec_profile(const Schedule& s, const LatencyCoefficients& c, const Workload& w) {
    std::vector<ExecProfile> out;
    out.reserve(s.request_count());
    for (const auto& batch : s.batches) {
        const int b = static_cast<int>(batch.size());
        for (int id : batch) {
            const Request& r = require_predicted(w, id, "schedule");
            const int lo = *r.predicted_output_len;
            out.push_back({id, predict_exec(c, b, r.input_len, lo), predict_prefill(c, b, r.input_len),
                           predict_tpot(c, b, r.input_len, lo), is_extrapolated(r.input_len, lo)});
        }
    }
    return out;
}

std::vector<double> waiting_times(const Schedule& s, const std::vector<ExecProfile>& profiles) {
    std::vector<double> waits;
    waits.reserve(profiles.size());
    double elapsed = 0.0;
    std::size_t i = 0;
    for (const auto& batch : s.batches) {
        double makespan = 0.0;
        for (std::size_t k = 0; k < batch.size(); ++k, ++i) {
            waits.push_back(elapsed);
            makespan = max_of(makespan, profiles[i].exec_ms);
        }
        elapsed += makespan;
    }
    return waits;
}

bool meets_slo(const SloSpec& slo, double e2e_ms, double ttft_ms, double tpot_ms) {
    if (slo.kind == SloKind::E2E) return e2e_ms <= *slo.e2e_ms;
    return ttft_ms <= *slo.ttft_ms && tpot_ms <= *slo.tpot_ms;
}

namespace {
// batch_exec_profile + waiting_times + the metrics pass of P:src/objective.cpp fused into one pass
// over the schedule (one request lookup each); the same operations in the same order, so every
// metric, n, t and g are bit-identical to the three-pass form
EvaluatedSchedule evaluate_owned(Schedule&& s, const LatencyCoefficients& c, const Workload& w) {
    EvaluatedSchedule ev;
    ev.per_request.reserve(s.request_count());
    double elapsed = 0.0;
    for (const auto& batch : s.batches) {
        const int b = static_cast<int>(batch.size());
        double makespan = 0.0;
        for (int id : batch) {
            const Request& r = require_predicted(w, id, "schedule");
            const int lo = *r.predicted_output_len;
            RequestMetrics m;
            m.request_id = id;
            m.wait_ms = elapsed;
            m.exec_ms = predict_exec(c, b, r.input_len, lo);
            m.e2e_ms = m.exec_ms + elapsed;
            m.ttft_ms = predict_prefill(c, b, r.input_len) + elapsed;
            m.tpot_ms = predict_tpot(c, b, r.input_len, lo);
            m.extrapolated = is_extrapolated(r.input_len, lo);
            m.slo_met = meets_slo(w.class_of(r).slo, m.e2e_ms, m.ttft_ms, m.tpot_ms);
            makespan = max_of(makespan, m.exec_ms);
            ev.n += m.slo_met ? 1 : 0;
            ev.t_ms += m.e2e_ms;
            ev.per_request.push_back(m);
        }
        elapsed += makespan;
    }
    ev.g = ev.t_ms > 0.0 ? static_cast<double>(ev.n) / ev.t_ms : 0.0;
    ev.schedule = std::move(s);
    return ev;
}
}  // namespace

EvaluatedSchedule evaluate(const Schedule& s, const LatencyCoefficients& c, const Workload& w) {
    return evaluate_owned(Schedule(s), c, w);
}

// ================================================================ priority mapper
void AnnealConfig::validate() const {
    if (!(t0 > t_thres) || !(t_thres > 0.0)) throw DataError("AnnealConfig: requires t0 > t_thres > 0");
    if (iter < 1) throw DataError("AnnealConfig: iter must be >= 1");
    if (!(tau > 0.0) || !(tau < 1.0)) throw DataError("AnnealConfig: tau must be in (0,1)");
    if (objective_scale && !(*objective_scale >= 0.0)) throw DataError("AnnealConfig: objective_scale must be >= 0");
    if (engine.mode == SearchMode::Chains && engine.chains < 1) throw DataError("AnnealConfig: engine.chains must be >= 1");
    if (!(engine.budget_ms >= 0.0)) throw DataError("AnnealConfig: engine.budget_ms must be >= 0");
    for (double m : engine.scale_ladder)
        if (!(m >= 0.0)) throw DataError("AnnealConfig: scale_ladder entries must be >= 0");
}

namespace {
// doubles <-> integers in the same order (-0.0 and +0.0 share key 0)
inline long long dkey(double x) {
    long long b;
    std::memcpy(&b, &x, sizeof b);
    return b >= 0 ? b : LLONG_MIN - b;
}
inline double dval(long long k) {
    const long long b = k >= 0 ? k : LLONG_MIN - k;
    double x;
    std::memcpy(&x, &b, sizeof x);
    return x;
}
}  // namespace

// The largest d with fl(d + c) <= s. fl(d + c) is nondecreasing in d, so the d that pass form a
// down-set: bracket its end from s - c by doubling steps in key space, then bisect (<= ~130 probes;
// a walk one ulp at a time would need up to 2^52 steps when s - c is near 0 and c is not).
double latest_start(double s, double c) {
    const double d0 = s - c;
    if (std::isnan(d0)) return -std::numeric_limits<double>::infinity();
    if (std::isinf(d0)) return d0;
    const long long kmax = dkey(std::numeric_limits<double>::max()), kmin = dkey(-std::numeric_limits<double>::max());
    auto ok = [&](long long k) { return dval(k) + c <= s; };
    long long lo, hi;  // ok(lo), !ok(hi) (hi may be one past the finite range)
    const long long k0 = dkey(d0);
    if (ok(k0)) {
        lo = k0;
        long long step = 1;
        for (;;) {
            const long long t = lo + step > kmax ? kmax + 1 : lo + step;
            if (t > kmax || !ok(t)) {
                hi = t;
                break;
            }
            lo = t, step *= 2;
        }
    } else {
        hi = k0;
        long long step = 1;
        for (;;) {
            const long long t = hi - step < kmin ? kmin : hi - step;
            if (ok(t)) {
                lo = t;
                break;
            }
            if (t == kmin) return -std::numeric_limits<double>::infinity();
            hi = t, step *= 2;
        }
    }
    while (hi - lo > 1) {
        const long long m = lo + (hi - lo) / 2;
        if (ok(m)) lo = m;
        else hi = m;
    }
    return dval(lo);
}

namespace {

Schedule pack_greedy(const std::vector<int>& ordered, int max_batch) {
    Schedule s;
    for (std::size_t i = 0; i < ordered.size(); i += max_batch)
        s.batches.emplace_back(ordered.begin() + i, ordered.begin() + std::min(ordered.size(), i + max_batch));
    return s;
}

}  // namespace

std::pair<Schedule, Schedule> initial_candidates(const Workload& w, const std::vector<int>& ids,
                                                 const LatencyCoefficients& c, int max_batch) {
    // ascending (key, id): the comparator of P:src/priority_mapper.cpp:297-308, its keys computed
    // once per id
    const std::size_t n = ids.size();
    std::vector<double> exec_key(n), arrival_key(n);
    for (std::size_t i = 0; i < n; ++i) {
        const Request& r = require_predicted(w, ids[i], "initial_candidates");
        exec_key[i] = predict_exec(c, max_batch, r.input_len, *r.predicted_output_len);
        arrival_key[i] = r.arrival_time_ms;
    }
    auto ordered = [&](const std::vector<double>& key) {
        std::vector<int> out(n);
        const std::vector<int> pos = order_by_key(key, &ids);
        for (std::size_t i = 0; i < n; ++i) out[i] = ids[pos[i]];
        return out;
    };
    return {pack_greedy(ordered(exec_key), max_batch), pack_greedy(ordered(arrival_key), max_batch)};
}

std::optional<EvaluatedSchedule> shortcut_check(const Schedule& sorted_schedule, const LatencyCoefficients& c,
                                                const Workload& w) {
    EvaluatedSchedule ev = evaluate(sorted_schedule, c, w);
    if (ev.n == static_cast<int>(ev.per_request.size())) return ev;
    return std::nullopt;
}

// Schedule-level moves with the reference's draw discipline (P:src/priority_mapper.cpp:41-90,322-338)
namespace {

std::pair<int, int> locate(const Schedule& s, std::size_t flat_pos) {
    for (int k = 0; k < static_cast<int>(s.batches.size()); ++k) {
        if (flat_pos < s.batches[k].size()) return {k, static_cast<int>(flat_pos)};
        flat_pos -= s.batches[k].size();
    }
    return {-1, -1};
}

void drop_if_empty(Schedule& s, int k) {
    if (s.batches[k].empty()) s.batches.erase(s.batches.begin() + k);
}

std::optional<Schedule> move_squeeze(const Schedule& s, Rng& rng, int max_batch) {
    if (s.batches.size() < 2) return std::nullopt;
    const std::size_t head = s.batches.front().size();
    const auto [k, j] = locate(s, head + rng.uniform_index(s.request_count() - head));
    if (static_cast<int>(s.batches[k - 1].size()) >= max_batch) return std::nullopt;
    Schedule out = s;
    out.batches[k - 1].push_back(out.batches[k][j]);
    out.batches[k].erase(out.batches[k].begin() + j);
    drop_if_empty(out, k);
    return out;
}

std::optional<Schedule> move_delay(const Schedule& s, Rng& rng, int max_batch) {
    const std::size_t n = s.request_count();
    if (n == 0) return std::nullopt;
    const auto [k, j] = locate(s, rng.uniform_index(n));
    const bool has_next = k + 1 < static_cast<int>(s.batches.size());
    if (has_next && static_cast<int>(s.batches[k + 1].size()) >= max_batch) return std::nullopt;
    Schedule out = s;
    const int id = out.batches[k][j];
    if (has_next) out.batches[k + 1].push_back(id);
    else out.batches.push_back({id});
    out.batches[k].erase(out.batches[k].begin() + j);
    drop_if_empty(out, k);
    return out;
}

std::optional<Schedule> move_swap(const Schedule& s, Rng& rng) {
    const std::size_t n = s.request_count();
    if (n < 2) return std::nullopt;
    const std::size_t a = rng.uniform_index(n);
    std::size_t b = rng.uniform_index(n - 1);
    if (b >= a) ++b;
    const auto la = locate(s, a), lb = locate(s, b);
    Schedule out = s;
    std::swap(out.batches[la.first][la.second], out.batches[lb.first][lb.second]);
    return out;
}

}  // namespace

Schedule neighbor(const Schedule& s, Rng& rng, int max_batch) {
    if (s.request_count() == 0) return s;
    for (int attempt = 0; attempt < 8; ++attempt) {
        std::optional<Schedule> out;
        switch (rng.uniform_index(3)) {
            case 0: out = move_squeeze(s, rng, max_batch); break;
            case 1: out = move_delay(s, rng, max_batch); break;
            default: out = move_swap(s, rng); break;
        }
        if (out) return std::move(*out);
    }
    if (auto out = move_swap(s, rng)) return std::move(*out);
    return s;
}

// ---------------------------------------------------------------- engine contexts
namespace {

struct CtxDeleter {
    void operator()(slo_ctx* c) const { slo_ctx_destroy(c); }
};
using CtxPtr = std::unique_ptr<slo_ctx, CtxDeleter>;

// A small pool of engine contexts per device, so concurrent anneal() calls (allowed by
// the reference contract) each own a context while they run.
class CtxPool {
public:
    static CtxPool& get() {
        static CtxPool* pool = new CtxPool();  // leaked on purpose: no CUDA teardown at exit
        return *pool;
    }
    CtxPtr acquire(int device) {
        {
            std::lock_guard<std::mutex> g(mu_);
            auto& v = free_[device];
            if (!v.empty()) {
                CtxPtr c(v.back());
                v.pop_back();
                return c;
            }
        }
        slo_ctx* c = nullptr;
        if (slo_ctx_create(device, &c) != SLO_OK) throw EngineError(std::string("B200 engine: ") + slo_last_error());
        return CtxPtr(c);
    }
    void release(int device, CtxPtr c) {
        std::lock_guard<std::mutex> g(mu_);
        free_[device].push_back(c.release());
    }

private:
    std::mutex mu_;
    std::unordered_map<int, std::vector<slo_ctx*>> free_;
};

int resolve_device(int requested) {
    if (requested >= 0) return requested;
    if (const char* e = std::getenv("SLOSCHED_DEVICE")) return std::atoi(e);
    return 0;
}

void engine_check(int rc) {
    if (rc == SLO_OK) return;
    const std::string msg = slo_last_error();
    if (rc == SLO_ERR_DATA) throw DataError(msg);
    if (rc == SLO_ERR_CAPACITY) throw CapacityError(msg);
    if (rc == SLO_ERR_ARG) throw std::invalid_argument(msg);
    throw EngineError("B200 engine: " + msg);
}

struct GroupDeleter {
    void operator()(slo_group* g) const { slo_group_destroy(g); }
};
using GroupPtr = std::unique_ptr<slo_group, GroupDeleter>;

// Device groups (one context per device + one NCCL communicator) keyed by their device list;
// creating a communicator is expensive (tens of ms), so groups are kept for reuse.
class GroupPool {
public:
    static GroupPool& get() {
        static GroupPool* pool = new GroupPool();  // leaked on purpose, like CtxPool
        return *pool;
    }
    GroupPtr acquire(const std::vector<int>& devs) {
        {
            std::lock_guard<std::mutex> g(mu_);
            auto& v = free_[devs];
            if (!v.empty()) {
                GroupPtr p(v.back());
                v.pop_back();
                return p;
            }
        }
        slo_group* g = nullptr;
        if (int rc = slo_group_create(static_cast<int32_t>(devs.size()), devs.data(), &g)) engine_check(rc);
        return GroupPtr(g);
    }
    void release(const std::vector<int>& devs, GroupPtr g) {
        std::lock_guard<std::mutex> l(mu_);
        free_[devs].push_back(g.release());
    }

private:
    std::mutex mu_;
    std::map<std::vector<int>, std::vector<slo_group*>> free_;
};

// Where one anneal() runs: a pooled context on one device, the caller's rank context (one
// process per GPU, NCCL communicator attached), or a pooled group of devices in this process.
class EngineHandle {
public:
    explicit EngineHandle(const EngineOptions& eo) {
        if (eo.comm_ctx) {
            external_ = eo.comm_ctx;
        } else if (eo.devices.size() > 1) {
            devs_ = eo.devices;
        } else {
            device_ = eo.devices.size() == 1 ? eo.devices[0] : resolve_device(eo.device);
        }
    }
    ~EngineHandle() {
        if (!ok_) return;  // a failed call destroys its context / group instead of pooling it
        if (ctx_) CtxPool::get().release(device_, std::move(ctx_));
        if (group_) GroupPool::get().release(devs_, std::move(group_));
    }
    void problem_set(int n, int mb, const double* exec, const double* deadline) {
        ok_ = false;
        if (!devs_.empty()) {
            group_ = GroupPool::get().acquire(devs_);
            engine_check(slo_group_problem_set(group_.get(), n, mb, exec, deadline));
        } else {
            if (!external_) ctx_ = CtxPool::get().acquire(device_);
            engine_check(slo_problem_set(ctx(), n, mb, exec, deadline));
        }
        ok_ = true;
    }
    bool ready() const { return group_ || ctx_ || external_; }
    // the chain slice of this call: the caller's, else (rank context) this rank's share
    void slice(const EngineOptions& eo, int chains, int* b, int* e) const {
        *b = eo.chain_begin, *e = eo.chain_end < 0 ? chains : eo.chain_end;
        if (external_ && eo.chain_end < 0) {
            int32_t nr = 1, rk = 0;
            engine_check(slo_ctx_comm_info(external_, &nr, &rk));
            const int base = chains / nr, extra = chains % nr;
            *b = rk * base + std::min<int>(rk, extra);
            *e = *b + base + (rk < extra ? 1 : 0);
        }
    }
    void anneal(const slo_chain_params& prm, const std::vector<int>& sp, const std::vector<int>& ss,
                std::vector<int>& bp, std::vector<int>& bs, int* nb, slo_chain_result* cr) {
        ok_ = false;
        if (group_ && prm.rng_mode == SLO_RNG_PHILOX)
            engine_check(slo_group_anneal_chains(group_.get(), &prm, sp.data(), ss.data(), static_cast<int>(ss.size()),
                                                 bp.data(), bs.data(), nb, cr));
        else
            engine_check(slo_anneal_chains(ctx(), &prm, sp.data(), ss.data(), static_cast<int>(ss.size()), bp.data(),
                                           bs.data(), nb, cr));
        ok_ = true;
        exchanged_ = true;
    }
    // A rank context whose call fails before its exchange joins it with an empty slot, so the
    // other ranks' collective completes (and they report the job's result without this rank).
    void abandon(int n) noexcept {
        if (external_ && !exchanged_ && n >= 1 && n <= SLO_MAX_N) {
            int32_t nr = 1, rk = 0;
            if (slo_ctx_comm_info(external_, &nr, &rk) == SLO_OK && nr > 1) slo_ctx_exchange_empty(external_, n);
        }
        exchanged_ = true;
    }

private:
    slo_ctx* ctx() const { return external_ ? external_ : (ctx_ ? ctx_.get() : slo_group_ctx(group_.get(), 0)); }
    int device_ = 0;
    std::vector<int> devs_;
    slo_ctx* external_ = nullptr;
    bool exchanged_ = false;
    CtxPtr ctx_;
    GroupPtr group_;
    bool ok_ = true;
};

}  // namespace

namespace {
// Host worker threads shared by every anneal() call (its table build, the deadline-first variants,
// the table upload): spawning threads per call cost ~20-40 us each on the decision's critical path.
// A TaskGroup waits for its tasks in wait() and in its destructor (an early return or an exception
// never leaves a task running on the caller's stack); a waiting thread runs queued tasks itself, so
// nested groups cannot starve the pool.
class HostPool {
public:
    static HostPool& get() {
        static HostPool p(std::max(2u, std::min(8u, std::thread::hardware_concurrency())));
        return p;
    }
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> g(mu_);
            q_.push_back(std::move(f));
        }
        cv_.notify_one();
    }
    bool try_run_one() {
        std::function<void()> f;
        {
            std::lock_guard<std::mutex> g(mu_);
            if (q_.empty()) return false;
            f = std::move(q_.front());
            q_.pop_front();
        }
        f();
        return true;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }

private:
    explicit HostPool(unsigned n) {
        for (unsigned i = 0; i < n; ++i)
            th_.emplace_back([this] {
                while (true) {
                    std::function<void()> f;
                    {
                        std::unique_lock<std::mutex> l(mu_);
                        cv_.wait(l, [&] { return stop_ || !q_.empty(); });
                        if (q_.empty()) return;
                        f = std::move(q_.front());
                        q_.pop_front();
                    }
                    f();
                }
            });
    }
    std::vector<std::thread> th_;
    std::deque<std::function<void()>> q_;
    std::mutex mu_;
    std::condition_variable cv_;
    bool stop_ = false;
};

class TaskGroup {
public:
    template <typename F>
    void run(F&& f) {
        {
            std::lock_guard<std::mutex> g(mu_);
            ++pending_;
        }
        HostPool::get().submit([this, fn = std::forward<F>(f)]() mutable {
            std::exception_ptr e;
            try {
                fn();
            } catch (...) {
                e = std::current_exception();
            }
            std::lock_guard<std::mutex> g(mu_);
            if (e && !err_) err_ = e;
            if (--pending_ == 0) cv_.notify_all();
        });
    }
    void wait() {
        drain();
        std::exception_ptr e;
        {
            std::lock_guard<std::mutex> g(mu_);
            std::swap(e, err_);
        }
        if (e) std::rethrow_exception(e);
    }
    ~TaskGroup() { drain(); }

private:
    void drain() {
        while (true) {
            {
                std::lock_guard<std::mutex> g(mu_);
                if (pending_ == 0) return;
            }
            if (HostPool::get().try_run_one()) continue;
            std::unique_lock<std::mutex> l(mu_);
            cv_.wait_for(l, std::chrono::microseconds(50), [&] { return pending_ == 0; });
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    int pending_ = 0;
    std::exception_ptr err_;
};
}  // namespace

void cost_tables(const Workload& w, const std::vector<int>& ids, const LatencyCoefficients& c, int max_batch,
                 std::vector<double>& exec, std::vector<double>& deadline) {
    std::vector<int> sorted_ids = ids;
    std::sort(sorted_ids.begin(), sorted_ids.end());
    if (std::adjacent_find(sorted_ids.begin(), sorted_ids.end()) != sorted_ids.end())
        throw DataError("duplicate request id in the request set");
    const int n = static_cast<int>(sorted_ids.size());
    exec.assign((std::size_t)n * max_batch, 0.0);
    deadline.assign((std::size_t)n * max_batch, 0.0);
    auto fill = [&](int i0, int i1) {
        for (int i = i0; i < i1; ++i) {
            const Request& r = require_predicted(w, sorted_ids[i], "anneal");
            const SloSpec& slo = w.class_of(r).slo;
            const int lo = *r.predicted_output_len;
            for (int b = 1; b <= max_batch; ++b) {
                const double e = predict_exec(c, b, r.input_len, lo);
                double d;
                if (slo.kind == SloKind::E2E) {
                    d = latest_start(*slo.e2e_ms, e);
                } else {
                    const double tp = predict_tpot(c, b, r.input_len, lo);
                    d = tp <= *slo.tpot_ms ? latest_start(*slo.ttft_ms, predict_prefill(c, b, r.input_len))
                                           : -std::numeric_limits<double>::infinity();
                }
                exec[(std::size_t)(b - 1) * n + i] = e;
                deadline[(std::size_t)(b - 1) * n + i] = d;
            }
        }
    };
    // large queues: the rows are independent, fill them on up to 4 threads
    const int parts = static_cast<int>(std::min<std::size_t>(4, (std::size_t)n * max_batch / 2048 + 1));
    TaskGroup rest;
    for (int k = 1; k < parts; ++k) rest.run([&fill, k, n, parts] { fill(n * k / parts, n * (k + 1) / parts); });
    fill(0, n / parts);
    rest.wait();
    // No batch can start later than the sum of every request's largest exec (a makespan is at
    // most the sum of its members'). A deadline at or beyond that bound is met in every schedule:
    // store +inf, which leaves every exact compare unchanged and lets the chain kernel count such
    // requests without walking them (loose classes such as "offline" would otherwise keep every
    // unit live). The margin covers the chain kernel's tick rounding (<= n half-ticks of elapsed).
    double horizon = 0.0;
    for (int i = 0; i < n; ++i) {
        double m = 0.0;
        for (int b = 1; b <= max_batch; ++b) m = std::max(m, exec[(std::size_t)(b - 1) * n + i]);
        horizon += m;
    }
    const double never_late = horizon * (1.0 + 1e-9) + 1.0;
    for (double& d : deadline)
        if (d >= never_late) d = std::numeric_limits<double>::infinity();
}

namespace {

// Deadline-first candidate over dense indices (tables [mb][n] from cost_tables): perm + batch sizes.
// Requests in ascending order of a due key (variant 0: latest start in a full batch, 1: latest
// start alone, 2: latest completion in a full batch); kept set in ascending (exec, index) order cut
// into batches of mb (a trailing partial batch uses its own size's tables); a request is kept when
// every kept request still starts by its latest start, otherwise the longest kept one (the last)
// is dropped (as in Moore-Hodgson; with batching this is a heuristic: the kept set need not stay
// feasible, and the exact evaluation decides). O(n * kept).
constexpr int kDeadlineVariants = 3;


// exec_order: every dense index in ascending (full-batch exec, index) order (shared by the variants)
void deadline_first_dense(int n, int mb, const std::vector<double>& exec, const std::vector<double>& deadline,
                          int variant, const std::vector<int>& exec_order, std::vector<int>& perm,
                          std::vector<int>& sizes) {
    const double* ef = exec.data() + (std::size_t)(mb - 1) * n;
    const double* df = deadline.data() + (std::size_t)(mb - 1) * n;
    std::vector<double> due(n);
    for (int i = 0; i < n; ++i)
        due[i] = variant == 1 ? deadline[i] : (variant == 2 ? df[i] + ef[i] : df[i]);
    const std::vector<int> order = order_by_key(due);  // ascending due, ties by index
    auto by_exec = [&](int a, int b) { return ef[a] != ef[b] ? ef[a] < ef[b] : a < b; };
    std::vector<int> kept;
    kept.reserve(n);
    // start[k] = start time of kept batch k, valid for k <= `valid` (it depends on batches < k only);
    // later entries are recomputed when a check first needs them (no eager re-time after a drop)
    std::vector<double> start((std::size_t)n + 2, 0.0);
    int valid = 0;
    // the kept requests' full-batch (exec, latest start), in kept order: full batches read them
    // contiguously (the trailing partial batch gathers its own size's tables)
    std::vector<double> ke, kd;
    ke.reserve(n), kd.reserve(n);
    auto batch = [&](int k, double& mk) {  // latest-start test of batch k at start[k]; mk = its makespan
        const int m = static_cast<int>(kept.size());
        const int b0 = k * mb, sz = std::min(mb, m - b0);
        const double s0 = start[k];
        bool ok = true;
        mk = 0.0;
        if (sz == mb) {
            for (int j = b0; j < b0 + sz; ++j) {
                ok = ok && s0 <= kd[j];
                mk = std::max(mk, ke[j]);
            }
            return ok;
        }
        const double* e = exec.data() + (std::size_t)(sz - 1) * n;
        const double* d = deadline.data() + (std::size_t)(sz - 1) * n;
        for (int j = b0; j < b0 + sz; ++j) {
            ok = ok && s0 <= d[kept[j]];
            mk = std::max(mk, e[kept[j]]);
        }
        return ok;
    };
    // every kept request of batches k0.. starts by its latest start (stops at the first that does not)
    auto check_from = [&](int k0) {
        double mk;
        for (; valid < k0; ++valid) {  // batches before k0: times only
            batch(valid, mk);
            start[valid + 1] = start[valid] + mk;
        }
        const int nb = (static_cast<int>(kept.size()) + mb - 1) / mb;
        for (int k = k0; k < nb; ++k) {
            if (!batch(k, mk)) {
                valid = k;
                return false;
            }
            start[k + 1] = start[k] + mk;
        }
        valid = nb;
        return true;
    };
    for (int i : order) {
        if (!(df[i] >= 0.0)) continue;  // cannot start in time even first (in a full batch)
        const auto it = std::lower_bound(kept.begin(), kept.end(), i, by_exec);
        const int p = static_cast<int>(it - kept.begin());
        kept.insert(it, i);
        ke.insert(ke.begin() + p, ef[i]), kd.insert(kd.begin() + p, df[i]);
        valid = std::min(valid, p / mb);  // batches from p / mb on changed
        if (!check_from(p / mb)) {  // Moore-Hodgson: drop the longest kept request
            kept.pop_back(), ke.pop_back(), kd.pop_back();
            valid = std::min(valid, std::min(p, static_cast<int>(kept.size())) / mb);
        }
    }
    std::vector<char> in(n, 0);
    perm.clear(), sizes.clear();
    for (int i : kept) perm.push_back(i), in[i] = 1;
    for (int b0 = 0; b0 < static_cast<int>(kept.size()); b0 += mb)
        sizes.push_back(std::min(mb, static_cast<int>(kept.size()) - b0));
    std::vector<int> rest;  // the dropped requests in (exec, index) order: a filter of exec_order
    rest.reserve(n - kept.size());
    for (int i : exec_order)
        if (!in[i]) rest.push_back(i);
    for (std::size_t b0 = 0; b0 < rest.size(); b0 += mb) {
        const int sz = static_cast<int>(std::min<std::size_t>(mb, rest.size() - b0));
        for (int j = 0; j < sz; ++j) perm.push_back(rest[b0 + j]);
        sizes.push_back(sz);
    }
}

Schedule schedule_of(const std::vector<int>& perm, const std::vector<int>& sizes, const std::vector<int>& sorted_ids) {
    Schedule s;
    int pos = 0;
    for (int sz : sizes) {
        Batch b;
        for (int j = 0; j < sz; ++j) b.push_back(sorted_ids[perm[pos++]]);
        s.batches.push_back(std::move(b));
    }
    return s;
}

// CostModel::score (P:src/priority_mapper.cpp:259-279) over the dense tables, the reference's
// operand order (== evaluate().g bit-for-bit, as K1).
double dense_score(int n, const std::vector<double>& exec, const std::vector<double>& deadline,
                   const std::vector<int>& perm, const std::vector<int>& sizes) {
    double elapsed = 0.0, total = 0.0;
    int met = 0, pos = 0;
    for (int sz : sizes) {
        const double* e = exec.data() + (std::size_t)(sz - 1) * n;
        const double* d = deadline.data() + (std::size_t)(sz - 1) * n;
        double makespan = 0.0;
        for (int j = 0; j < sz; ++j, ++pos) {
            const int i = perm[pos];
            const double e2e = elapsed + e[i];
            total += e2e;
            met += elapsed <= d[i];
            makespan = std::max(makespan, e[i]);
        }
        elapsed += makespan;
    }
    return total > 0.0 ? static_cast<double>(met) / total : 0.0;
}

// All variants (one host thread each), scored exactly; the best by G (lowest variant on ties).
// Returns its G (dense_score == evaluate().g bit-for-bit); the full evaluation is left to the
// caller, which needs it only when this candidate is the answer.
double best_deadline_first(int n, int mb, const std::vector<double>& exec, const std::vector<double>& deadline,
                           std::vector<int>& perm, std::vector<int>& sizes) {
    struct Cand {
        std::vector<int> perm, sizes;
        double g = 0.0;
    };
    std::vector<Cand> cand(kDeadlineVariants);
    const std::vector<int> exec_order =  // (full-batch exec, index): a strict total order
        order_by_key(std::vector<double>(exec.begin() + (std::size_t)(mb - 1) * n, exec.begin() + (std::size_t)mb * n));
    auto build = [&](int v) {
        deadline_first_dense(n, mb, exec, deadline, v, exec_order, cand[v].perm, cand[v].sizes);
        cand[v].g = dense_score(n, exec, deadline, cand[v].perm, cand[v].sizes);
    };
    TaskGroup others;
    for (int v = 1; v < kDeadlineVariants; ++v) others.run([&build, v] { build(v); });
    build(0);
    others.wait();
    int best = 0;
    for (int v = 1; v < kDeadlineVariants; ++v)
        if (cand[v].g > cand[best].g) best = v;
    perm = std::move(cand[best].perm), sizes = std::move(cand[best].sizes);
    return cand[best].g;
}

}  // namespace

namespace detail {
slo_ctx* acquire_ctx(int device) { return CtxPool::get().acquire(device).release(); }
void release_ctx(int device, slo_ctx* ctx) { CtxPool::get().release(device, CtxPtr(ctx)); }
int resolve_device(int requested) { return ::slosched::resolve_device(requested); }
void check(int rc) { engine_check(rc); }
}  // namespace detail

Schedule deadline_first_candidate(const Workload& w, const std::vector<int>& ids, const LatencyCoefficients& c,
                                  int max_batch) {
    if (max_batch < 1) throw DataError("deadline_first_candidate: max_batch must be >= 1");
    std::vector<double> exec, deadline;
    cost_tables(w, ids, c, max_batch, exec, deadline);
    std::vector<int> sorted_ids = ids, perm, sizes;
    std::sort(sorted_ids.begin(), sorted_ids.end());
    best_deadline_first(static_cast<int>(sorted_ids.size()), max_batch, exec, deadline, perm, sizes);
    return schedule_of(perm, sizes, sorted_ids);
}

AnnealResult anneal(const Workload& w, const std::vector<int>& ids, const LatencyCoefficients& c,
                    const AnnealConfig& cfg, int max_batch) {
    cfg.validate();
    if (max_batch < 1) throw DataError("anneal: max_batch must be >= 1");
    AnnealResult res;
    // The cost tables (and, for the chains, the deadline-first candidate) are built on a second
    // host thread while this one builds and scores the reference's two candidates.
    const int n = static_cast<int>(ids.size());
    std::vector<int> sorted_ids = ids;
    std::sort(sorted_ids.begin(), sorted_ids.end());
    std::vector<double> exec, deadline;
    std::vector<int> dl_perm, dl_sizes;
    std::optional<double> g_dl;  // G of the deadline-first candidate (evaluated in full only if returned)
    const bool want_dl = cfg.engine.mode == SearchMode::Chains && cfg.engine.deadline_start;
    // the engine (context, rank context or device group) gets the tables on the same thread, as
    // soon as they exist
    EngineHandle eng(cfg.engine);
    // one rank of a multi-process job that fails before its exchange still joins it (EngineHandle::
    // abandon), so its peers are not left waiting in the collective
    struct AbandonOnThrow {
        EngineHandle& e;
        int n;
        const int pending = std::uncaught_exceptions();
        ~AbandonOnThrow() {
            if (std::uncaught_exceptions() > pending) e.abandon(n);
        }
    } abandon_on_throw{eng, n};
    TaskGroup tables;
    tables.run([&] {
        cost_tables(w, ids, c, max_batch, exec, deadline);
        // the upload (context, tables, device-side tick tables) overlaps the deadline-first start
        TaskGroup upload;
        upload.run([&] {
            if (n >= 1 && n <= SLO_MAX_N && max_batch <= SLO_MAX_MB)
                eng.problem_set(n, max_batch, exec.data(), deadline.data());
        });
        if (want_dl) g_dl = best_deadline_first(n, max_batch, exec, deadline, dl_perm, dl_sizes);
        upload.wait();
    });
    auto [sorted_s, input_s] = initial_candidates(w, ids, c, max_batch);
    EvaluatedSchedule ev_sorted = evaluate(sorted_s, c, w);
    res.stats.g_sorted_start = ev_sorted.g;
    if (ev_sorted.n == static_cast<int>(ev_sorted.per_request.size())) {  // shortcut, :350-354
        res.stats.shortcut = true;
        res.best = std::move(ev_sorted);
        return res;
    }
    EvaluatedSchedule ev_input = evaluate(input_s, c, w);
    res.stats.g_input_start = ev_input.g;

    // CostModel tables over dense indices (rank of the sorted id), :205-231, with the SLO
    // test folded into a per-(batch size, request) deadline
    if (n > SLO_MAX_N) throw CapacityError("anneal: " + std::to_string(n) + " requests exceed the engine limit of 4096");
    if (max_batch > SLO_MAX_MB) throw CapacityError("anneal: max_batch above the engine limit of 16");
    tables.wait();
    const bool use_sorted = ev_sorted.g >= ev_input.g;
    const Schedule& start = use_sorted ? sorted_s : input_s;
    std::vector<int> start_perm, start_sizes;
    start_perm.reserve(n);
    for (const auto& b : start.batches) {
        start_sizes.push_back(static_cast<int>(b.size()));
        for (int id : b)
            start_perm.push_back(static_cast<int>(std::lower_bound(sorted_ids.begin(), sorted_ids.end(), id) - sorted_ids.begin()));
    }
    // score(start) == evaluate(start).g bit-for-bit (same operand order), :362-370
    double f = use_sorted ? ev_sorted.g : ev_input.g;
    // engine extension: the chains start from the deadline-first candidate when it scores higher
    if (g_dl) {
        res.stats.g_deadline_start = *g_dl;
        if (*g_dl > f) f = *g_dl, start_perm = dl_perm, start_sizes = dl_sizes;
    }
    const double scale = cfg.objective_scale ? *cfg.objective_scale : (f > 0.0 ? cfg.t0 / f : cfg.t0);
    res.stats.objective_scale_used = scale;

    const EngineOptions& eo = cfg.engine;
    slo_chain_params prm{};
    prm.t0 = cfg.t0;
    prm.t_thres = cfg.t_thres;
    prm.iter = cfg.iter;
    prm.tau = cfg.tau;
    prm.seed = cfg.seed;
    prm.objective_scale = scale;
    prm.rng_mode = eo.mode == SearchMode::Replay ? SLO_RNG_XOSHIRO_REPLAY : SLO_RNG_PHILOX;
    prm.chains = eo.mode == SearchMode::Replay ? 1 : eo.chains;
    prm.chain_begin = 0, prm.chain_end = 1;
    if (eo.mode != SearchMode::Replay) eng.slice(eo, eo.chains, &prm.chain_begin, &prm.chain_end);
    prm.budget_ns = static_cast<int64_t>(eo.budget_ms * 1e6);
    prm.n_scale_mult = static_cast<int32_t>(eo.scale_ladder.size());
    prm.scale_mult = eo.scale_ladder.empty() ? nullptr : eo.scale_ladder.data();
    prm.max_blocks = eo.max_blocks;

    std::vector<int> best_perm(n), best_sizes(n);
    int best_nb = 0;
    slo_chain_result cr{};
    if (!eng.ready()) throw EngineError("B200 engine: no context for the problem");
    eng.anneal(prm, start_perm, start_sizes, best_perm, best_sizes, &best_nb, &cr);

    res.stats.proposals = cr.proposals;
    res.stats.accepted = cr.accepted;
    res.stats.chains_run = cr.chains_run;
    res.stats.levels_run = cr.levels_run;
    res.stats.best_chain = cr.chain;
    res.stats.engine_g = cr.g;
    res.stats.engine_t = cr.t;
    res.stats.kernel_ms = cr.kernel_ms;
    res.stats.exchange_ms = cr.exchange_ms;
    res.stats.devices = cr.nranks;

    Schedule best;
    int pos = 0;
    for (int k = 0; k < best_nb; ++k) {
        Batch b;
        for (int j = 0; j < best_sizes[k]; ++j) b.push_back(sorted_ids[best_perm[pos++]]);
        best.batches.push_back(std::move(b));
    }
    // final evaluation through the objective; both starts stay a floor, :404-410
    EvaluatedSchedule ev_best = evaluate_owned(std::move(best), c, w);
    const double floor_g = std::max(ev_sorted.g, ev_input.g);
    // Replay mode keeps the reference's ">=" floor (:406-410) bit for bit. In Chains mode the chains'
    // winner replaces the starts only when it strictly improves the reference's objective -- the
    // reference's own best-so-far rule (`f > best_f`, :392-400): on an exact tie the start stands,
    // as it would in the reference's walk (an equal-G plan found on the tick grid is not preferred)
    const bool strict = eo.mode == SearchMode::Chains;
    const bool beats = strict ? ev_best.g > floor_g && (!g_dl || ev_best.g > *g_dl)
                              : ev_best.g >= floor_g && (!g_dl || ev_best.g >= *g_dl);
    if (beats) res.best = std::move(ev_best);
    else if (g_dl && *g_dl > floor_g) res.best = evaluate(schedule_of(dl_perm, dl_sizes, sorted_ids), c, w);
    else res.best = use_sorted ? std::move(ev_sorted) : std::move(ev_input);
    return res;
}

ExhaustiveResult exhaustive(const Workload& w, const std::vector<int>& ids, const LatencyCoefficients& c,
                            int max_batch, int n_cap) {
    const int n = static_cast<int>(ids.size());
    if (n > n_cap)
        throw CapacityError("exhaustive: " + std::to_string(n) + " requests exceed cap of " + std::to_string(n_cap) +
                            " (search space is O(N! * 2^N))");
    if (max_batch < 1) throw DataError("exhaustive: max_batch must be >= 1");
    ExhaustiveResult res;
    if (n == 0) {  // the single (empty) schedule
        res.best = evaluate(Schedule{}, c, w);
        res.schedules_evaluated = 1;
        return res;
    }
    std::vector<int> sorted_ids = ids;
    std::sort(sorted_ids.begin(), sorted_ids.end());
    std::vector<double> exec, deadline;
    const int mb = std::min(max_batch, n);  // compositions never use parts above n
    cost_tables(w, ids, c, mb, exec, deadline);
    const int device = resolve_device(-1);
    CtxPtr ctx = CtxPool::get().acquire(device);
    std::vector<int> perm(n), sizes(n);
    int nb = 0;
    double g = 0.0, t = 0.0;
    std::uint64_t evaluated = 0;
    engine_check(slo_problem_set(ctx.get(), n, mb, exec.data(), deadline.data()));
    engine_check(slo_exhaustive(ctx.get(), n_cap, perm.data(), sizes.data(), &nb, &g, &t, &evaluated));
    CtxPool::get().release(device, std::move(ctx));
    Schedule best;
    for (int k = 0, pos = 0; k < nb; ++k) {
        Batch b;
        for (int j = 0; j < sizes[k]; ++j) b.push_back(sorted_ids[perm[pos++]]);
        best.batches.push_back(std::move(b));
    }
    res.best = evaluate(best, c, w);
    res.schedules_evaluated = evaluated;
    return res;
}

// ================================================================ scheduler (P:src/scheduler.cpp)
long long token_capacity(std::uint64_t remaining, double mu, double sigma) {
    if (!(sigma > 0.0)) throw std::invalid_argument("token_capacity: sigma must be > 0");
    if (!(mu > 0.0) || mu > 1.0) throw std::invalid_argument("token_capacity: mu must be in (0,1]");
    return static_cast<long long>(std::floor(static_cast<double>(remaining) * mu / sigma));
}

AssignmentResult assign_instances(const Workload& w, const std::vector<InstanceState>& instances,
                                  const LatencyCoefficients& c) {
    if (instances.empty()) throw DataError("assign_instances: need at least one instance");
    for (const auto& inst : instances) inst.validate();
    std::vector<double> key;
    std::vector<int> rid;
    key.reserve(w.requests.size()), rid.reserve(w.requests.size());
    for (const auto& r : w.requests) {
        if (!r.predicted_output_len) throw DataError("assign_instances: request missing predicted length");
        key.push_back(predict_exec(c, 1, r.input_len, *r.predicted_output_len)), rid.push_back(r.id);
    }
    std::vector<int> order;  // ids in ascending (exec alone, id)
    order.reserve(rid.size());
    for (int i : order_by_key(key, &rid)) order.push_back(rid[i]);
    const std::size_t k = instances.size();
    std::vector<double> remaining(k);
    for (std::size_t i = 0; i < k; ++i) remaining[i] = static_cast<double>(instances[i].remaining_mem);
    auto roomiest = [&]() {
        std::size_t best = 0;
        long long best_cap = -1;
        for (std::size_t i = 0; i < k; ++i) {
            const long long cap = token_capacity(static_cast<std::uint64_t>(remaining[i]), instances[i].mem_utility,
                                                 instances[i].bytes_per_token);
            if (i == 0 || cap > best_cap) best = i, best_cap = cap;
        }
        return std::pair<std::size_t, long long>{best, best_cap};
    };
    AssignmentResult res;
    res.per_instance.resize(k);
    for (int id : order) {
        const Request& r = *w.find_request(id);
        const long long need = r.input_len + *r.predicted_output_len;
        auto [inst, cap] = roomiest();
        if (cap < need) {  // new epoch: memory resets to totals
            for (std::size_t i = 0; i < k; ++i) remaining[i] = static_cast<double>(instances[i].total_mem);
            res.epochs++;
            std::tie(inst, cap) = roomiest();
            if (cap < need) throw CapacityError("request " + std::to_string(id) + " cannot fit any instance");
        }
        res.per_instance[inst].push_back(id);
        remaining[inst] -= static_cast<double>(need) * instances[inst].bytes_per_token / instances[inst].mem_utility;
        if (remaining[inst] < 0.0) remaining[inst] = 0.0;
    }
    return res;
}

std::optional<Batch> dispatch(InstanceQueue& q, bool ready) {
    if (!ready || q.pending.empty()) return std::nullopt;
    Batch next = std::move(q.pending.front());
    q.pending.pop_front();
    return next;
}

ScheduleAllResult schedule_all(const Workload& w, const std::vector<InstanceState>& instances,
                               const LatencyCoefficients& c, const AnnealConfig& cfg, Policy policy,
                               int exhaustive_cap) {
    if (policy == Policy::FCFS) throw std::invalid_argument("schedule_all: FCFS is a simulator baseline, not a mapper policy");
    const auto t_start = std::chrono::steady_clock::now();
    ScheduleAllResult res;
    res.assignment = assign_instances(w, instances, c);
    const std::size_t k = instances.size();
    res.per_instance.resize(k);
    res.stats.resize(k);
    res.queues.resize(k);
    // Per-instance anneals are independent (disjoint request sets, own derived seeds; the
    // reference runs them one after another, P:src/scheduler.cpp:109-123, SPEC:377-378 allows
    // concurrency). In Chains mode each instance gets its own host thread, engine context and
    // stream, and a 1/k share of the SMs, so the k launches run side by side on the GPU.
    std::vector<AnnealConfig> per(k, cfg);
    const bool concurrent = k > 1 && cfg.engine.mode == SearchMode::Chains && cfg.engine.concurrent_instances;
    const std::vector<int>& devs = cfg.engine.devices;
    if (concurrent && devs.size() > 1) {
        // instances are placed one per GPU (round robin); instances sharing a GPU split its SMs
        std::map<int, int> on_dev;
        for (std::size_t i = 0; i < k; ++i) ++on_dev[devs[i % devs.size()]];
        for (std::size_t i = 0; i < k; ++i) {
            const int d = devs[i % devs.size()];
            per[i].engine.devices = {d};
            if (cfg.engine.max_blocks <= 0 && on_dev[d] > 1) {
                CtxPtr ctx = CtxPool::get().acquire(d);
                const int sms = slo_ctx_sm_count(ctx.get());
                CtxPool::get().release(d, std::move(ctx));
                per[i].engine.max_blocks = std::max(1, sms / on_dev[d]);
            }
        }
    } else if (concurrent && cfg.engine.max_blocks <= 0) {
        const int device = devs.size() == 1 ? devs[0] : resolve_device(cfg.engine.device);
        CtxPtr ctx = CtxPool::get().acquire(device);
        const int sms = slo_ctx_sm_count(ctx.get());
        CtxPool::get().release(device, std::move(ctx));
        for (auto& p : per) p.engine.max_blocks = std::max(1, sms / static_cast<int>(k));
    }
    for (std::size_t i = 0; i < k; ++i) per[i].seed = Rng::derive(cfg.seed, static_cast<std::uint64_t>(instances[i].id));
    std::vector<AnnealResult> out(k);
    auto run_one = [&](std::size_t i) {
        if (policy == Policy::EXHAUSTIVE)  // P:src/scheduler.cpp:118-120: no stats for the oracle
            out[i].best = exhaustive(w, res.assignment.per_instance[i], c, instances[i].max_batch_size,
                                     exhaustive_cap).best;
        else
            out[i] = anneal(w, res.assignment.per_instance[i], c, per[i], instances[i].max_batch_size);
    };
    if (concurrent) {
        std::vector<std::exception_ptr> errs(k);
        std::vector<std::thread> pool;
        for (std::size_t i = 0; i < k; ++i)
            pool.emplace_back([&, i] {
                try {
                    run_one(i);
                } catch (...) {
                    errs[i] = std::current_exception();
                }
            });
        for (auto& t : pool) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    } else {
        for (std::size_t i = 0; i < k; ++i) run_one(i);
    }
    for (std::size_t i = 0; i < k; ++i) {
        res.per_instance[i] = std::move(out[i].best);
        res.stats[i] = out[i].stats;
        for (const auto& b : res.per_instance[i].schedule.batches) res.queues[i].pending.push_back(b);
    }
    res.overhead_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    return res;
}

// ================================================================ synthetic inputs
// (P:src/workload.cpp:138-183, P:src/output_estimator.cpp:361-415)
std::pair<TaskClass, TaskClass> default_slo_classes() {
    TaskClass code{0, "code", SloSpec::e2e(30000.0), {}};
    TaskClass chat{1, "chat", SloSpec::ttft_tpot(10000.0, 50.0), {}};
    return {code, chat};
}

std::pair<TaskClass, TaskClass> default_synth_classes(const LengthDists& d) {
    auto [code, chat] = default_slo_classes();
    code.output_prior = GaussianPrior{d.code_output_mean, d.code_output_std};
    chat.output_prior = GaussianPrior{d.chat_output_mean, d.chat_output_std};
    return {code, chat};
}

namespace {
int clamp_tokens(double v) { return std::clamp(static_cast<int>(std::llround(v)), 1, kValidatedMaxLen); }
int at_least_one(double v) { return std::max(1, static_cast<int>(std::llround(v))); }
}  // namespace

std::vector<Request> generate_mixed(int n, std::uint64_t seed, const TaskClass& code_class, const TaskClass& chat_class,
                                    const LengthDists& d) {
    Rng rng(seed);
    const int n_code = (n + 1) / 2;
    std::vector<Request> out;
    out.reserve(static_cast<std::size_t>(std::max(n, 0)));
    for (int i = 0; i < n; ++i) {
        const bool code = i < n_code;
        Request r;
        r.task_class_id = code ? code_class.id : chat_class.id;
        const double median = code ? d.code_input_median : d.chat_input_median;
        const double sigma = code ? d.code_input_sigma : d.chat_input_sigma;
        r.input_len = clamp_tokens(median * std::exp(sigma * rng.normal()));
        r.true_output_len = clamp_tokens(rng.normal(code ? d.code_output_mean : d.chat_output_mean,
                                                    code ? d.code_output_std : d.chat_output_std));
        out.push_back(r);
    }
    rng.shuffle(out);
    for (int i = 0; i < n; ++i) out[i].id = i;
    return out;
}

void assign_predicted_lengths_from_priors(std::vector<Request>& reqs, const std::vector<TaskClass>& classes, Rng& rng) {
    for (auto& r : reqs) {
        if (r.predicted_output_len) continue;
        const TaskClass* cls = nullptr;
        for (const auto& c : classes)
            if (c.id == r.task_class_id) cls = &c;
        if (!cls) throw DataError("estimator: unknown task_class_id " + std::to_string(r.task_class_id));
        if (auto g = std::get_if<GaussianPrior>(&cls->output_prior)) r.predicted_output_len = at_least_one(rng.normal(g->mean_tokens, g->std_tokens));
        else if (auto rp = std::get_if<RangePrior>(&cls->output_prior)) r.predicted_output_len = static_cast<int>(rng.uniform_int(rp->low, rp->high));
        else r.predicted_output_len = 256;
    }
}

}  // namespace slosched
