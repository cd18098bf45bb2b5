// Online rolling-window rescheduling (BASELINE configs[4]) in the library.
//
// The reference schedules in synchronous waves and has no online mode; this driver is
// built on the library's entry points: arrivals join the least-loaded instance, every window each
// instance's queue is re-planned (GPU chains under the per-window budget, or FCFS) with
// slack-adjusted SLOs, and the plans run on the library's replay (realize_batches: the reference
// simulator's ground truth, P:src/simulator.cpp:17-74, noise 0) until the next window boundary.
// paper_2504_14966_b200/online.py is its Python face (and keeps a Python loop for caller-supplied
// planners); both produce identical results on the same stream (tests/test_online.py).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_set>

#include "internal.hpp"
#include "slosched_b200.hpp"
#include "slosched_gpu.h"

namespace slosched {

namespace {

// n_instances workers kept for the whole run: each window, worker k plans instance k when it is
// active (the planning of a window runs concurrently, one engine context per instance)
class WindowWorkers {
public:
    explicit WindowWorkers(int k) : err_(k) {
        for (int i = 0; i < k; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~WindowWorkers() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // run job(k) for every k with active[k], wait for all; rethrows the first failure
    void run(const std::vector<char>& active, const std::function<void(int)>& job) {
        {
            std::lock_guard<std::mutex> g(mu_);
            active_ = &active, job_ = &job;
            pending_ = static_cast<int>(th_.size());
            ++gen_;
        }
        cv_.notify_all();
        std::unique_lock<std::mutex> l(mu_);
        done_cv_.wait(l, [this] { return pending_ == 0; });
        for (auto& e : err_)
            if (e) {
                std::exception_ptr x = e;
                for (auto& e2 : err_) e2 = nullptr;
                std::rethrow_exception(x);
            }
    }

private:
    void loop(int i) {
        unsigned long long seen = 0;
        while (true) {
            const std::vector<char>* act;
            const std::function<void(int)>* job;
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_, act = active_, job = job_;
            }
            if ((*act)[i]) {
                try {
                    (*job)(i);
                } catch (...) {
                    err_[i] = std::current_exception();
                }
            }
            std::lock_guard<std::mutex> g(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::vector<std::exception_ptr> err_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::vector<char>* active_ = nullptr;
    const std::function<void(int)>* job_ = nullptr;
    unsigned long long gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};

constexpr double kImpossibleMs = 1e-9;  // an SLO whose slack is gone: positive (valid) but unreachable

std::pair<TaskClass, TaskClass> stream_classes() {
    return {TaskClass{0, "code", SloSpec::e2e(30000.0), {}}, TaskClass{1, "chat", SloSpec::ttft_tpot(10000.0, 50.0), {}}};
}

}  // namespace

OnlineResult run_online(const OnlineStream& st, const LatencyCoefficients& c, const OnlineConfig& cfg) {
    const int n = static_cast<int>(st.arrival_ms.size());
    const int k = cfg.n_instances;
    if (k < 1) throw DataError("run_online: need at least one instance");
    if (!(cfg.window_ms > 0.0)) throw DataError("run_online: window_ms must be > 0");
    if (cfg.max_batch < 1) throw DataError("run_online: max_batch must be >= 1");
    if (!(cfg.dispatch_gap_ms >= 0.0)) throw DataError("run_online: dispatch_gap_ms must be >= 0");
    if (cfg.policy != Policy::SA && cfg.policy != Policy::FCFS)
        throw std::invalid_argument("run_online: policy must be SA or FCFS");
    if (st.cls.size() != (size_t)n || st.input_len.size() != (size_t)n || st.true_out.size() != (size_t)n ||
        st.pred_out.size() != (size_t)n)
        throw DataError("run_online: stream arrays differ in length");
    for (int i = 0; i < n; ++i)
        if (!std::isfinite(st.arrival_ms[i]) || st.arrival_ms[i] < 0.0 || (i > 0 && st.arrival_ms[i] < st.arrival_ms[i - 1]))
            throw DataError("run_online: arrival times must be finite, >= 0 and nondecreasing");
    const std::vector<int> devs = cfg.devices.empty() ? std::vector<int>{detail::resolve_device(-1)} : cfg.devices;
    std::vector<int> dev_of(k), share(k, 0);
    for (int i = 0; i < k; ++i) dev_of[i] = devs[i % devs.size()];
    if (cfg.policy == Policy::SA)
        for (int d : devs) {
            if (std::find(dev_of.begin(), dev_of.end(), d) == dev_of.end()) continue;
            slo_ctx* ctx = detail::acquire_ctx(d);
            const int sms = slo_ctx_sm_count(ctx);
            detail::release_ctx(d, ctx);
            const int on = static_cast<int>(std::count(dev_of.begin(), dev_of.end(), d));
            for (int i = 0; i < k; ++i)
                if (dev_of[i] == d) share[i] = std::max(1, sms / on);
        }
    auto [code, chat] = stream_classes();
    auto work1 = [&](int i) {  // predicted work at batch size 1: the assignment key
        return predict_prefill(c, 1, st.input_len[i]) + predict_decode_total(c, 1, st.input_len[i], st.pred_out[i]);
    };

    std::vector<std::vector<int>> queue(k);
    std::vector<double> busy(k, 0.0), load(k, 0.0);
    OnlineResult res;
    int next_arrival = 0, done = 0;
    double t_win = 0.0, host_ms = 1.5;
    std::unique_ptr<WindowWorkers> workers;
    if (cfg.policy == Policy::SA) workers = std::make_unique<WindowWorkers>(k);
    std::vector<std::vector<Batch>> plans(k);
    std::vector<double> kernel_ms(k, 0.0);
    std::vector<std::uint64_t> props(k, 0);
    while (done < n && (cfg.max_windows < 0 || res.windows < cfg.max_windows)) {
        const double t_next = t_win + cfg.window_ms;
        // arrivals up to this window start join the least-loaded instance
        while (next_arrival < n && st.arrival_ms[next_arrival] <= t_win) {
            const int i = next_arrival;
            int best = 0;
            double best_key = 0.0;
            for (int j = 0; j < k; ++j) {
                const double key = std::max(busy[j], t_win) + load[j];
                if (j == 0 || key < best_key) best = j, best_key = key;
            }
            queue[best].push_back(i);
            load[best] += work1(i);
            ++next_arrival;
        }
        bool any = false;
        for (const auto& q : queue) any = any || !q.empty();
        if (!any && next_arrival < n) {  // idle: jump to the first window holding an arrival
            t_win = std::max(t_win, std::ceil(st.arrival_ms[next_arrival] / cfg.window_ms) * cfg.window_ms);
            continue;
        }
        ++res.windows;
        std::vector<char> active(k, 0);
        for (int j = 0; j < k; ++j) active[j] = !queue[j].empty();
        const auto t0 = std::chrono::steady_clock::now();
        if (cfg.policy == Policy::SA) {
            const double kernel_budget = std::max(0.5, cfg.budget_ms - host_ms - 0.3);
            const int wins = res.windows;
            workers->run(active, [&](int j) {
                const std::vector<int>& ids = queue[j];
                const double start = std::max(busy[j], t_win);
                // each request in a class of its own: its SLO less the time it has already waited
                std::vector<TaskClass> classes;
                std::vector<Request> reqs;
                classes.reserve(ids.size()), reqs.reserve(ids.size());
                for (std::size_t q = 0; q < ids.size(); ++q) {
                    const int i = ids[q];
                    const double waited = start - st.arrival_ms[i];
                    TaskClass tc;
                    tc.id = static_cast<int>(q);
                    tc.slo = st.cls[i] == 0 ? SloSpec::e2e(std::max(30000.0 - waited, kImpossibleMs))
                                            : SloSpec::ttft_tpot(std::max(10000.0 - waited, kImpossibleMs), 50.0);
                    classes.push_back(std::move(tc));
                    Request r;
                    r.id = i, r.task_class_id = static_cast<int>(q), r.input_len = st.input_len[i];
                    r.true_output_len = st.true_out[i], r.predicted_output_len = st.pred_out[i];
                    r.arrival_time_ms = st.arrival_ms[i];
                    reqs.push_back(r);
                }
                const Workload w = validate_workload(std::move(reqs), std::move(classes));
                AnnealConfig a;
                a.t0 = cfg.t0, a.tau = cfg.tau, a.iter = cfg.iter;
                a.seed = cfg.seed * 1000003ull + static_cast<std::uint64_t>(wins) * 131ull + static_cast<std::uint64_t>(j);
                a.engine.chains = std::min(cfg.chains, std::max(cfg.chains_min,
                                                                cfg.chains_per_request * static_cast<int>(ids.size())));
                a.engine.budget_ms = kernel_budget;
                a.engine.scale_ladder = cfg.scale_ladder;
                a.engine.max_blocks = share[j];
                a.engine.devices = {dev_of[j]};
                a.engine.deadline_start = cfg.deadline_start;
                const AnnealResult r = anneal(w, ids, c, a, cfg.max_batch);
                plans[j] = r.best.schedule.batches;
                kernel_ms[j] = r.stats.kernel_ms;
                props[j] = r.stats.proposals;
            });
        } else {
            for (int j = 0; j < k; ++j) {
                if (!active[j]) continue;
                std::vector<std::pair<double, int>> order;
                for (int i : queue[j]) order.emplace_back(st.arrival_ms[i], i);
                std::sort(order.begin(), order.end());
                plans[j].clear();
                for (std::size_t q = 0; q < order.size(); q += cfg.max_batch) {
                    Batch b;
                    for (std::size_t z = q; z < std::min(order.size(), q + cfg.max_batch); ++z) b.push_back(order[z].second);
                    plans[j].push_back(std::move(b));
                }
                kernel_ms[j] = 0.0, props[j] = 0;
            }
        }
        const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        res.overhead_ms.push_back(wall);
        if (cfg.policy == Policy::SA) {  // host share of this window: wall less the longest kernel
            double kmax = 0.0;
            for (int j = 0; j < k; ++j)
                if (active[j]) kmax = std::max(kmax, kernel_ms[j]);
            const double now = wall - kmax;
            host_ms = res.windows <= 1 ? now : std::max(0.9 * host_ms + 0.1 * now, now * 0.5);
        }
        // execute each plan until the next window boundary (the library's replay)
        for (int j = 0; j < k; ++j) {
            if (!active[j]) continue;
            ++res.decisions;
            res.proposals += props[j];
            std::vector<Request> reqs;
            for (const Batch& b : plans[j])
                for (int i : b) {
                    Request r;
                    r.id = i, r.task_class_id = st.cls[i], r.input_len = st.input_len[i];
                    r.true_output_len = st.true_out[i], r.predicted_output_len = st.pred_out[i];
                    r.arrival_time_ms = st.arrival_ms[i];
                    reqs.push_back(r);
                }
            const Workload w = validate_workload(std::move(reqs), {code, chat});
            Rng rng(0);
            std::vector<RequestMetrics> recs;
            const ReplayResult rr = realize_batches(plans[j], w, c, std::max(busy[j], t_win), cfg.dispatch_gap_ms,
                                                    cfg.dispatch_gap_ms, t_next, 0.0, rng, recs, true);
            double lat = 0.0;
            for (const auto& m : recs) {
                res.n_met += m.slo_met ? 1 : 0;
                lat += m.e2e_ms;
            }
            res.total_latency_ms += lat;
            busy[j] = rr.clock;
            if (rr.batches_started > 0) {
                std::unordered_set<int> started;
                for (int b = 0; b < rr.batches_started; ++b)
                    for (int i : plans[j][b]) started.insert(i), load[j] -= work1(i);
                std::vector<int> keep;
                for (int i : queue[j])
                    if (!started.count(i)) keep.push_back(i);
                queue[j].swap(keep);
                done += static_cast<int>(started.size());
            }
        }
        t_win = t_next;
    }
    res.n = done;
    return res;
}

}  // namespace slosched
