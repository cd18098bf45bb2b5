// Evaluation harness around the GPU scheduler: the output-length estimator, the realized-attainment
// replay (synthetic backend), the FCFS baseline and the compare / sweep / perturb drivers.
//
// Reference behaviour this follows (P: = /root/reference/proj/):
//   estimator   P:src/output_estimator.cpp:10-78   Welford update, fitted -> prior -> 256 prediction
//   replay      P:src/simulator.cpp:17-74          latency model over TRUE lengths, one noise factor
//                                                  per request, batches back to back + dispatch gap
//   FCFS        P:src/simulator.cpp:76-123         arrival order, earliest-ready instance
//   compare     P:src/simulator.cpp:148-220        per (policy, seed) rows + medians
//   sweep       P:tools/slosched.cpp:335-378       G of schedule_all over a (t0, iter) grid
//   perturb     P:tools/slosched.cpp:382-448       realized G under perturbed predictor coefficients
// Every number a caller compares with the reference is produced in the reference's arithmetic
// (operand order, draw order), so the replay and the estimator are bit-identical to it.
//
// B200 side: the annealing inside compare / sweep / perturb is schedule_all on the GPU; sweep and
// perturb launch all their cells at once (one host thread per cell, each annealing on its own
// engine context with a share of the SMs) and the sweep scores every cell's per-instance
// schedules with one launch of the bit-exact evaluator (evaluate_batch, K1) per instance.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <exception>
#include <future>
#include <limits>
#include <map>
#include <queue>
#include <stdexcept>
#include <thread>

#include "internal.hpp"
#include "slosched_b200.hpp"
#include "slosched_gpu.h"

namespace slosched {

// ================================================================ estimator
double LengthModel::sample_variance() const { return count >= 2 ? m2 / static_cast<double>(count - 1) : 0.0; }
double LengthModel::sample_std() const { return std::sqrt(sample_variance()); }

void observe(LengthModel& m, int actual_len) {
    if (actual_len < 1) throw DataError("observe: non-positive length");
    // Welford: the running mean moves by delta / count, m2 by delta times the new deviation
    const double x = static_cast<double>(actual_len);
    ++m.count;
    const double delta = x - m.mean;
    m.mean += delta / static_cast<double>(m.count);
    m.m2 += delta * (x - m.mean);
}

namespace {
int round_at_least_one(double v) { return std::max(1, static_cast<int>(std::llround(v))); }
}  // namespace

int predict_len(const LengthModel& m, Rng& rng) {
    if (m.count >= 2) return round_at_least_one(rng.normal(m.mean, m.sample_std()));
    if (const auto* g = std::get_if<GaussianPrior>(&m.prior)) return round_at_least_one(rng.normal(g->mean_tokens, g->std_tokens));
    if (const auto* r = std::get_if<RangePrior>(&m.prior)) return static_cast<int>(rng.uniform_int(r->low, r->high));
    return kDefaultOutputLen;
}

int simulate_predictor_error(int true_len, double error_pct, Rng& rng) {
    if (error_pct < 0.0) throw std::invalid_argument("simulate_predictor_error: error_pct must be >= 0");
    if (error_pct == 0.0) return std::max(1, true_len);
    return round_at_least_one(static_cast<double>(true_len) * (1.0 + rng.uniform(-error_pct, error_pct)));
}

Estimator::Estimator(const std::vector<TaskClass>& classes) {
    models_.reserve(classes.size());
    for (const auto& c : classes) {
        LengthModel m;
        m.task_class_id = c.id;
        m.prior = c.output_prior;
        models_.push_back(std::move(m));
    }
}

LengthModel& Estimator::model_for(int task_class_id) {
    auto it = std::find_if(models_.begin(), models_.end(), [&](const LengthModel& m) { return m.task_class_id == task_class_id; });
    if (it == models_.end()) throw DataError("estimator: unknown task_class_id " + std::to_string(task_class_id));
    return *it;
}

void Estimator::observe_output(int task_class_id, int actual_len) { observe(model_for(task_class_id), actual_len); }
int Estimator::predict(int task_class_id, Rng& rng) { return predict_len(model_for(task_class_id), rng); }

void assign_predicted_lengths(std::vector<Request>& requests, Estimator& est, Rng& rng) {
    for (auto& r : requests)
        if (!r.predicted_output_len) r.predicted_output_len = est.predict(r.task_class_id, rng);
}

// ================================================================ replay
MetricsReport MetricsReport::from_records(std::vector<RequestMetrics> records, double overhead_ms) {
    MetricsReport rep;
    rep.per_request = std::move(records);
    rep.scheduling_overhead_ms = overhead_ms;
    for (const auto& r : rep.per_request) {  // record order: the sum is the reference's
        rep.n_met += r.slo_met ? 1 : 0;
        rep.total_latency_ms += r.e2e_ms;
    }
    const double cnt = static_cast<double>(rep.per_request.size());
    if (!rep.per_request.empty()) {
        rep.slo_attainment = static_cast<double>(rep.n_met) / cnt;
        rep.avg_latency_ms = rep.total_latency_ms / cnt;
        rep.g = rep.total_latency_ms > 0.0 ? static_cast<double>(rep.n_met) / rep.total_latency_ms : 0.0;
    }
    return rep;
}

ReplayResult realize_batches(const std::vector<Batch>& batches, const Workload& w, const LatencyCoefficients& c,
                             double clock0, double first_gap, double gap, double until, double noise_pct, Rng& rng,
                             std::vector<RequestMetrics>& records, bool from_arrival) {
    ReplayResult res;
    double clock = clock0;
    for (const Batch& batch : batches) {
        if (clock >= until) break;
        const double start = clock + (res.batches_started == 0 ? first_gap : gap);
        const int b = static_cast<int>(batch.size());
        double makespan = 0.0;
        for (int id : batch) {
            const Request* r = w.find_request(id);
            if (!r) throw DataError("simulator: schedule references unknown request " + std::to_string(id));
            const int lo = r->true_output_len;
            // one factor per request (drawn in member order), shared by prefill and decode
            const double f = noise_pct > 0.0 ? 1.0 + rng.uniform(-noise_pct, noise_pct) : 1.0;
            const double prefill = predict_prefill(c, b, r->input_len) * f;
            const double exec = predict_exec(c, b, r->input_len, lo) * f;
            RequestMetrics m;
            m.request_id = id;
            m.wait_ms = from_arrival ? start - r->arrival_time_ms : start;
            m.exec_ms = exec;
            m.e2e_ms = m.wait_ms + exec;
            m.ttft_ms = m.wait_ms + prefill;
            m.tpot_ms = (exec - prefill) / static_cast<double>(lo);
            m.extrapolated = is_extrapolated(r->input_len, lo);
            m.slo_met = meets_slo(w.class_of(*r).slo, m.e2e_ms, m.ttft_ms, m.tpot_ms);
            records.push_back(m);
            makespan = std::max(makespan, exec);
        }
        clock = start + makespan;
        ++res.batches_started;
    }
    res.clock = clock;
    return res;
}

MetricsReport run(const std::vector<Schedule>& schedules, const Workload& w, const std::vector<InstanceState>& instances,
                  const LatencyCoefficients& c, const SimConfig& sim, double overhead_ms) {
    if (schedules.size() != instances.size()) throw DataError("simulator: schedule count does not match instance count");
    // instances are independent replays (own derived noise stream): replayed side by side, records
    // concatenated in instance order (the order the report sums them in)
    const std::size_t k = instances.size();
    std::vector<std::vector<RequestMetrics>> per(k);
    auto one = [&](std::size_t i) {
        Rng rng(Rng::derive(sim.seed, static_cast<std::uint64_t>(instances[i].id)));
        realize_batches(schedules[i].batches, w, c, 0.0, 0.0, sim.dispatch_gap_ms,
                        std::numeric_limits<double>::infinity(), sim.noise_pct, rng, per[i]);
    };
    std::size_t total = 0;
    for (const auto& s : schedules) total += s.request_count();
    if (k > 1 && total >= 4096) {
        std::vector<std::future<void>> fs;
        for (std::size_t i = 1; i < k; ++i) fs.push_back(std::async(std::launch::async, one, i));
        std::exception_ptr err;
        try {
            one(0);
        } catch (...) {
            err = std::current_exception();
        }
        for (auto& f : fs) {
            try {
                f.get();
            } catch (...) {
                if (!err) err = std::current_exception();
            }
        }
        if (err) std::rethrow_exception(err);
    } else {
        for (std::size_t i = 0; i < k; ++i) one(i);
    }
    std::vector<RequestMetrics> records;
    records.reserve(total);
    for (auto& v : per) records.insert(records.end(), v.begin(), v.end());
    return MetricsReport::from_records(std::move(records), overhead_ms);
}

FcfsResult run_fcfs(const Workload& w, const std::vector<InstanceState>& instances, const LatencyCoefficients& c,
                    const SimConfig& sim) {
    if (instances.empty()) throw DataError("run_fcfs: need at least one instance");
    for (const auto& inst : instances) inst.validate();
    // arrival order, ties by id
    std::vector<std::pair<double, int>> order;
    order.reserve(w.requests.size());
    for (const auto& r : w.requests) order.emplace_back(r.arrival_time_ms, r.id);
    std::sort(order.begin(), order.end());
    FcfsResult res;
    res.schedules.resize(instances.size());
    std::vector<RequestMetrics> records;
    // the earliest-ready instance takes the next greedy batch (ties: lowest instance index)
    using Slot = std::pair<double, std::size_t>;
    std::priority_queue<Slot, std::vector<Slot>, std::greater<>> ready;
    for (std::size_t i = 0; i < instances.size(); ++i) ready.emplace(0.0, i);
    Rng rng(sim.seed);  // one stream for the whole baseline, batches in dispatch order
    for (std::size_t pos = 0; pos < order.size();) {
        const auto [clock, inst] = ready.top();
        ready.pop();
        const std::size_t take = std::min<std::size_t>(instances[inst].max_batch_size, order.size() - pos);
        Batch batch;
        for (std::size_t j = 0; j < take; ++j) batch.push_back(order[pos + j].second);
        pos += take;
        const double gap = res.schedules[inst].batches.empty() ? 0.0 : sim.dispatch_gap_ms;
        const ReplayResult rr = realize_batches({batch}, w, c, clock, gap, gap, std::numeric_limits<double>::infinity(),
                                                sim.noise_pct, rng, records);
        res.schedules[inst].batches.push_back(std::move(batch));
        ready.emplace(rr.clock, inst);
    }
    res.report = MetricsReport::from_records(std::move(records), 0.0);
    return res;
}

double median(std::vector<double> v) {
    if (v.empty()) return 0.0;
    std::sort(v.begin(), v.end());
    const std::size_t mid = v.size() / 2;
    return v.size() % 2 ? v[mid] : 0.5 * (v[mid - 1] + v[mid]);
}

std::string policy_name(Policy p) {
    switch (p) {
        case Policy::SA: return "sa";
        case Policy::EXHAUSTIVE: return "exhaustive";
        case Policy::FCFS: return "fcfs";
    }
    return "?";
}

Policy parse_policy(const std::string& name) {
    if (name == "sa") return Policy::SA;
    if (name == "exhaustive") return Policy::EXHAUSTIVE;
    if (name == "fcfs") return Policy::FCFS;
    throw DataError("unknown policy '" + name + "' (expected sa, exhaustive, or fcfs)");
}

ComparisonTable compare(const Workload& w, const std::vector<InstanceState>& instances, const LatencyCoefficients& c,
                        const std::vector<Policy>& policies, const std::vector<std::uint64_t>& seeds,
                        const AnnealConfig& anneal_cfg, const SimConfig& sim_cfg, int exhaustive_cap) {
    int mb = 0;
    for (const auto& inst : instances) mb = std::max(mb, inst.max_batch_size);
    ComparisonTable table;
    for (Policy policy : policies) {
        for (std::uint64_t seed : seeds) {
            SimConfig sim = sim_cfg;
            sim.seed = seed;
            MetricsReport rep;
            if (policy == Policy::FCFS) {
                const auto t0 = std::chrono::steady_clock::now();
                rep = run_fcfs(w, instances, c, sim).report;
                rep.scheduling_overhead_ms =
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            } else {
                AnnealConfig cfg = anneal_cfg;
                cfg.seed = seed;
                ScheduleAllResult sr = schedule_all(w, instances, c, cfg, policy, exhaustive_cap);
                std::vector<Schedule> plans;
                plans.reserve(sr.per_instance.size());
                for (auto& ev : sr.per_instance) plans.push_back(std::move(ev.schedule));
                rep = run(plans, w, instances, c, sim, sr.overhead_ms);
            }
            ComparisonRow row;
            row.policy = policy_name(policy);
            row.seed = seed;
            row.n_requests = static_cast<int>(w.requests.size());
            row.max_batch = mb;
            row.attainment = rep.slo_attainment;
            row.avg_latency_ms = rep.avg_latency_ms;
            row.g_req_per_ms = rep.g;
            row.overhead_ms = rep.scheduling_overhead_ms;
            table.rows.push_back(row);
        }
    }
    for (Policy policy : policies) {
        std::vector<double> att, lat, g, ovh;
        for (const auto& r : table.rows) {
            if (r.policy != policy_name(policy)) continue;
            att.push_back(r.attainment), lat.push_back(r.avg_latency_ms), g.push_back(r.g_req_per_ms),
                ovh.push_back(r.overhead_ms);
        }
        ComparisonRow med;
        med.policy = policy_name(policy);
        med.n_requests = static_cast<int>(w.requests.size());
        med.max_batch = mb;
        med.attainment = median(att), med.avg_latency_ms = median(lat), med.g_req_per_ms = median(g),
        med.overhead_ms = median(ovh);
        table.medians.push_back(med);
    }
    return table;
}

// ================================================================ batched scoring (K1)
std::vector<ScheduleScore> evaluate_batch(const std::vector<Schedule>& schedules, const LatencyCoefficients& c,
                                          const Workload& w, int max_batch, int device) {
    std::vector<ScheduleScore> out(schedules.size());
    if (schedules.empty()) return out;
    std::vector<int> ids = schedules[0].flatten();
    std::sort(ids.begin(), ids.end());
    const int n = static_cast<int>(ids.size());
    if (n == 0) return out;
    if (n > SLO_MAX_N) throw CapacityError("evaluate_batch: more than 4096 requests");
    if (max_batch < 1) throw DataError("evaluate_batch: max_batch must be >= 1");
    if (max_batch > SLO_MAX_MB) throw CapacityError("evaluate_batch: max_batch above the engine limit of 16");
    const int words = (n + 31) / 32;
    std::vector<std::uint16_t> perms(schedules.size() * static_cast<std::size_t>(n));
    std::vector<std::uint32_t> bits(schedules.size() * static_cast<std::size_t>(words), 0u);
    for (std::size_t s = 0; s < schedules.size(); ++s) {
        if (!schedules[s].is_partition_of(ids, max_batch))
            throw DataError("evaluate_batch: every schedule must partition the same requests into batches of <= max_batch");
        int pos = 0;
        for (const Batch& b : schedules[s].batches) {
            for (int id : b)
                perms[s * n + pos++] = static_cast<std::uint16_t>(std::lower_bound(ids.begin(), ids.end(), id) - ids.begin());
            bits[s * words + ((pos - 1) >> 5)] |= 1u << ((pos - 1) & 31);
        }
    }
    std::vector<double> exec, deadline;
    cost_tables(w, ids, c, max_batch, exec, deadline);
    const int dev = detail::resolve_device(device);
    slo_ctx* ctx = detail::acquire_ctx(dev);
    std::vector<int32_t> nm(schedules.size());
    std::vector<double> t(schedules.size()), g(schedules.size());
    int rc = slo_problem_set(ctx, n, max_batch, exec.data(), deadline.data());
    if (rc == SLO_OK)
        rc = slo_evaluate_batch(ctx, static_cast<int32_t>(schedules.size()), perms.data(), bits.data(), nm.data(), t.data(),
                                g.data());
    if (rc == SLO_OK) detail::release_ctx(dev, ctx);
    else slo_ctx_destroy(ctx);
    detail::check(rc);
    for (std::size_t s = 0; s < schedules.size(); ++s) out[s] = ScheduleScore{nm[s], t[s], g[s]};
    return out;
}

// ================================================================ sweep / perturb
namespace {

// At most this many driver cells anneal at once (each on its own engine contexts with a share of
// the SMs): enough to fill the GPU with the small queues of a sweep, few enough that a large grid
// neither starves every cell of SMs nor holds hundreds of contexts' buffers.
constexpr std::size_t kMaxInflightCells = 8;

// Run job(i) for i in [0, count) on up to kMaxInflightCells host threads pulling job indices;
// exceptions are rethrown in job order after all finished.
template <typename F>
void run_concurrent(std::size_t count, F&& job) {
    std::vector<std::exception_ptr> errs(count);
    std::atomic<std::size_t> next{0};
    std::vector<std::thread> th;
    const std::size_t workers = std::min(count, kMaxInflightCells);
    th.reserve(workers);
    for (std::size_t w = 0; w < workers; ++w)
        th.emplace_back([&] {
            for (std::size_t i; (i = next.fetch_add(1)) < count;) {
                try {
                    job(i);
                } catch (...) {
                    errs[i] = std::current_exception();
                }
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

// SMs per anneal when `jobs` schedule_all calls over `k` instances run (at most
// kMaxInflightCells at once; Chains mode)
int sm_share(const AnnealConfig& cfg, std::size_t jobs, std::size_t k) {
    jobs = std::min(jobs, kMaxInflightCells);
    const int dev = detail::resolve_device(cfg.engine.device);
    slo_ctx* ctx = detail::acquire_ctx(dev);
    const int sms = slo_ctx_sm_count(ctx);
    detail::release_ctx(dev, ctx);
    return std::max(1, sms / static_cast<int>(std::max<std::size_t>(1, jobs * k)));
}

double* coeff_field(LatencyCoefficients& c, const std::string& name) {
    static const std::map<std::string, double LatencyCoefficients::*> f = {
        {"alpha_p", &LatencyCoefficients::alpha_p}, {"beta_p", &LatencyCoefficients::beta_p},
        {"gamma_p", &LatencyCoefficients::gamma_p}, {"delta_p", &LatencyCoefficients::delta_p},
        {"alpha_d", &LatencyCoefficients::alpha_d}, {"beta_d", &LatencyCoefficients::beta_d},
        {"gamma_d", &LatencyCoefficients::gamma_d}, {"delta_d", &LatencyCoefficients::delta_d}};
    auto it = f.find(name);
    if (it == f.end()) throw DataError("unknown coefficient '" + name + "'");
    return &(c.*(it->second));
}

}  // namespace

std::vector<SweepRow> sweep(const std::vector<Workload>& per_seed, const std::vector<std::uint64_t>& seeds,
                            const std::vector<InstanceState>& instances, const LatencyCoefficients& c,
                            const AnnealConfig& base, const std::vector<double>& t0_grid,
                            const std::vector<int>& iter_grid) {
    if (t0_grid.empty() || iter_grid.empty()) throw DataError("sweep: grids must be non-empty");
    if (per_seed.size() != seeds.size()) throw DataError("sweep: one workload per seed");
    const std::size_t cells = t0_grid.size() * iter_grid.size(), ns = seeds.size(), k = instances.size();
    // every (cell, seed) schedule_all at once
    std::vector<ScheduleAllResult> res(cells * ns);
    const bool chains = base.engine.mode == SearchMode::Chains;
    const int share = chains && base.engine.max_blocks <= 0 ? sm_share(base, cells * ns, k) : base.engine.max_blocks;
    auto job = [&](std::size_t j) {
        const std::size_t cell = j / ns, s = j % ns;
        AnnealConfig cfg = base;
        cfg.t0 = t0_grid[cell / iter_grid.size()];
        cfg.iter = iter_grid[cell % iter_grid.size()];
        cfg.seed = seeds[s];
        cfg.engine.max_blocks = share;
        res[j] = schedule_all(per_seed[s], instances, c, cfg);
    };
    if (chains) run_concurrent(cells * ns, job);
    else for (std::size_t j = 0; j < cells * ns; ++j) job(j);
    // score: per (seed, instance), all cells' schedules in one evaluator launch
    std::vector<SweepRow> rows;
    std::vector<std::vector<ScheduleScore>> score(cells * ns, std::vector<ScheduleScore>(k));
    for (std::size_t s = 0; s < ns; ++s)
        for (std::size_t i = 0; i < k; ++i) {
            std::vector<Schedule> batch;
            for (std::size_t cell = 0; cell < cells; ++cell) batch.push_back(res[cell * ns + s].per_instance[i].schedule);
            if (batch[0].request_count() == 0) continue;  // an instance without requests scores 0 / 0
            const auto sc = evaluate_batch(batch, c, per_seed[s], instances[i].max_batch_size, base.engine.device);
            for (std::size_t cell = 0; cell < cells; ++cell) score[cell * ns + s][i] = sc[cell];
        }
    for (std::size_t cell = 0; cell < cells; ++cell)
        for (std::size_t s = 0; s < ns; ++s) {
            int met = 0;
            double total = 0.0;
            for (std::size_t i = 0; i < k; ++i) met += score[cell * ns + s][i].n, total += score[cell * ns + s][i].t_ms;
            SweepRow r;
            r.t0 = t0_grid[cell / iter_grid.size()];
            r.iter = iter_grid[cell % iter_grid.size()];
            r.seed = seeds[s];
            r.g_req_per_ms = total > 0.0 ? met / total : 0.0;
            rows.push_back(r);
        }
    return rows;
}

std::vector<PerturbRow> perturb(const std::vector<Workload>& per_seed, const std::vector<std::uint64_t>& seeds,
                                const std::vector<InstanceState>& instances, const LatencyCoefficients& truth,
                                const AnnealConfig& base, const SimConfig& sim_cfg,
                                const std::vector<std::string>& params, const std::vector<double>& factors) {
    if (per_seed.size() != seeds.size()) throw DataError("perturb: one workload per seed");
    for (const auto& p : params) {
        LatencyCoefficients probe = truth;
        coeff_field(probe, p);  // unknown names fail before any GPU work
    }
    // job 0..ns-1: the baselines (predictor == truth); then (param, factor, seed)
    const std::size_t ns = seeds.size(), cases = params.size() * factors.size();
    const std::size_t jobs = ns * (1 + cases);
    std::vector<double> g(jobs);
    const bool chains = base.engine.mode == SearchMode::Chains;
    const int share = chains && base.engine.max_blocks <= 0 ? sm_share(base, jobs, instances.size()) : base.engine.max_blocks;
    auto job = [&](std::size_t j) {
        const std::size_t s = j % ns, cs = j / ns;
        LatencyCoefficients predictor = truth;
        if (cs > 0) *coeff_field(predictor, params[(cs - 1) / factors.size()]) *= factors[(cs - 1) % factors.size()];
        AnnealConfig cfg = base;
        cfg.seed = seeds[s];
        cfg.engine.max_blocks = share;
        const ScheduleAllResult r = schedule_all(per_seed[s], instances, predictor, cfg);
        std::vector<Schedule> plans;
        for (const auto& ev : r.per_instance) plans.push_back(ev.schedule);
        SimConfig sim = sim_cfg;
        sim.seed = seeds[s];
        g[j] = run(plans, per_seed[s], instances, truth, sim, r.overhead_ms).g;
    };
    if (chains) run_concurrent(jobs, job);
    else for (std::size_t j = 0; j < jobs; ++j) job(j);
    std::vector<PerturbRow> rows;
    for (std::size_t cs = 1; cs <= cases; ++cs)
        for (std::size_t s = 0; s < ns; ++s) {
            PerturbRow r;
            r.param = params[(cs - 1) / factors.size()];
            r.factor = factors[(cs - 1) % factors.size()];
            r.seed = seeds[s];
            r.g_req_per_ms = g[cs * ns + s];
            r.baseline_g = g[s];
            r.degradation_pct = r.baseline_g > 0.0 ? (r.baseline_g - r.g_req_per_ms) / r.baseline_g * 100.0 : 0.0;
            rows.push_back(r);
        }
    return rows;
}

}  // namespace slosched
