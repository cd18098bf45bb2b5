// extern "C" face of the UNMODIFIED reference library -- TEST INFRASTRUCTURE.
//
// Compiled together with /root/reference/proj/src/*.cpp (see oracle/Makefile)
// into oracle/_ref/libslosched_ref.so. Only tests/, __graft_entry__.smoke()
// and bench.py's reference / cpu_baseline legs load it, and only as the
// checker or the timed CPU baseline -- never on the product path.
//
// Every function builds reference types from flat arrays and calls the
// reference's own public API:
//   generate_mixed / Estimator   P:src/workload.cpp:158-183, P:src/output_estimator.cpp:385-415
//   evaluate                     P:src/objective.cpp:55-82
//   initial_candidates           P:src/priority_mapper.cpp:292-311
//   neighbor                     P:src/priority_mapper.cpp:322-338
//   anneal                       P:src/priority_mapper.cpp:340-411
//   exhaustive                   P:src/priority_mapper.cpp:440-517
//   schedule_all                 P:src/scheduler.cpp:92-129
//   run / run_fcfs               P:src/simulator.cpp:49-123
//   Estimator                    P:src/output_estimator.cpp:10-78
// Errors map to codes: 1 DataError, 2 CapacityError, 6 std::invalid_argument,
// 9 anything else; the message is kept in ref_last_error().
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "slosched/latency_model.hpp"
#include "slosched/objective.hpp"
#include "slosched/output_estimator.hpp"
#include "slosched/priority_mapper.hpp"
#include "slosched/rng.hpp"
#include "slosched/scheduler.hpp"
#include "slosched/simulator.hpp"
#include "slosched/workload.hpp"

using namespace slosched;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const DataError& e) {
        g_err = e.what();
        return 1;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

LatencyCoefficients coeffs_of(const double* c) {
    return {c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]};
}

struct Flat {
    int n;
    const int *id, *cls, *in_len, *true_out, *pred_out;
    const double* arrival;
    int n_classes;
    const int *class_id, *kind;
    const double *e2e, *ttft, *tpot;
};

Workload build(const Flat& f) {
    std::vector<TaskClass> classes;
    for (int c = 0; c < f.n_classes; ++c) {
        TaskClass t;
        t.id = f.class_id[c];
        t.name = "c" + std::to_string(t.id);
        t.slo = f.kind[c] == 0 ? SloSpec::e2e(f.e2e[c]) : SloSpec::ttft_tpot(f.ttft[c], f.tpot[c]);
        classes.push_back(t);
    }
    std::vector<Request> reqs;
    for (int i = 0; i < f.n; ++i) {
        Request r;
        r.id = f.id[i];
        r.task_class_id = f.cls[i];
        r.input_len = f.in_len[i];
        r.true_output_len = f.true_out[i];
        if (f.pred_out[i] >= 0) r.predicted_output_len = f.pred_out[i];
        r.arrival_time_ms = f.arrival[i];
        reqs.push_back(r);
    }
    return validate_workload(std::move(reqs), std::move(classes));
}

Schedule schedule_of(const int* ids, const int* sizes, int nb) {
    Schedule s;
    int pos = 0;
    for (int k = 0; k < nb; ++k) {
        s.batches.emplace_back(ids + pos, ids + pos + sizes[k]);
        pos += sizes[k];
    }
    return s;
}

void emit(const Schedule& s, int* ids, int* sizes, int* nb) {
    int pos = 0;
    for (const auto& b : s.batches) {
        sizes[(*nb)++] = static_cast<int>(b.size());
        for (int id : b) ids[pos++] = id;
    }
}

AnnealConfig config_of(const double* cfg, std::uint64_t seed) {
    // cfg = {t0, t_thres, iter, tau, has_scale, scale}
    AnnealConfig c;
    c.t0 = cfg[0];
    c.t_thres = cfg[1];
    c.iter = static_cast<int>(cfg[2]);
    c.tau = cfg[3];
    c.seed = seed;
    if (cfg[4] != 0.0) c.objective_scale = cfg[5];
    return c;
}

}  // namespace

#define FLAT_ARGS                                                                          \
    int n, const int *id, const int *cls, const int *in_len, const int *true_out,         \
        const int *pred_out, const double *arrival, int n_classes, const int *class_id,   \
        const int *kind, const double *e2e, const double *ttft, const double *tpot
#define FLAT_PASS Flat{n, id, cls, in_len, true_out, pred_out, arrival, n_classes, class_id, kind, e2e, ttft, tpot}

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Rng stream: next_u64 x count (P:include/slosched/rng.hpp:24-34)
void ref_rng_u64(std::uint64_t seed, int count, std::uint64_t* out) {
    Rng r(seed);
    for (int i = 0; i < count; ++i) out[i] = r.next_u64();
}

// uniform_index(bounds[i]) in sequence from one Rng (rng.hpp:46-57)
void ref_rng_index(std::uint64_t seed, int count, const std::uint64_t* bounds, std::uint64_t* out) {
    Rng r(seed);
    for (int i = 0; i < count; ++i) out[i] = r.uniform_index(bounds[i]);
}

void ref_rng_uniform(std::uint64_t seed, int count, double* out) {
    Rng r(seed);
    for (int i = 0; i < count; ++i) out[i] = r.uniform();
}

void ref_rng_normal(std::uint64_t seed, int count, double* out) {
    Rng r(seed);
    for (int i = 0; i < count; ++i) out[i] = r.normal();
}

std::uint64_t ref_rng_derive(std::uint64_t seed, std::uint64_t stream) { return Rng::derive(seed, stream); }

// predict_prefill / per_token_decode / decode_total / exec / tpot (latency_model.cpp:86-113)
int ref_predict(const double* c, int b, int li, int lo, double* out5) {
    return guarded([&] {
        const auto k = coeffs_of(c);
        out5[0] = predict_prefill(k, b, li);
        out5[1] = predict_per_token_decode(k, b, li);
        out5[2] = predict_decode_total(k, b, li, lo);
        out5[3] = predict_exec(k, b, li, lo);
        out5[4] = lo > 0 ? predict_tpot(k, b, li, lo) : 0.0;
    });
}

// generate_mixed(n, seed, default_synth_classes()) then, for predict_mode 1,
// the CLI's estimator pass with Rng(derive(seed, 0x9e37)) (P:tools/slosched.cpp:131-142);
// predict_mode 0 copies the true lengths (tests' mixed_workload helper).
int ref_generate_mixed(int n, std::uint64_t seed, int predict_mode, int* id, int* cls, int* in_len,
                       int* true_out, int* pred_out, double* arrival) {
    return guarded([&] {
        auto [code, chat] = default_synth_classes();
        auto reqs = generate_mixed(n, seed, code, chat);
        if (predict_mode == 1) {
            Estimator est({code, chat});
            Rng rng(Rng::derive(seed, 0x9e37));
            assign_predicted_lengths(reqs, est, rng);
        } else {
            for (auto& r : reqs) r.predicted_output_len = r.true_output_len;
        }
        for (int i = 0; i < n; ++i) {
            id[i] = reqs[i].id;
            cls[i] = reqs[i].task_class_id;
            in_len[i] = reqs[i].input_len;
            true_out[i] = reqs[i].true_output_len;
            pred_out[i] = *reqs[i].predicted_output_len;
            arrival[i] = reqs[i].arrival_time_ms;
        }
    });
}

// evaluate(); per-request arrays are in flattened schedule order
int ref_evaluate(FLAT_ARGS, const double* c, const int* s_ids, const int* s_sizes, int s_nb,
                 int* n_met, double* t, double* g, double* wait, double* exec, double* e2e_out,
                 double* ttft_out, double* tpot_out, int* met) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        const auto ev = evaluate(schedule_of(s_ids, s_sizes, s_nb), coeffs_of(c), w);
        *n_met = ev.n;
        *t = ev.t_ms;
        *g = ev.g;
        for (std::size_t i = 0; i < ev.per_request.size(); ++i) {
            const auto& m = ev.per_request[i];
            if (wait) wait[i] = m.wait_ms;
            if (exec) exec[i] = m.exec_ms;
            if (e2e_out) e2e_out[i] = m.e2e_ms;
            if (ttft_out) ttft_out[i] = m.ttft_ms;
            if (tpot_out) tpot_out[i] = m.tpot_ms;
            if (met) met[i] = m.slo_met ? 1 : 0;
        }
    });
}

int ref_initial_candidates(FLAT_ARGS, const double* c, const int* ids, int n_ids, int max_batch,
                           int* sorted_ids, int* sorted_sizes, int* sorted_nb, int* input_ids,
                           int* input_sizes, int* input_nb) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        auto [s, in] = initial_candidates(w, std::vector<int>(ids, ids + n_ids), coeffs_of(c), max_batch);
        *sorted_nb = 0;
        *input_nb = 0;
        emit(s, sorted_ids, sorted_sizes, sorted_nb);
        emit(in, input_ids, input_sizes, input_nb);
    });
}

// `steps` chained neighbor() calls from one Rng(seed)
int ref_neighbor_walk(const int* s_ids, const int* s_sizes, int s_nb, std::uint64_t seed, int steps,
                      int max_batch, int* out_ids, int* out_sizes, int* out_nb) {
    return guarded([&] {
        Schedule s = schedule_of(s_ids, s_sizes, s_nb);
        Rng rng(seed);
        for (int i = 0; i < steps; ++i) s = neighbor(s, rng, max_batch);
        *out_nb = 0;
        emit(s, out_ids, out_sizes, out_nb);
    });
}

// anneal(); stats6 = {proposals, accepted, shortcut, g_sorted, g_input, scale}
int ref_anneal(FLAT_ARGS, const double* c, const int* ids, int n_ids, const double* cfg,
               std::uint64_t seed, int max_batch, int* out_ids, int* out_sizes, int* out_nb,
               int* n_met, double* t, double* g, double* stats6) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        const auto res = anneal(w, std::vector<int>(ids, ids + n_ids), coeffs_of(c),
                                config_of(cfg, seed), max_batch);
        *out_nb = 0;
        emit(res.best.schedule, out_ids, out_sizes, out_nb);
        *n_met = res.best.n;
        *t = res.best.t_ms;
        *g = res.best.g;
        stats6[0] = static_cast<double>(res.stats.proposals);
        stats6[1] = static_cast<double>(res.stats.accepted);
        stats6[2] = res.stats.shortcut ? 1.0 : 0.0;
        stats6[3] = res.stats.g_sorted_start;
        stats6[4] = res.stats.g_input_start;
        stats6[5] = res.stats.objective_scale_used;
    });
}

// CPU baseline: `threads` independent anneal() chains (seeds seed0 .. seed0+threads-1),
// one std::thread each, `reps` calls per thread. Reports the summed proposals, the
// wall time of the whole parallel region and the best result over all chains.
int ref_anneal_parallel(FLAT_ARGS, const double* c, const int* ids, int n_ids, const double* cfg,
                        std::uint64_t seed0, int max_batch, int threads, int reps,
                        double* out_proposals, double* out_wall_ms, int* best_n_met,
                        double* best_g) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        const std::vector<int> idv(ids, ids + n_ids);
        const auto k = coeffs_of(c);
        std::vector<std::uint64_t> props(threads, 0);
        std::vector<double> gs(threads, -1.0);
        std::vector<int> ns(threads, 0);
        std::vector<std::string> errs(threads);
        const auto t_start = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int th = 0; th < threads; ++th) {
            pool.emplace_back([&, th] {
                try {
                    for (int r = 0; r < reps; ++r) {
                        const auto res = anneal(w, idv, k, config_of(cfg, seed0 + th + static_cast<std::uint64_t>(r) * threads), max_batch);
                        props[th] += res.stats.proposals;
                        if (res.best.g > gs[th]) {
                            gs[th] = res.best.g;
                            ns[th] = res.best.n;
                        }
                    }
                } catch (const std::exception& e) {
                    errs[th] = e.what();
                }
            });
        }
        for (auto& t : pool) t.join();
        *out_wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        for (const auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        double total = 0.0;
        *best_g = -1.0;
        for (int th = 0; th < threads; ++th) {
            total += static_cast<double>(props[th]);
            if (gs[th] > *best_g) {
                *best_g = gs[th];
                *best_n_met = ns[th];
            }
        }
        *out_proposals = total;
    });
}

int ref_exhaustive(FLAT_ARGS, const double* c, const int* ids, int n_ids, int max_batch, int n_cap,
                   int* out_ids, int* out_sizes, int* out_nb, int* n_met, double* t, double* g,
                   double* evaluated) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        const auto res = exhaustive(w, std::vector<int>(ids, ids + n_ids), coeffs_of(c), max_batch, n_cap);
        *out_nb = 0;
        emit(res.best.schedule, out_ids, out_sizes, out_nb);
        *n_met = res.best.n;
        *t = res.best.t_ms;
        *g = res.best.g;
        *evaluated = static_cast<double>(res.schedules_evaluated);
    });
}

// schedule_all(Policy::SA); instances given as arrays; outputs per instance
// concatenated: inst_nb[i] batches, inst_count[i] requests; plus n/t/g per instance
int ref_schedule_all(FLAT_ARGS, const double* c, int n_inst, const int* inst_id,
                     const double* total_mem, const double* remaining_mem, const double* mu,
                     const double* sigma, const int* inst_mb, const double* cfg, std::uint64_t seed,
                     int* out_ids, int* out_sizes, int* inst_nb, int* inst_count, int* inst_n,
                     double* inst_t, double* inst_g, int* epochs) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        std::vector<InstanceState> fleet;
        for (int i = 0; i < n_inst; ++i) {
            InstanceState s;
            s.id = inst_id[i];
            s.total_mem = static_cast<std::uint64_t>(total_mem[i]);
            s.remaining_mem = static_cast<std::uint64_t>(remaining_mem[i]);
            s.mem_utility = mu[i];
            s.bytes_per_token = sigma[i];
            s.max_batch_size = inst_mb[i];
            fleet.push_back(s);
        }
        const auto res = schedule_all(w, fleet, coeffs_of(c), config_of(cfg, seed));
        int pos = 0, kb = 0;
        for (int i = 0; i < n_inst; ++i) {
            const auto& ev = res.per_instance[i];
            inst_nb[i] = static_cast<int>(ev.schedule.batches.size());
            inst_count[i] = static_cast<int>(ev.schedule.request_count());
            inst_n[i] = ev.n;
            inst_t[i] = ev.t_ms;
            inst_g[i] = ev.g;
            for (const auto& b : ev.schedule.batches) {
                out_sizes[kb++] = static_cast<int>(b.size());
                for (int id2 : b) out_ids[pos++] = id2;
            }
        }
        *epochs = res.assignment.epochs;
    });
}

}  // extern "C"

namespace {
std::vector<InstanceState> fleet_of(int n_inst, const int* inst_id, const double* total_mem,
                                    const double* remaining_mem, const double* mu, const double* sigma,
                                    const int* inst_mb) {
    std::vector<InstanceState> fleet;
    for (int i = 0; i < n_inst; ++i) {
        InstanceState s;
        s.id = inst_id[i];
        s.total_mem = static_cast<std::uint64_t>(total_mem[i]);
        s.remaining_mem = static_cast<std::uint64_t>(remaining_mem[i]);
        s.mem_utility = mu[i];
        s.bytes_per_token = sigma[i];
        s.max_batch_size = inst_mb[i];
        fleet.push_back(s);
    }
    return fleet;
}
// records as 8 doubles each: id, wait, exec, e2e, ttft, tpot, met, extrapolated; report as 6
void dump(const MetricsReport& r, double* rec, double* rep) {
    for (std::size_t i = 0; i < r.per_request.size(); ++i) {
        const auto& m = r.per_request[i];
        double* o = rec + 8 * i;
        o[0] = m.request_id, o[1] = m.wait_ms, o[2] = m.exec_ms, o[3] = m.e2e_ms, o[4] = m.ttft_ms, o[5] = m.tpot_ms;
        o[6] = m.slo_met ? 1.0 : 0.0, o[7] = m.extrapolated ? 1.0 : 0.0;
    }
    rep[0] = r.slo_attainment, rep[1] = r.avg_latency_ms, rep[2] = r.g, rep[3] = r.scheduling_overhead_ms;
    rep[4] = r.n_met, rep[5] = r.total_latency_ms;
}
}  // namespace

extern "C" {

// run() over per-instance schedules (inst_nb[i] batches each, concatenated)
int ref_run(FLAT_ARGS, const double* c, int n_inst, const int* inst_id, const double* total_mem,
            const double* remaining_mem, const double* mu, const double* sigma, const int* inst_mb,
            const int* s_ids, const int* s_sizes, const int* inst_nb, double noise, double gap,
            std::uint64_t seed, double overhead, double* rec, double* rep) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        const auto fleet = fleet_of(n_inst, inst_id, total_mem, remaining_mem, mu, sigma, inst_mb);
        std::vector<Schedule> plans;
        int pos = 0, kb = 0;
        for (int i = 0; i < n_inst; ++i) {
            plans.push_back(schedule_of(s_ids + pos, s_sizes + kb, inst_nb[i]));
            pos += static_cast<int>(plans.back().request_count());
            kb += inst_nb[i];
        }
        SimConfig sim;
        sim.noise_pct = noise, sim.dispatch_gap_ms = gap, sim.seed = seed;
        dump(run(plans, w, fleet, coeffs_of(c), sim, overhead), rec, rep);
    });
}

int ref_run_fcfs(FLAT_ARGS, const double* c, int n_inst, const int* inst_id, const double* total_mem,
                 const double* remaining_mem, const double* mu, const double* sigma, const int* inst_mb,
                 double noise, double gap, std::uint64_t seed, int* out_ids, int* out_sizes, int* inst_nb,
                 double* rec, double* rep) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        SimConfig sim;
        sim.noise_pct = noise, sim.dispatch_gap_ms = gap, sim.seed = seed;
        const FcfsResult r = run_fcfs(w, fleet_of(n_inst, inst_id, total_mem, remaining_mem, mu, sigma, inst_mb),
                                      coeffs_of(c), sim);
        int pos = 0, kb = 0;
        for (int i = 0; i < n_inst; ++i) {
            int nb = 0;
            emit(r.schedules[i], out_ids + pos, out_sizes + kb, &nb);
            inst_nb[i] = nb;
            pos += static_cast<int>(r.schedules[i].request_count());
            kb += nb;
        }
        dump(r.report, rec, rep);
    });
}

// Estimator: observe (class, len) pairs in order, then predict with Rng(seed)
int ref_estimator(int n_classes, const int* class_id, const int* prior_kind, const double* prior_a,
                  const double* prior_b, int n_obs, const int* obs_cls, const int* obs_len, int n_pred,
                  const int* pred_cls, std::uint64_t seed, int* pred_out, long long* model_count,
                  double* model_mean, double* model_m2) {
    return guarded([&] {
        std::vector<TaskClass> classes(n_classes);
        for (int k = 0; k < n_classes; ++k) {
            classes[k].id = class_id[k];
            classes[k].slo = SloSpec::e2e(1.0);
            if (prior_kind[k] == 1) classes[k].output_prior = GaussianPrior{prior_a[k], prior_b[k]};
            else if (prior_kind[k] == 2)
                classes[k].output_prior = RangePrior{static_cast<int>(prior_a[k]), static_cast<int>(prior_b[k])};
        }
        Estimator est(classes);
        for (int i = 0; i < n_obs; ++i) est.observe_output(obs_cls[i], obs_len[i]);
        for (int k = 0; k < n_classes; ++k) {
            const LengthModel& m = est.model_for(class_id[k]);
            model_count[k] = m.count, model_mean[k] = m.mean, model_m2[k] = m.m2;
        }
        Rng rng(seed);
        for (int i = 0; i < n_pred; ++i) pred_out[i] = est.predict(pred_cls[i], rng);
    });
}

// compare(): rows as 6 doubles (policy code, seed, attainment, avg latency, g, overhead), medians too
int ref_compare(FLAT_ARGS, const double* c, int n_inst, const int* inst_id, const double* total_mem,
                const double* remaining_mem, const double* mu, const double* sigma, const int* inst_mb,
                int n_pol, const int* policies, int n_seeds, const std::uint64_t* seeds, const double* cfg,
                double noise, double gap, int n_cap, double* rows, double* medians) {
    return guarded([&] {
        Workload w = build(FLAT_PASS);
        std::vector<Policy> pol;
        for (int i = 0; i < n_pol; ++i) pol.push_back(static_cast<Policy>(policies[i]));
        SimConfig sim;
        sim.noise_pct = noise, sim.dispatch_gap_ms = gap;
        const auto t = compare(w, fleet_of(n_inst, inst_id, total_mem, remaining_mem, mu, sigma, inst_mb),
                               coeffs_of(c), pol, std::vector<std::uint64_t>(seeds, seeds + n_seeds),
                               config_of(cfg, 0), sim, n_cap);
        auto put = [](const ComparisonRow& r, double* o) {
            o[0] = static_cast<double>(parse_policy(r.policy)), o[1] = static_cast<double>(r.seed);
            o[2] = r.attainment, o[3] = r.avg_latency_ms, o[4] = r.g_req_per_ms, o[5] = r.overhead_ms;
        };
        for (std::size_t i = 0; i < t.rows.size(); ++i) put(t.rows[i], rows + 6 * i);
        for (std::size_t i = 0; i < t.medians.size(); ++i) put(t.medians[i], medians + 6 * i);
    });
}

}  // extern "C"
