// Flat C ABI (include/slosched_api.h) over the C++ scheduler API.
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "slosched_api.h"
#include "slosched_b200.hpp"
#include "slosched_gpu.h"

using namespace slosched;

namespace {

thread_local std::string g_api_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return SLO_OK;
    } catch (const DataError& e) {
        g_api_err = e.what();
        return SLO_ERR_DATA;
    } catch (const CapacityError& e) {
        g_api_err = e.what();
        return SLO_ERR_CAPACITY;
    } catch (const std::invalid_argument& e) {
        g_api_err = e.what();
        return SLO_ERR_ARG;
    } catch (const EngineError& e) {
        g_api_err = e.what();
        return SLO_ERR_CUDA;
    } catch (const std::exception& e) {
        g_api_err = e.what();
        return SLO_ERR_STATE;
    }
}

LatencyCoefficients coeffs_of(const double* c) { return {c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]}; }

Workload workload_of(const slosched_workload* v) {
    if (!v) throw std::invalid_argument("null workload");
    std::vector<TaskClass> classes;
    for (int c = 0; c < v->n_classes; ++c) {
        TaskClass t;
        t.id = v->class_id[c];
        t.name = "class" + std::to_string(t.id);
        t.slo = v->kind[c] == 0 ? SloSpec::e2e(v->e2e[c]) : SloSpec::ttft_tpot(v->ttft[c], v->tpot[c]);
        classes.push_back(std::move(t));
    }
    std::vector<Request> reqs(v->n);
    for (int i = 0; i < v->n; ++i) {
        Request& r = reqs[i];
        r.id = v->id[i];
        r.task_class_id = v->cls[i];
        r.input_len = v->in_len[i];
        r.true_output_len = v->true_out[i];
        if (v->pred_out[i] >= 0) r.predicted_output_len = v->pred_out[i];
        r.arrival_time_ms = v->arrival[i];
    }
    return validate_workload(std::move(reqs), std::move(classes));
}

Schedule schedule_of(const int32_t* ids, const int32_t* sizes, int32_t nb) {
    Schedule s;
    int pos = 0;
    for (int k = 0; k < nb; ++k) {
        s.batches.emplace_back(ids + pos, ids + pos + sizes[k]);
        pos += sizes[k];
    }
    return s;
}

int emit(const Schedule& s, int32_t* ids, int32_t* sizes) {
    int pos = 0, nb = 0;
    for (const auto& b : s.batches) {
        sizes[nb++] = static_cast<int32_t>(b.size());
        for (int id : b) ids[pos++] = id;
    }
    return nb;
}

std::vector<InstanceState> fleet_of(const slosched_fleet* f) {
    if (!f) throw std::invalid_argument("null fleet");
    std::vector<InstanceState> fleet(f->n);
    for (int i = 0; i < f->n; ++i) {
        fleet[i].id = f->id[i];
        fleet[i].total_mem = static_cast<std::uint64_t>(f->total_mem[i]);
        fleet[i].remaining_mem = static_cast<std::uint64_t>(f->remaining_mem[i]);
        fleet[i].mem_utility = f->mu[i];
        fleet[i].bytes_per_token = f->sigma[i];
        fleet[i].max_batch_size = f->max_batch[i];
    }
    return fleet;
}

SimConfig sim_of(const slosched_sim_config* s) {
    SimConfig c;
    if (s) c.noise_pct = s->noise_pct, c.dispatch_gap_ms = s->dispatch_gap_ms, c.seed = s->seed;
    return c;
}

void records_out(const std::vector<RequestMetrics>& v, slosched_record* out) {
    if (!out) return;
    for (std::size_t i = 0; i < v.size(); ++i) {
        const auto& m = v[i];
        out[i] = slosched_record{m.request_id, m.wait_ms, m.exec_ms, m.e2e_ms, m.ttft_ms, m.tpot_ms, m.slo_met ? 1 : 0,
                                 m.extrapolated ? 1 : 0};
    }
}

void report_out(const MetricsReport& r, slosched_report* out) {
    if (out)
        *out = slosched_report{r.slo_attainment, r.avg_latency_ms, r.g, r.scheduling_overhead_ms, r.n_met,
                               r.total_latency_ms};
}

// the reference CLI's synthetic workload for a seed (P:tools/slosched.cpp:119-142)
Workload synth_workload(int n, std::uint64_t seed, int predict_mode) {
    auto [code, chat] = default_synth_classes();
    auto reqs = generate_mixed(n, seed, code, chat);
    if (predict_mode == 1) {
        Rng rng(Rng::derive(seed, 0x9e37));
        assign_predicted_lengths_from_priors(reqs, {code, chat}, rng);
    } else {
        for (auto& r : reqs) r.predicted_output_len = r.true_output_len;
    }
    return validate_workload(std::move(reqs), {code, chat});
}

AnnealConfig config_of(const slosched_anneal_config* c) {
    AnnealConfig a;
    if (!c) return a;
    a.t0 = c->t0;
    a.t_thres = c->t_thres;
    a.iter = c->iter;
    a.tau = c->tau;
    a.seed = c->seed;
    if (c->has_objective_scale) a.objective_scale = c->objective_scale;
    a.engine.mode = c->mode == 1 ? SearchMode::Replay : SearchMode::Chains;
    a.engine.chains = c->chains;
    a.engine.budget_ms = c->budget_ms;
    if (c->n_scale_ladder > 0) a.engine.scale_ladder.assign(c->scale_ladder, c->scale_ladder + c->n_scale_ladder);
    a.engine.device = c->device;
    a.engine.chain_begin = c->chain_begin;
    a.engine.chain_end = c->chain_end;
    a.engine.concurrent_instances = c->sequential_instances == 0;
    a.engine.max_blocks = c->max_blocks;
    a.engine.deadline_start = c->start_policy == 0;
    if (c->n_devices > 0 && c->devices) a.engine.devices.assign(c->devices, c->devices + c->n_devices);
    a.engine.comm_ctx = static_cast<slo_ctx*>(c->comm_ctx);
    return a;
}

void stats_out(const AnnealStats& s, slosched_anneal_stats* o) {
    if (!o) return;
    o->proposals = s.proposals;
    o->accepted = s.accepted;
    o->shortcut = s.shortcut ? 1 : 0;
    o->g_sorted_start = s.g_sorted_start;
    o->g_input_start = s.g_input_start;
    o->objective_scale_used = s.objective_scale_used;
    o->chains_run = s.chains_run;
    o->levels_run = s.levels_run;
    o->best_chain = s.best_chain;
    o->engine_g = s.engine_g;
    o->engine_t = s.engine_t;
    o->kernel_ms = s.kernel_ms;
    o->g_deadline_start = s.g_deadline_start;
    o->exchange_ms = s.exchange_ms;
    o->devices = s.devices;
}

}  // namespace

extern "C" {

const char* slosched_last_error(void) { return g_api_err.c_str(); }

int slosched_predict(const double* c, int32_t b, int32_t li, int32_t lo, double* out5) {
    return guarded([&] {
        const auto k = coeffs_of(c);
        out5[0] = predict_prefill(k, b, li);
        out5[1] = predict_per_token_decode(k, b, li);
        out5[2] = predict_decode_total(k, b, li, lo);
        out5[3] = predict_exec(k, b, li, lo);
        out5[4] = lo > 0 ? predict_tpot(k, b, li, lo) : 0.0;
    });
}

double slosched_latest_start(double s, double c) { return latest_start(s, c); }

int slosched_generate_mixed(int32_t n, uint64_t seed, int32_t predict_mode, int32_t* id, int32_t* cls,
                            int32_t* in_len, int32_t* true_out, int32_t* pred_out, double* arrival) {
    return guarded([&] {
        if (n < 0) throw std::invalid_argument("generate_mixed: n must be >= 0");
        auto [code, chat] = default_synth_classes();
        auto reqs = generate_mixed(n, seed, code, chat);
        if (predict_mode == 1) {
            Rng rng(Rng::derive(seed, 0x9e37));
            assign_predicted_lengths_from_priors(reqs, {code, chat}, rng);
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

int slosched_evaluate(const slosched_workload* w, const double* c, const int32_t* ids, const int32_t* sizes, int32_t nb,
                      int32_t* n_met, double* t, double* g, double* wait, double* exec, double* e2e, double* ttft,
                      double* tpot, int32_t* met, int32_t* extrapolated) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        const auto ev = evaluate(schedule_of(ids, sizes, nb), coeffs_of(c), wl);
        *n_met = ev.n;
        *t = ev.t_ms;
        *g = ev.g;
        for (std::size_t i = 0; i < ev.per_request.size(); ++i) {
            const auto& m = ev.per_request[i];
            if (wait) wait[i] = m.wait_ms;
            if (exec) exec[i] = m.exec_ms;
            if (e2e) e2e[i] = m.e2e_ms;
            if (ttft) ttft[i] = m.ttft_ms;
            if (tpot) tpot[i] = m.tpot_ms;
            if (met) met[i] = m.slo_met ? 1 : 0;
            if (extrapolated) extrapolated[i] = m.extrapolated ? 1 : 0;
        }
    });
}

int slosched_initial_candidates(const slosched_workload* w, const double* c, const int32_t* ids, int32_t n,
                                int32_t max_batch, int32_t* sorted_ids, int32_t* sorted_sizes, int32_t* sorted_nb,
                                int32_t* input_ids, int32_t* input_sizes, int32_t* input_nb) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        auto [s, i] = initial_candidates(wl, std::vector<int>(ids, ids + n), coeffs_of(c), max_batch);
        *sorted_nb = emit(s, sorted_ids, sorted_sizes);
        *input_nb = emit(i, input_ids, input_sizes);
    });
}

int slosched_deadline_first_candidate(const slosched_workload* w, const double* c, const int32_t* ids, int32_t n,
                                      int32_t max_batch, int32_t* out_ids, int32_t* out_sizes, int32_t* out_nb) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        *out_nb = emit(deadline_first_candidate(wl, std::vector<int>(ids, ids + n), coeffs_of(c), max_batch), out_ids,
                       out_sizes);
    });
}

int slosched_neighbor_walk(const int32_t* ids, const int32_t* sizes, int32_t nb, uint64_t seed, int32_t steps,
                           int32_t max_batch, int32_t* out_ids, int32_t* out_sizes, int32_t* out_nb) {
    return guarded([&] {
        Schedule s = schedule_of(ids, sizes, nb);
        Rng rng(seed);
        for (int i = 0; i < steps; ++i) s = neighbor(s, rng, max_batch);
        *out_nb = emit(s, out_ids, out_sizes);
    });
}

int slosched_anneal(const slosched_workload* w, const double* c, const int32_t* ids, int32_t n,
                    const slosched_anneal_config* cfg, int32_t max_batch, int32_t* out_ids, int32_t* out_sizes,
                    int32_t* out_nb, int32_t* n_met, double* t, double* g, slosched_anneal_stats* stats) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        const AnnealResult r = anneal(wl, std::vector<int>(ids, ids + n), coeffs_of(c), config_of(cfg), max_batch);
        *out_nb = emit(r.best.schedule, out_ids, out_sizes);
        *n_met = r.best.n;
        *t = r.best.t_ms;
        *g = r.best.g;
        stats_out(r.stats, stats);
    });
}

int slosched_schedule_all(const slosched_workload* w, const double* c, int32_t n_inst, const int32_t* inst_id,
                          const double* total_mem, const double* remaining_mem, const double* mu, const double* sigma,
                          const int32_t* inst_mb, const slosched_anneal_config* cfg, int32_t* out_ids,
                          int32_t* out_sizes, int32_t* inst_nb, int32_t* inst_count, int32_t* inst_n, double* inst_t,
                          double* inst_g, int32_t* epochs, double* overhead_ms) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        std::vector<InstanceState> fleet(n_inst);
        for (int i = 0; i < n_inst; ++i) {
            fleet[i].id = inst_id[i];
            fleet[i].total_mem = static_cast<std::uint64_t>(total_mem[i]);
            fleet[i].remaining_mem = static_cast<std::uint64_t>(remaining_mem[i]);
            fleet[i].mem_utility = mu[i];
            fleet[i].bytes_per_token = sigma[i];
            fleet[i].max_batch_size = inst_mb[i];
        }
        const auto res = schedule_all(wl, fleet, coeffs_of(c), config_of(cfg));
        int pos = 0, kb = 0;
        for (int i = 0; i < n_inst; ++i) {
            const auto& ev = res.per_instance[i];
            inst_nb[i] = static_cast<int32_t>(ev.schedule.batches.size());
            inst_count[i] = static_cast<int32_t>(ev.schedule.request_count());
            inst_n[i] = ev.n;
            inst_t[i] = ev.t_ms;
            inst_g[i] = ev.g;
            for (const auto& b : ev.schedule.batches) {
                out_sizes[kb++] = static_cast<int32_t>(b.size());
                for (int id : b) out_ids[pos++] = id;
            }
        }
        *epochs = res.assignment.epochs;
        if (overhead_ms) *overhead_ms = res.overhead_ms;
    });
}

int slosched_exhaustive(const slosched_workload* w, const double* c, const int32_t* ids, int32_t n, int32_t max_batch,
                        int32_t n_cap, int32_t* out_ids, int32_t* out_sizes, int32_t* out_nb, int32_t* n_met,
                        double* t, double* g, uint64_t* evaluated) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        const ExhaustiveResult r = exhaustive(wl, std::vector<int>(ids, ids + n), coeffs_of(c), max_batch, n_cap);
        *out_nb = emit(r.best.schedule, out_ids, out_sizes);
        *n_met = r.best.n;
        *t = r.best.t_ms;
        *g = r.best.g;
        *evaluated = r.schedules_evaluated;
    });
}

int slosched_build_tables(const slosched_workload* w, const double* c, const int32_t* ids, int32_t n,
                          int32_t max_batch, double* exec, double* deadline) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        std::vector<double> e, d;
        cost_tables(wl, std::vector<int>(ids, ids + n), coeffs_of(c), max_batch, e, d);
        std::memcpy(exec, e.data(), e.size() * sizeof(double));
        std::memcpy(deadline, d.data(), d.size() * sizeof(double));
    });
}

int slosched_run(const slosched_workload* w, const double* c, const slosched_fleet* f, const int32_t* ids,
                 const int32_t* sizes, const int32_t* inst_nb, const slosched_sim_config* sim, double overhead_ms,
                 slosched_record* records, slosched_report* report) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        const auto fleet = fleet_of(f);
        std::vector<Schedule> plans(fleet.size());
        int pos = 0, kb = 0;
        for (std::size_t i = 0; i < fleet.size(); ++i) {
            plans[i] = schedule_of(ids + pos, sizes + kb, inst_nb[i]);
            pos += static_cast<int>(plans[i].request_count());
            kb += inst_nb[i];
        }
        const MetricsReport r = run(plans, wl, fleet, coeffs_of(c), sim_of(sim), overhead_ms);
        records_out(r.per_request, records);
        report_out(r, report);
    });
}

int slosched_run_fcfs(const slosched_workload* w, const double* c, const slosched_fleet* f,
                      const slosched_sim_config* sim, int32_t* out_ids, int32_t* out_sizes, int32_t* inst_nb,
                      slosched_record* records, slosched_report* report) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        const FcfsResult r = run_fcfs(wl, fleet_of(f), coeffs_of(c), sim_of(sim));
        int pos = 0, kb = 0;
        for (std::size_t i = 0; i < r.schedules.size(); ++i) {
            inst_nb[i] = emit(r.schedules[i], out_ids + pos, out_sizes + kb);
            pos += static_cast<int>(r.schedules[i].request_count());
            kb += inst_nb[i];
        }
        records_out(r.report.per_request, records);
        report_out(r.report, report);
    });
}

int slosched_realize_batches(const slosched_workload* w, const double* c, const int32_t* ids, const int32_t* sizes,
                             int32_t nb, double clock0, double first_gap, double gap, double until, double noise_pct,
                             uint64_t seed, int32_t from_arrival, slosched_record* records, double* clock,
                             int32_t* started) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        Rng rng(seed);
        std::vector<RequestMetrics> rec;
        const ReplayResult r = realize_batches(schedule_of(ids, sizes, nb).batches, wl, coeffs_of(c), clock0, first_gap,
                                               gap, until, noise_pct, rng, rec, from_arrival != 0);
        records_out(rec, records);
        *clock = r.clock;
        *started = r.batches_started;
    });
}

int slosched_estimator(int32_t n_classes, const int32_t* class_id, const int32_t* prior_kind, const double* prior_a,
                       const double* prior_b, int32_t n_obs, const int32_t* obs_cls, const int32_t* obs_len,
                       int32_t n_pred, const int32_t* pred_cls, uint64_t seed, int32_t* pred_out, int64_t* model_count,
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
            if (model_count) model_count[k] = m.count;
            if (model_mean) model_mean[k] = m.mean;
            if (model_m2) model_m2[k] = m.m2;
        }
        Rng rng(seed);
        for (int i = 0; i < n_pred; ++i) pred_out[i] = est.predict(pred_cls[i], rng);
    });
}

int slosched_compare(const slosched_workload* w, const double* c, const slosched_fleet* f, int32_t n_pol,
                     const int32_t* policies, int32_t n_seeds, const uint64_t* seeds, const slosched_anneal_config* cfg,
                     const slosched_sim_config* sim, int32_t exhaustive_cap, slosched_row* rows, slosched_row* medians) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        std::vector<Policy> pol;
        for (int i = 0; i < n_pol; ++i) {
            if (policies[i] < 0 || policies[i] > 2) throw DataError("compare: unknown policy code");
            pol.push_back(static_cast<Policy>(policies[i]));
        }
        const ComparisonTable t = compare(wl, fleet_of(f), coeffs_of(c), pol, std::vector<std::uint64_t>(seeds, seeds + n_seeds),
                                          config_of(cfg), sim_of(sim), exhaustive_cap);
        auto row_out = [&](const ComparisonRow& r) {
            return slosched_row{static_cast<int32_t>(parse_policy(r.policy)), r.seed, r.n_requests, r.max_batch,
                                r.attainment, r.avg_latency_ms, r.g_req_per_ms, r.overhead_ms};
        };
        for (std::size_t i = 0; i < t.rows.size(); ++i) rows[i] = row_out(t.rows[i]);
        for (std::size_t i = 0; i < t.medians.size(); ++i) medians[i] = row_out(t.medians[i]);
    });
}

int slosched_sweep(int32_t n_requests, int32_t predict_mode, int32_t n_seeds, const uint64_t* seeds,
                   const slosched_fleet* f, const double* c, const slosched_anneal_config* cfg, int32_t n_t0,
                   const double* t0_grid, int32_t n_iter, const int32_t* iter_grid, double* g_out) {
    return guarded([&] {
        std::vector<Workload> per;
        for (int s = 0; s < n_seeds; ++s) per.push_back(synth_workload(n_requests, seeds[s], predict_mode));
        const auto rows = sweep(per, std::vector<std::uint64_t>(seeds, seeds + n_seeds), fleet_of(f), coeffs_of(c),
                                config_of(cfg), std::vector<double>(t0_grid, t0_grid + n_t0),
                                std::vector<int>(iter_grid, iter_grid + n_iter));
        for (std::size_t i = 0; i < rows.size(); ++i) g_out[i] = rows[i].g_req_per_ms;
    });
}

int slosched_perturb(int32_t n_requests, int32_t predict_mode, int32_t n_seeds, const uint64_t* seeds,
                     const slosched_fleet* f, const double* truth, const slosched_anneal_config* cfg,
                     const slosched_sim_config* sim, int32_t n_params, const char* const* params, int32_t n_factors,
                     const double* factors, double* g_out, double* baseline_out, double* degradation_out) {
    return guarded([&] {
        std::vector<Workload> per;
        for (int s = 0; s < n_seeds; ++s) per.push_back(synth_workload(n_requests, seeds[s], predict_mode));
        std::vector<std::string> ps(params, params + n_params);
        const auto rows = perturb(per, std::vector<std::uint64_t>(seeds, seeds + n_seeds), fleet_of(f), coeffs_of(truth),
                                  config_of(cfg), sim_of(sim), ps, std::vector<double>(factors, factors + n_factors));
        for (std::size_t i = 0; i < rows.size(); ++i) {
            g_out[i] = rows[i].g_req_per_ms;
            baseline_out[i] = rows[i].baseline_g;
            degradation_out[i] = rows[i].degradation_pct;
        }
    });
}

int slosched_evaluate_batch(const slosched_workload* w, const double* c, int32_t n_sched, int32_t n, const int32_t* ids,
                            const int32_t* sizes, const int32_t* nb, int32_t max_batch, int32_t* n_met, double* t,
                            double* g) {
    return guarded([&] {
        const Workload wl = workload_of(w);
        std::vector<Schedule> sch(n_sched);
        int kb = 0;
        for (int s = 0; s < n_sched; ++s) {
            sch[s] = schedule_of(ids + static_cast<std::size_t>(s) * n, sizes + kb, nb[s]);
            kb += nb[s];
        }
        const auto sc = evaluate_batch(sch, coeffs_of(c), wl, max_batch);
        for (int s = 0; s < n_sched; ++s) n_met[s] = sc[s].n, t[s] = sc[s].t_ms, g[s] = sc[s].g;
    });
}

int slosched_run_online(int32_t n, const double* arrival_ms, const int32_t* cls, const int32_t* input_len,
                        const int32_t* true_out, const int32_t* pred_out, const double* c,
                        const slosched_online_config* cfg, slosched_online_result* out, double* overhead_ms,
                        int32_t overhead_cap) {
    return guarded([&] {
        if (!cfg || !out) throw std::invalid_argument("run_online: null argument");
        if (n < 0) throw DataError("run_online: negative request count");
        if (n > 0 && (!arrival_ms || !cls || !input_len || !true_out || !pred_out))
            throw std::invalid_argument("run_online: null stream array");
        if (overhead_cap > 0 && !overhead_ms) throw std::invalid_argument("run_online: null overhead_ms");
        OnlineStream st;
        st.arrival_ms.assign(arrival_ms, arrival_ms + n);
        st.cls.assign(cls, cls + n), st.input_len.assign(input_len, input_len + n);
        st.true_out.assign(true_out, true_out + n), st.pred_out.assign(pred_out, pred_out + n);
        OnlineConfig oc;
        if (cfg->policy != 0 && cfg->policy != 2) throw DataError("run_online: policy must be 0 (SA) or 2 (FCFS)");
        oc.policy = static_cast<Policy>(cfg->policy);
        oc.n_instances = cfg->n_instances, oc.window_ms = cfg->window_ms, oc.max_batch = cfg->max_batch;
        oc.budget_ms = cfg->budget_ms, oc.chains = cfg->chains, oc.chains_per_request = cfg->chains_per_request;
        oc.chains_min = cfg->chains_min, oc.seed = cfg->seed, oc.dispatch_gap_ms = cfg->dispatch_gap_ms;
        if (cfg->n_devices > 0) oc.devices.assign(cfg->devices, cfg->devices + cfg->n_devices);
        if (cfg->n_scale_ladder > 0) oc.scale_ladder.assign(cfg->scale_ladder, cfg->scale_ladder + cfg->n_scale_ladder);
        oc.t0 = cfg->t0, oc.tau = cfg->tau, oc.iter = cfg->iter, oc.deadline_start = cfg->deadline_start != 0;
        oc.max_windows = cfg->max_windows;
        const OnlineResult r = run_online(st, coeffs_of(c), oc);
        *out = slosched_online_result{r.n, r.n_met, r.total_latency_ms, r.windows, r.decisions, r.proposals};
        for (int i = 0; i < std::min<int>(overhead_cap, static_cast<int>(r.overhead_ms.size())); ++i)
            overhead_ms[i] = r.overhead_ms[i];
    });
}

}  // extern "C"
