// Flat C ABI (include/slosched_api.h) over the C++ scheduler API.
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

}  // extern "C"
