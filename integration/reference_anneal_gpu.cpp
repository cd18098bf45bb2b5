// Reference-side binding: the file a maintainer of the reference adds next to
// P:src/priority_mapper.cpp to run anneal() on the B200 engine. It depends only on the
// reference's own headers and on the flat C ABI include/slosched_api.h (no torch, no CUDA
// headers), and links against libslosched_b200.so.
//
// anneal_gpu() has the signature of slosched::anneal (P:include/slosched/priority_mapper.hpp:67-69)
// plus the engine options; a maintainer swaps it in by making anneal() forward to it. Errors
// are rethrown as the reference's exception types (DataError / CapacityError /
// std::invalid_argument), so CLI exit codes (P:tools/slosched.cpp:668-677) are unchanged.
//
// For the parity tests this file is compiled with the unmodified reference sources into
// oracle/_ref/libslosched_refshim.so (oracle/Makefile, target refshim); refshim_anneal_gpu()
// is the extern "C" face the tests call.
#include <stdexcept>
#include <string>
#include <vector>

#include "slosched/objective.hpp"
#include "slosched/priority_mapper.hpp"
#include "slosched_api.h"

namespace slosched {

struct GpuOptions {
    int mode = 0;     // 0 = GPU chains (Philox), 1 = exact replay of the reference walk
    int chains = 4096;
    double budget_ms = 0.0;
    std::vector<double> scale_ladder;
};

AnnealResult anneal_gpu(const Workload& workload, const std::vector<int>& request_ids,
                        const LatencyCoefficients& coeffs, const AnnealConfig& config, int max_batch,
                        const GpuOptions& opt) {
    // structure-of-arrays view of the workload (ids, classes, lengths, SLOs)
    const int n_all = static_cast<int>(workload.requests.size());
    std::vector<int32_t> id(n_all), cls(n_all), in_len(n_all), true_out(n_all), pred(n_all);
    std::vector<double> arrival(n_all);
    for (int i = 0; i < n_all; ++i) {
        const Request& r = workload.requests[i];
        id[i] = r.id, cls[i] = r.task_class_id, in_len[i] = r.input_len, true_out[i] = r.true_output_len;
        pred[i] = r.predicted_output_len ? *r.predicted_output_len : -1;
        arrival[i] = r.arrival_time_ms;
    }
    const int n_cls = static_cast<int>(workload.classes.size());
    std::vector<int32_t> cid(n_cls), kind(n_cls);
    std::vector<double> e2e(n_cls, 0.0), ttft(n_cls, 0.0), tpot(n_cls, 0.0);
    for (int c = 0; c < n_cls; ++c) {
        const SloSpec& s = workload.classes[c].slo;
        cid[c] = workload.classes[c].id;
        kind[c] = s.kind == SloKind::E2E ? 0 : 1;
        if (s.e2e_ms) e2e[c] = *s.e2e_ms;
        if (s.ttft_ms) ttft[c] = *s.ttft_ms;
        if (s.tpot_ms) tpot[c] = *s.tpot_ms;
    }
    const slosched_workload view{n_all,         id.data(),   cls.data(),  in_len.data(), true_out.data(),
                                 pred.data(),   arrival.data(), n_cls,    cid.data(),    kind.data(),
                                 e2e.data(),    ttft.data(), tpot.data()};
    const double c8[8] = {coeffs.alpha_p, coeffs.beta_p, coeffs.gamma_p, coeffs.delta_p,
                          coeffs.alpha_d, coeffs.beta_d, coeffs.gamma_d, coeffs.delta_d};
    slosched_anneal_config cfg{};
    cfg.t0 = config.t0, cfg.t_thres = config.t_thres, cfg.iter = config.iter, cfg.tau = config.tau;
    cfg.seed = config.seed;
    cfg.has_objective_scale = config.objective_scale ? 1 : 0;
    cfg.objective_scale = config.objective_scale ? *config.objective_scale : 0.0;
    cfg.mode = opt.mode, cfg.chains = opt.chains, cfg.budget_ms = opt.budget_ms;
    cfg.n_scale_ladder = static_cast<int32_t>(opt.scale_ladder.size());
    cfg.scale_ladder = opt.scale_ladder.empty() ? nullptr : opt.scale_ladder.data();
    cfg.device = -1, cfg.chain_begin = 0, cfg.chain_end = -1;

    const int n = static_cast<int>(request_ids.size());
    std::vector<int32_t> ids32(request_ids.begin(), request_ids.end());
    std::vector<int32_t> out_ids(n > 0 ? n : 1), out_sizes(n > 0 ? n : 1);
    int32_t nb = 0, n_met = 0;
    double t = 0.0, g = 0.0;
    slosched_anneal_stats st{};
    const int rc = slosched_anneal(&view, c8, ids32.data(), n, &cfg, max_batch, out_ids.data(), out_sizes.data(),
                                   &nb, &n_met, &t, &g, &st);
    if (rc != 0) {
        const std::string msg = slosched_last_error();
        if (rc == 1) throw DataError(msg);
        if (rc == 2) throw CapacityError(msg);
        if (rc == 6) throw std::invalid_argument(msg);
        throw std::runtime_error("B200 engine: " + msg);
    }
    Schedule best;
    for (int k = 0, pos = 0; k < nb; ++k) {
        best.batches.emplace_back(out_ids.begin() + pos, out_ids.begin() + pos + out_sizes[k]);
        pos += out_sizes[k];
    }
    AnnealResult res;
    res.best = evaluate(best, coeffs, workload);  // the reference's own objective fills per_request
    res.stats.proposals = st.proposals;
    res.stats.accepted = st.accepted;
    res.stats.shortcut = st.shortcut != 0;
    res.stats.g_sorted_start = st.g_sorted_start;
    res.stats.g_input_start = st.g_input_start;
    res.stats.objective_scale_used = st.objective_scale_used;
    return res;
}

}  // namespace slosched

// ---------------------------------------------------------------- test face (flat arrays)
extern "C" int refshim_anneal_gpu(int n_all, const int* id, const int* cls, const int* in_len, const int* true_out,
                                  const int* pred_out, const double* arrival, int n_classes, const int* class_id,
                                  const int* kind, const double* e2e, const double* ttft, const double* tpot,
                                  const double* c, const int* ids, int n_ids, const double* cfg6, unsigned long long seed,
                                  int max_batch, int mode, int chains, int* out_ids, int* out_sizes, int* out_nb,
                                  int* n_met, double* t, double* g, double* stats2) {
    using namespace slosched;
    try {
        std::vector<TaskClass> classes;
        for (int k = 0; k < n_classes; ++k) {
            TaskClass tc;
            tc.id = class_id[k];
            tc.name = "c" + std::to_string(tc.id);
            tc.slo = kind[k] == 0 ? SloSpec::e2e(e2e[k]) : SloSpec::ttft_tpot(ttft[k], tpot[k]);
            classes.push_back(tc);
        }
        std::vector<Request> reqs;
        for (int i = 0; i < n_all; ++i) {
            Request r;
            r.id = id[i], r.task_class_id = cls[i], r.input_len = in_len[i], r.true_output_len = true_out[i];
            if (pred_out[i] >= 0) r.predicted_output_len = pred_out[i];
            r.arrival_time_ms = arrival[i];
            reqs.push_back(r);
        }
        const Workload w = validate_workload(std::move(reqs), std::move(classes));
        AnnealConfig ac;
        ac.t0 = cfg6[0], ac.t_thres = cfg6[1], ac.iter = static_cast<int>(cfg6[2]), ac.tau = cfg6[3], ac.seed = seed;
        if (cfg6[4] != 0.0) ac.objective_scale = cfg6[5];
        GpuOptions opt;
        opt.mode = mode, opt.chains = chains;
        const AnnealResult r = anneal_gpu(w, std::vector<int>(ids, ids + n_ids),
                                          {c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]}, ac, max_batch, opt);
        int pos = 0, nb = 0;
        for (const auto& b : r.best.schedule.batches) {
            out_sizes[nb++] = static_cast<int>(b.size());
            for (int x : b) out_ids[pos++] = x;
        }
        *out_nb = nb, *n_met = r.best.n, *t = r.best.t_ms, *g = r.best.g;
        stats2[0] = static_cast<double>(r.stats.proposals), stats2[1] = static_cast<double>(r.stats.accepted);
        return 0;
    } catch (const DataError&) {
        return 1;
    } catch (const CapacityError&) {
        return 2;
    } catch (const std::invalid_argument&) {
        return 6;
    } catch (const std::exception&) {
        return 9;
    }
}
