// C++ caller of the evaluation harness (include/slosched_b200.hpp, "evaluation harness"): the
// reference's simulator / estimator / compare driver names, with the annealing on the GPU.
//
//   examples/_build/harness_example [n]
//
// Prints one line per step; exit code = number of failed checks:
//   Estimator      Welford model over observed lengths; the queue's predictions drawn from it
//   run_fcfs       the FCFS baseline replays every request
//   compare        SA (GPU chains) vs FCFS over two seeds, medians
//   evaluate_batch two schedules in one evaluator launch == evaluate(), bit for bit
//   run            the SA plans replayed on the synthetic backend
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "slosched_b200.hpp"

using namespace slosched;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 200;
    int failures = 0;
    auto check = [&](bool ok, const char* what) {
        std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
        if (!ok) ++failures;
    };
    try {
        auto [code, chat] = default_synth_classes();
        // estimator: observe realized lengths, then predict for a fresh queue
        Estimator est({code, chat});
        Rng obs(7);
        for (int i = 0; i < 500; ++i) est.observe_output(i % 2, 1 + static_cast<int>(obs.uniform_index(1500)));
        const LengthModel& m0 = est.model_for(0);
        std::printf("estimator: class 0 count=%lld mean=%.3f std=%.3f\n", m0.count, m0.mean, m0.sample_std());
        check(m0.count == 250 && m0.mean > 600.0 && m0.mean < 900.0, "Estimator Welford model");
        std::vector<Request> reqs = generate_mixed(n, 1, code, chat);
        Rng pr(Rng::derive(1, 0x9e37));
        assign_predicted_lengths(reqs, est, pr);
        const Workload w = validate_workload(reqs, {code, chat});

        std::vector<InstanceState> fleet;
        for (int i = 0; i < 3; ++i) {
            InstanceState s;
            s.id = i;
            s.total_mem = s.remaining_mem = 1ULL << 35;
            s.bytes_per_token = 262144.0;
            s.max_batch_size = 4;
            fleet.push_back(s);
        }
        const LatencyCoefficients c = table_coefficients();
        SimConfig sim;
        sim.noise_pct = 0.1;
        sim.seed = 3;
        const FcfsResult f = run_fcfs(w, fleet, c, sim);
        std::printf("run_fcfs: attainment=%.4f avg_latency_ms=%.1f g=%.6e\n", f.report.slo_attainment,
                    f.report.avg_latency_ms, f.report.g);
        check(static_cast<int>(f.report.per_request.size()) == n, "run_fcfs replays every request");

        AnnealConfig cfg;
        cfg.engine.chains = 2048;
        cfg.engine.budget_ms = 3.0;
        cfg.engine.scale_ladder = {1e3, 1e4, 1e5};
        const ComparisonTable t = compare(w, fleet, c, {Policy::SA, Policy::FCFS}, {1, 2}, cfg, sim);
        for (const auto& r : t.medians)
            std::printf("compare median %-5s attainment=%.4f avg_latency_ms=%.1f g=%.6e overhead_ms=%.2f\n",
                        r.policy.c_str(), r.attainment, r.avg_latency_ms, r.g_req_per_ms, r.overhead_ms);
        check(t.rows.size() == 4 && t.medians.size() == 2, "compare rows and medians");

        // evaluate_batch: the instance-0 plans of both seeds' SA runs, scored in one launch
        const ScheduleAllResult sa = schedule_all(w, fleet, c, cfg);
        std::vector<Schedule> plans = {sa.per_instance[0].schedule, sa.per_instance[0].schedule};
        std::reverse(plans[1].batches.begin(), plans[1].batches.end());
        const auto sc = evaluate_batch(plans, c, w, 4);
        bool eq = true;
        for (std::size_t i = 0; i < plans.size(); ++i) {
            const EvaluatedSchedule ev = evaluate(plans[i], c, w);
            eq = eq && sc[i].n == ev.n && sc[i].t_ms == ev.t_ms && sc[i].g == ev.g;
        }
        check(eq, "evaluate_batch == evaluate (bit for bit)");
        const MetricsReport rep = run({sa.per_instance[0].schedule, sa.per_instance[1].schedule,
                                       sa.per_instance[2].schedule}, w, fleet, c, sim, sa.overhead_ms);
        std::printf("run(SA plans): attainment=%.4f g=%.6e overhead_ms=%.2f\n", rep.slo_attainment, rep.g,
                    rep.scheduling_overhead_ms);
        check(rep.n_met >= 0 && static_cast<int>(rep.per_request.size()) == n, "run replays the SA plans");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 100;
    }
    std::printf("failures=%d\n", failures);
    return failures;
}
