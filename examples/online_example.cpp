// C++ caller of the online driver (include/slosched_b200.hpp, "online driver"): a Poisson stream of
// the reference's synthetic requests over k instances, re-planned every window on the GPU.
//
//   examples/_build/online_example [n] [instances]
//
// Prints one line per policy and the checks; exit code = number of failed checks:
//   every request is served under both policies
//   the GPU chains meet at least as many SLOs as FCFS
//   one planning-overhead entry per window
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "slosched_b200.hpp"

using namespace slosched;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 1500;
    const int k = argc > 2 ? std::atoi(argv[2]) : 2;
    int failures = 0;
    auto check = [&](bool ok, const char* what) {
        std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
        if (!ok) ++failures;
    };
    try {
        auto [code, chat] = default_synth_classes();
        std::vector<Request> reqs = generate_mixed(n, 4, code, chat);
        Rng prior(5);
        assign_predicted_lengths_from_priors(reqs, {code, chat}, prior);
        // Poisson arrivals at 0.9 of the fleet's capacity (~0.21 requests/s per instance)
        OnlineStream st;
        Rng rng(11);
        double t = 0.0;
        const double rate_per_ms = 0.9 * k * 0.21 / 1000.0;
        for (const Request& r : reqs) {
            t += -std::log(1.0 - rng.uniform()) / rate_per_ms;
            st.arrival_ms.push_back(t);
            st.cls.push_back(r.task_class_id), st.input_len.push_back(r.input_len);
            st.true_out.push_back(r.true_output_len), st.pred_out.push_back(*r.predicted_output_len);
        }
        const LatencyCoefficients c = table_coefficients();
        OnlineConfig cfg;
        cfg.n_instances = k;
        cfg.budget_ms = 5.0;
        cfg.chains = 1024;
        cfg.policy = Policy::SA;
        const OnlineResult sa = run_online(st, c, cfg);
        cfg.policy = Policy::FCFS;
        const OnlineResult fc = run_online(st, c, cfg);
        double mean = 0.0;
        for (double x : sa.overhead_ms) mean += x;
        mean /= sa.overhead_ms.empty() ? 1.0 : static_cast<double>(sa.overhead_ms.size());
        std::printf("sa:   attainment=%.4f windows=%d decisions=%d proposals=%llu planning %.3f ms/window\n",
                    sa.n_met / static_cast<double>(sa.n), sa.windows, sa.decisions,
                    static_cast<unsigned long long>(sa.proposals), mean);
        std::printf("fcfs: attainment=%.4f windows=%d\n", fc.n_met / static_cast<double>(fc.n), fc.windows);
        check(sa.n == n && fc.n == n, "every request served");
        check(sa.n_met >= fc.n_met, "GPU chains meet at least FCFS's SLOs");
        check(static_cast<int>(sa.overhead_ms.size()) == sa.windows, "one planning entry per window");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 100;
    }
    std::printf("failures=%d\n", failures);
    return failures;
}
