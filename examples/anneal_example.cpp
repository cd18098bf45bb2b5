// C++ caller of the B200 scheduler through the reference-shaped API (include/slosched_b200.hpp):
// the same types and entry points a reference user writes against (P:include/slosched/*.hpp).
//
//   build: python -m paper_2504_14966_b200.build   (also builds examples/_build/anneal_example)
//   run:   examples/_build/anneal_example [n]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "slosched_b200.hpp"

int main(int argc, char** argv) {
    using namespace slosched;
    const int n = argc > 1 ? std::atoi(argv[1]) : 1024;
    // the reference CLI's synthetic pipeline: generate_mixed + estimator cold start (P:tools/slosched.cpp:119-142)
    auto [code, chat] = default_synth_classes();
    std::vector<Request> reqs = generate_mixed(n, 0, code, chat);
    Rng rng(Rng::derive(0, 0x9e37));
    assign_predicted_lengths_from_priors(reqs, {code, chat}, rng);
    const Workload w = validate_workload(reqs, {code, chat});
    std::vector<int> ids;
    for (const auto& r : w.requests) ids.push_back(r.id);
    const LatencyCoefficients coeffs = table_coefficients();

    try {
        // GPU chains at a 10 ms scheduling budget
        AnnealConfig cfg;
        cfg.engine.chains = 16384;
        cfg.engine.budget_ms = 9.5;
        cfg.engine.scale_ladder = {1e4, 1e5, 1e6, 1e7, 1e8};
        const AnnealResult res = anneal(w, ids, coeffs, cfg, 4);
        std::printf("chains: n_met=%d g=%.9e t=%.6e proposals=%llu kernel_ms=%.3f chains=%d\n", res.best.n,
                    res.best.g, res.best.t_ms, (unsigned long long)res.stats.proposals, res.stats.kernel_ms,
                    res.stats.chains_run);

        // the reference's own walk, bit-for-bit (default AnnealConfig, seed 0)
        AnnealConfig rc;
        rc.engine.mode = SearchMode::Replay;
        const AnnealResult rep = anneal(w, ids, coeffs, rc, 4);
        std::printf("replay: n_met=%d g=%.9e proposals=%llu accepted=%llu\n", rep.best.n, rep.best.g,
                    (unsigned long long)rep.stats.proposals, (unsigned long long)rep.stats.accepted);

        // Algorithm 2 over four instances (per-instance anneals run concurrently on the GPU)
        std::vector<InstanceState> fleet;
        for (int i = 0; i < 4; ++i) {
            InstanceState s;
            s.id = i;
            s.total_mem = s.remaining_mem = 1ULL << 35;
            s.bytes_per_token = 262144.0;
            s.max_batch_size = 4;
            fleet.push_back(s);
        }
        AnnealConfig sc;
        sc.engine.chains = 2048;
        sc.engine.budget_ms = 2.0;
        const ScheduleAllResult all = schedule_all(w, fleet, coeffs, sc);
        int met = 0;
        for (const auto& ev : all.per_instance) met += ev.n;
        std::printf("schedule_all: instances=%zu n_met=%d overhead_ms=%.3f\n", all.per_instance.size(), met,
                    all.overhead_ms);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
