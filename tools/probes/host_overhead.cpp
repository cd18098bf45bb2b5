// Host-side cost of one anneal() call, phase by phase (tools/probes; built by hand):
//   g++ -std=c++17 -O2 -Iinclude tools/probes/host_overhead.cpp -o tools/probes/host_overhead \
//       -Lpaper_2504_14966_b200 -lslosched_b200 -Wl,-rpath,$PWD/paper_2504_14966_b200
// Prints the wall of the public anneal() (n = 6 and 1024, a one-level single-chain search, so the
// kernel is negligible) and of each engine call it makes.
#include <chrono>
#include <cstdio>
#include <vector>

#include "slosched_b200.hpp"
#include "slosched_gpu.h"

using namespace slosched;
using clk = std::chrono::steady_clock;

static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

int main() {
    const LatencyCoefficients c = table_coefficients();
    for (int n : {6, 32, 1024, 4096}) {
        auto [code, chat] = default_synth_classes();
        std::vector<Request> reqs = generate_mixed(n, 1, code, chat);
        for (auto& r : reqs) r.predicted_output_len = r.true_output_len;  // (predictions do not matter here)
        const Workload w = validate_workload(reqs, {code, chat});
        std::vector<int> ids;
        for (const auto& r : w.requests) ids.push_back(r.id);
        AnnealConfig a;
        a.t0 = 21.0, a.t_thres = 20.0, a.iter = 1;
        a.engine.chains = 1;
        for (int rep = 0; rep < 3; ++rep) anneal(w, ids, c, a, 4);
        const int R = 50;
        auto t0 = clk::now();
        for (int rep = 0; rep < R; ++rep) anneal(w, ids, c, a, 4);
        auto t1 = clk::now();
        std::printf("n=%d anneal() %.3f ms per call\n", n, ms(t0, t1) / R);
        {  // host pieces of anneal()
            std::vector<double> ex0, dl0;
            double tc = 0, ti = 0, te = 0, td = 0, ta = 0;
            for (int rep = 0; rep < R; ++rep) {
                auto b0 = clk::now();
                cost_tables(w, ids, c, 4, ex0, dl0);
                auto b1 = clk::now();
                auto cand = initial_candidates(w, ids, c, 4);
                auto b2 = clk::now();
                EvaluatedSchedule e1 = evaluate(cand.first, c, w);
                auto b3 = clk::now();
                Schedule d = deadline_first_candidate(w, ids, c, 4);
                auto b4 = clk::now();
                AnnealConfig a2 = a;
                a2.engine.deadline_start = true;
                anneal(w, ids, c, a2, 4);
                auto b5 = clk::now();
                tc += ms(b0, b1), ti += ms(b1, b2), te += ms(b2, b3), td += ms(b3, b4), ta += ms(b4, b5);
            }
            std::printf("n=%d cost_tables %.3f  initial_candidates %.3f  evaluate %.3f  deadline_first %.3f  "
                        "anneal(+deadline start) %.3f ms\n", n, tc / R, ti / R, te / R, td / R, ta / R);
        }
        // the engine calls alone
        std::vector<double> ex, dl;
        cost_tables(w, ids, c, 4, ex, dl);
        slo_ctx* ctx = nullptr;
        slo_ctx_create(0, &ctx);
        std::vector<int32_t> perm(n), sizes, bp(n), bs(n);
        for (int i = 0; i < n; ++i) perm[i] = i;
        for (int left = n; left > 0; left -= 4) sizes.push_back(left < 4 ? left : 4);
        slo_chain_params prm{};
        prm.t0 = 21.0, prm.t_thres = 20.0, prm.iter = 1, prm.tau = 0.5, prm.objective_scale = 1.0;
        prm.rng_mode = SLO_RNG_PHILOX, prm.chains = 1, prm.chain_begin = 0, prm.chain_end = 1;
        int32_t nb = 0;
        slo_chain_result cr{};
        double tp = 0, tq = 0, tl = 0, tf = 0;
        for (int rep = 0; rep < R + 3; ++rep) {
            auto a0 = clk::now();
            slo_problem_set(ctx, n, 4, ex.data(), dl.data());
            auto a1 = clk::now();
            slo_chains_prepare(ctx, &prm, perm.data(), sizes.data(), (int)sizes.size());
            auto a2 = clk::now();
            slo_chains_launch(ctx);
            auto a3 = clk::now();
            slo_chains_fetch(ctx, bp.data(), bs.data(), &nb, &cr);
            auto a4 = clk::now();
            if (rep >= 3) tp += ms(a0, a1), tq += ms(a1, a2), tl += ms(a2, a3), tf += ms(a3, a4);
        }
        std::printf("n=%d problem_set %.3f  prepare %.3f  launch %.3f  fetch %.3f ms (kernel %.3f)\n", n, tp / R,
                    tq / R, tl / R, tf / R, cr.kernel_ms);
        slo_ctx_destroy(ctx);
    }
    return 0;
}
