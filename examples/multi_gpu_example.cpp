// Multi-GPU check of the C++ entry point (include/slosched_b200.hpp): the same anneal() call with
// the chains sharded over several engine contexts must return exactly the schedule one context
// returns over the same global chain ids (chain moves depend only on the seed and the chain id).
//
//   examples/_build/multi_gpu_example [n]
//
// Cases (each prints one PASS/FAIL line; exit code = number of failures):
//   group {0}      one device through slo_group: NCCL communicator with ndev = 1 (ncclCommInitAll)
//   group {0,0}    two contexts on one GPU: peer-copy exchange onto member 0
//   group {0..k-1} every visible device (k >= 2 only): NCCL over NVLink
//   schedule_all   instances placed one per device (round robin over the device list)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "slosched_b200.hpp"
#include "slosched_gpu.h"

using namespace slosched;

namespace {

int failures = 0;

void check(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++failures;
}

bool same(const AnnealResult& a, const AnnealResult& b) {
    return a.best.schedule.batches == b.best.schedule.batches && a.best.g == b.best.g && a.best.n == b.best.n &&
           a.stats.best_chain == b.stats.best_chain && a.stats.engine_g == b.stats.engine_g &&
           a.stats.proposals == b.stats.proposals && a.stats.chains_run == b.stats.chains_run;
}

}  // namespace

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 512;
    auto [code, chat] = default_synth_classes();
    std::vector<Request> reqs = generate_mixed(n, 3, code, chat);
    Rng rng(Rng::derive(3, 0x9e37));
    assign_predicted_lengths_from_priors(reqs, {code, chat}, rng);
    const Workload w = validate_workload(reqs, {code, chat});
    std::vector<int> ids;
    for (const auto& r : w.requests) ids.push_back(r.id);
    const LatencyCoefficients coeffs = table_coefficients();

    try {
        AnnealConfig cfg;  // full ladder, no budget: the work is fixed, so results are comparable
        cfg.seed = 11;
        cfg.t0 = 200.0;
        cfg.iter = 40;
        cfg.engine.chains = 3001;  // odd: the slices differ in size
        cfg.engine.scale_ladder = {1.0, 1e3, 1e5};
        cfg.engine.devices = {0};
        const AnnealResult one = anneal(w, ids, coeffs, cfg, 4);
        std::printf("one context: n_met=%d g=%.9e chain=%d proposals=%llu\n", one.best.n, one.best.g,
                    one.stats.best_chain, (unsigned long long)one.stats.proposals);

        AnnealConfig two = cfg;
        two.engine.devices = {0, 0};
        const AnnealResult r2 = anneal(w, ids, coeffs, two, 4);
        check(same(one, r2) && r2.stats.devices == 2, "group {0,0} (peer exchange) == one context");
        std::printf("  exchange_ms=%.4f kernel_ms=%.3f\n", r2.stats.exchange_ms, r2.stats.kernel_ms);

        AnnealConfig three = cfg;
        three.engine.devices = {0, 0, 0};
        check(same(one, anneal(w, ids, coeffs, three, 4)), "group {0,0,0} (peer exchange) == one context");

        // one-device NCCL communicator through the C ABI directly
        {
            int dev0 = 0;
            slo_group* g = nullptr;
            int rc = slo_group_create(1, &dev0, &g);
            check(rc == SLO_OK && std::string(slo_group_transport(g)) == "nccl", "slo_group_create {0}: nccl");
            if (rc == SLO_OK) {
                std::vector<double> ex, dl;
                std::vector<int> sorted = ids;
                std::sort(sorted.begin(), sorted.end());
                cost_tables(w, sorted, coeffs, 4, ex, dl);
                rc = slo_group_problem_set(g, n, 4, ex.data(), dl.data());
                // start: the greedy sorted candidate in dense indices
                auto [s_sched, i_sched] = initial_candidates(w, ids, coeffs, 4);
                std::vector<int> sp, ss;
                for (const auto& b : s_sched.batches) {
                    ss.push_back((int)b.size());
                    for (int id : b) sp.push_back((int)(std::lower_bound(sorted.begin(), sorted.end(), id) - sorted.begin()));
                }
                slo_chain_params p{};
                p.t0 = 200.0, p.t_thres = 20.0, p.iter = 40, p.tau = 0.95, p.seed = 11, p.objective_scale = 1e7;
                p.rng_mode = SLO_RNG_PHILOX, p.chains = 1000, p.chain_begin = 0, p.chain_end = 1000;
                std::vector<int> bp(n), bs(n), bp1(n), bs1(n);
                int nb = 0, nb1 = 0;
                slo_chain_result r{}, r1{};
                if (rc == SLO_OK) rc = slo_group_anneal_chains(g, &p, sp.data(), ss.data(), (int)ss.size(), bp.data(),
                                                               bs.data(), &nb, &r);
                slo_ctx* c = nullptr;
                if (rc == SLO_OK) rc = slo_ctx_create(0, &c);
                if (rc == SLO_OK) rc = slo_problem_set(c, n, 4, ex.data(), dl.data());
                if (rc == SLO_OK) rc = slo_anneal_chains(c, &p, sp.data(), ss.data(), (int)ss.size(), bp1.data(),
                                                         bs1.data(), &nb1, &r1);
                if (rc != SLO_OK) std::printf("  error: %s\n", slo_last_error());
                check(rc == SLO_OK && bp == bp1 && nb == nb1 && r.g == r1.g && r.chain == r1.chain &&
                          r.proposals == r1.proposals && r.nranks == 1,
                      "slo_group {0} (NCCL all-gather, ndev=1) == slo_anneal_chains");
                std::printf("  nccl exchange_ms=%.4f\n", r.exchange_ms);
                slo_ctx_destroy(c);
                slo_group_destroy(g);
            }
        }

        int ndev = 0;
        {  // every visible device: NCCL over NVLink (multi-GPU boxes only)
            std::vector<int> all;
            for (int d = 0; d < 64; ++d) {
                slo_ctx* c = nullptr;
                if (slo_ctx_create(d, &c) != SLO_OK) break;
                slo_ctx_destroy(c);
                all.push_back(d);
            }
            ndev = (int)all.size();
            if (ndev >= 2) {
                AnnealConfig m = cfg;
                m.engine.devices = all;
                const AnnealResult rm = anneal(w, ids, coeffs, m, 4);
                check(same(one, rm) && rm.stats.devices == ndev, "group {all devices} (NCCL) == one context");
            } else {
                std::printf("SKIP group {all devices}: %d device(s) visible\n", ndev);
            }
        }

        // schedule_all with instances placed over a device list (here: two slots on GPU 0)
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
        sc.engine.chains = 1024;
        sc.t0 = 100.0, sc.iter = 20;
        const ScheduleAllResult base = schedule_all(w, fleet, coeffs, sc);
        AnnealConfig sp = sc;
        sp.engine.devices = {0, 0};
        const ScheduleAllResult placed = schedule_all(w, fleet, coeffs, sp);
        bool eq = base.per_instance.size() == placed.per_instance.size();
        for (std::size_t i = 0; eq && i < base.per_instance.size(); ++i)
            eq = base.per_instance[i].schedule.batches == placed.per_instance[i].schedule.batches &&
                 base.per_instance[i].g == placed.per_instance[i].g;
        check(eq, "schedule_all over a device list == schedule_all on one device");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 100;
    }
    std::printf("failures=%d\n", failures);
    return failures;
}
