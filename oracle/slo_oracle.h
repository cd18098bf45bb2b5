/* Plain-C restatement of the reference's SA scheduling hot path.
 *
 * TEST INFRASTRUCTURE ONLY: the checker the parity tests compare the CUDA path
 * against, and the "port" CPU baseline. Only tests/, __graft_entry__.smoke()
 * and bench.py's reference / cpu_baseline legs may load it. The product
 * (paper_2504_14966_b200) never links or calls it.
 *
 * Each function cites the reference file:line it restates (P: = /root/reference/proj/).
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * entry point with oracle/_ref (the unmodified reference compiled here) and
 * with the committed golden vectors in tests/golden/.
 */
#ifndef SLO_ORACLE_H
#define SLO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* xoshiro256++ seeded by splitmix64 (P:include/slosched/rng.hpp:14-100) */
typedef struct { uint64_t s[4]; } or_rng;
void or_rng_seed(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
double or_rng_uniform(or_rng* r);
uint64_t or_rng_index(or_rng* r, uint64_t n);
double or_rng_normal(or_rng* r);
uint64_t or_rng_derive(uint64_t seed, uint64_t stream);

/* latency model (P:src/latency_model.cpp:86-113); coeffs[8] = alpha_p..delta_d */
double or_predict_prefill(const double* c, int b, int li);
double or_predict_decode_total(const double* c, int b, int li, int lo);
double or_predict_exec(const double* c, int b, int li, int lo);
double or_predict_tpot(const double* c, int b, int li, int lo);

/* Flat workload: requests (pred_out < 0 means "no prediction") and SLO classes
 * (kind 0 = E2E, 1 = TTFT_TPOT), mirroring P:include/slosched/core.hpp:26-74. */
typedef struct {
    int n;
    const int *id, *cls, *in_len, *true_out, *pred_out;
    const double* arrival;
    int n_classes;
    const int *class_id, *kind;
    const double *e2e, *ttft, *tpot;
} or_workload;

/* generate_mixed + default_synth_classes (P:src/workload.cpp:138-183) and, for
 * predict_mode 1, the estimator cold-start draw from the class Gaussian prior
 * with Rng(derive(seed, 0x9e37)) (P:src/output_estimator.cpp:367-375,410-415;
 * P:tools/slosched.cpp:131-142). Class ids: 0 = code, 1 = chat. */
void or_generate_mixed(int n, uint64_t seed, int predict_mode, int* id, int* cls, int* in_len,
                       int* true_out, int* pred_out, double* arrival);

/* evaluate() (P:src/objective.cpp:55-82); per-request arrays (nullable) in
 * flattened order. Returns 0 or a negative error (-1 unknown id / missing prediction). */
int or_evaluate(const or_workload* w, const double* c, const int* ids, const int* sizes, int nb,
                int* n_met, double* t, double* g, double* wait, double* exec, double* e2e,
                double* ttft, double* tpot, int* met);

/* CostModel::score over dense-index schedules (P:src/priority_mapper.cpp:205-279):
 * tables are built for the request subset `ids`; dense index = rank of the id.
 * perms: count x n dense indices; sizes: count x n batch sizes (nb[k] used). */
int or_score_batch(const or_workload* w, const double* c, const int* ids, int n, int max_batch,
                   int count, const int* perms, const int* sizes, const int* nb, int* n_met,
                   double* t, double* g);

/* initial_candidates (P:src/priority_mapper.cpp:292-311) */
int or_initial_candidates(const or_workload* w, const double* c, const int* ids, int n, int max_batch,
                          int* sorted_ids, int* sorted_sizes, int* sorted_nb, int* input_ids,
                          int* input_sizes, int* input_nb);

/* anneal (P:src/priority_mapper.cpp:340-411). cfg = {t0, t_thres, iter, tau, has_scale, scale}.
 * stats6 = {proposals, accepted, shortcut, g_sorted, g_input, scale_used}.
 * Returns 0, -1 (unknown id / missing prediction) or -2 (bad config). */
int or_anneal(const or_workload* w, const double* c, const int* ids, int n, const double* cfg,
              uint64_t seed, int max_batch, int* out_ids, int* out_sizes, int* out_nb, int* n_met,
              double* t, double* g, double* stats6);

#ifdef __cplusplus
}
#endif

#endif
