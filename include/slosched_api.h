/* slosched_api.h -- flat C ABI of the scheduler entry points (include/slosched_b200.hpp)
 * for FFI callers (the Python package binds it with ctypes; a cgo/JNI binding would bind
 * the same symbols). Arrays in, arrays out; caller-owned buffers; int status return
 * (slo_status codes of slosched_gpu.h) with the message in slosched_last_error().
 *
 * Reference interface each function replaces (P: = /root/reference/proj/):
 *   slosched_anneal              anneal()              P:include/slosched/priority_mapper.hpp:67-69
 *   slosched_evaluate            evaluate()            P:include/slosched/objective.hpp:36-38
 *   slosched_initial_candidates  initial_candidates()  P:include/slosched/priority_mapper.hpp:46-49
 *   slosched_neighbor_walk       neighbor() x steps    P:include/slosched/priority_mapper.hpp:61
 *   slosched_schedule_all        schedule_all()        P:include/slosched/scheduler.hpp:54-59
 *   slosched_predict             predict_*()           P:include/slosched/latency_model.hpp:43-47
 *   slosched_generate_mixed      generate_mixed() + estimator cold start
 *                                                      P:include/slosched/workload.hpp:48-52
 *   slosched_build_tables        CostModel tables      P:src/priority_mapper.cpp:205-231
 */
#ifndef SLOSCHED_API_H
#define SLOSCHED_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Requests (pred_out < 0: no prediction) and SLO classes (kind 0 = E2E, 1 = TTFT_TPOT). */
typedef struct {
    int32_t n;
    const int32_t *id, *cls, *in_len, *true_out, *pred_out;
    const double* arrival;
    int32_t n_classes;
    const int32_t *class_id, *kind;
    const double *e2e, *ttft, *tpot;
} slosched_workload;

typedef struct {
    double t0, t_thres;
    int32_t iter;
    double tau;
    uint64_t seed;
    int32_t has_objective_scale;
    double objective_scale;
    int32_t mode;           /* 0 = GPU chains (Philox), 1 = exact replay of the reference walk */
    int32_t chains;
    double budget_ms;
    int32_t n_scale_ladder;
    const double* scale_ladder;
    int32_t device;         /* -1 = SLOSCHED_DEVICE or 0 */
    int32_t chain_begin, chain_end; /* chain_end < 0: all chains */
    int32_t sequential_instances;   /* schedule_all: 1 = one instance after another (default concurrent) */
    int32_t max_blocks;             /* > 0: cap the chain grid (concurrent callers share the GPU) */
    int32_t start_policy;           /* chains: 0 = best of the reference's two starts and the deadline-first
                                       candidate (default), 1 = the reference's two only */
    int32_t n_devices;              /* multi-GPU, one process: > 1 devices share the chains (slo_group) */
    const int32_t* devices;
    void* comm_ctx;                 /* multi-process: this rank's slo_ctx with an NCCL communicator
                                       (slo_ctx_comm_init); NULL otherwise */
} slosched_anneal_config;

typedef struct {
    uint64_t proposals, accepted;
    int32_t shortcut;
    double g_sorted_start, g_input_start, objective_scale_used;
    int32_t chains_run, levels_run, best_chain;
    double engine_g, engine_t, kernel_ms;
    double g_deadline_start;
    double exchange_ms;             /* multi-GPU: chain kernel end -> job-wide winner (device time) */
    int32_t devices;                /* devices whose chains the result covers */
} slosched_anneal_stats;

const char* slosched_last_error(void);

int slosched_predict(const double* coeffs8, int32_t b, int32_t input_len, int32_t output_len, double* out5);
double slosched_latest_start(double slo, double cost);

int slosched_generate_mixed(int32_t n, uint64_t seed, int32_t predict_mode, int32_t* id, int32_t* cls,
                            int32_t* in_len, int32_t* true_out, int32_t* pred_out, double* arrival);

int slosched_evaluate(const slosched_workload* w, const double* coeffs8, const int32_t* ids, const int32_t* sizes,
                      int32_t nb, int32_t* n_met, double* t, double* g, double* wait, double* exec, double* e2e,
                      double* ttft, double* tpot, int32_t* met, int32_t* extrapolated);

int slosched_initial_candidates(const slosched_workload* w, const double* coeffs8, const int32_t* ids, int32_t n,
                                int32_t max_batch, int32_t* sorted_ids, int32_t* sorted_sizes, int32_t* sorted_nb,
                                int32_t* input_ids, int32_t* input_sizes, int32_t* input_nb);

/* Engine extension (no reference counterpart): the deadline-first start of the chains. */
int slosched_deadline_first_candidate(const slosched_workload* w, const double* coeffs8, const int32_t* ids,
                                      int32_t n, int32_t max_batch, int32_t* out_ids, int32_t* out_sizes,
                                      int32_t* out_nb);

int slosched_neighbor_walk(const int32_t* ids, const int32_t* sizes, int32_t nb, uint64_t seed, int32_t steps,
                           int32_t max_batch, int32_t* out_ids, int32_t* out_sizes, int32_t* out_nb);

int slosched_anneal(const slosched_workload* w, const double* coeffs8, const int32_t* ids, int32_t n,
                    const slosched_anneal_config* cfg, int32_t max_batch, int32_t* out_ids, int32_t* out_sizes,
                    int32_t* out_nb, int32_t* n_met, double* t, double* g, slosched_anneal_stats* stats);

/* exhaustive() (P:include/slosched/priority_mapper.hpp:74-82): the GPU small-n oracle. */
int slosched_exhaustive(const slosched_workload* w, const double* coeffs8, const int32_t* ids, int32_t n,
                        int32_t max_batch, int32_t n_cap, int32_t* out_ids, int32_t* out_sizes, int32_t* out_nb,
                        int32_t* n_met, double* t, double* g, uint64_t* evaluated);

/* Instances as arrays; per-instance outputs concatenated in instance order. */
int slosched_schedule_all(const slosched_workload* w, const double* coeffs8, int32_t n_inst, const int32_t* inst_id,
                          const double* total_mem, const double* remaining_mem, const double* mu, const double* sigma,
                          const int32_t* inst_max_batch, const slosched_anneal_config* cfg, int32_t* out_ids,
                          int32_t* out_sizes, int32_t* inst_nb, int32_t* inst_count, int32_t* inst_n,
                          double* inst_t, double* inst_g, int32_t* epochs, double* overhead_ms);

/* exec[(b-1)*n + i], deadline[(b-1)*n + i] for dense index i = rank of ids[i] among ids. */
int slosched_build_tables(const slosched_workload* w, const double* coeffs8, const int32_t* ids, int32_t n,
                          int32_t max_batch, double* exec, double* deadline);

/* ---------------------------------------------------------------- evaluation harness
 * (include/slosched_b200.hpp "evaluation harness"; reference P:src/simulator.cpp:17-220,
 *  P:src/output_estimator.cpp:10-78, P:tools/slosched.cpp:297-448) */
typedef struct {
    int32_t n;
    const int32_t* id;
    const double *total_mem, *remaining_mem, *mu, *sigma;
    const int32_t* max_batch;
} slosched_fleet;

typedef struct {
    double noise_pct, dispatch_gap_ms;
    uint64_t seed;
} slosched_sim_config;

typedef struct {
    int32_t request_id;
    double wait_ms, exec_ms, e2e_ms, ttft_ms, tpot_ms;
    int32_t slo_met, extrapolated;
} slosched_record;

typedef struct {
    double slo_attainment, avg_latency_ms, g, scheduling_overhead_ms;
    int32_t n_met;
    double total_latency_ms;
} slosched_report;

typedef struct {
    int32_t policy; /* 0 sa, 1 exhaustive, 2 fcfs (Policy) */
    uint64_t seed;
    int32_t n_requests, max_batch;
    double attainment, avg_latency_ms, g_req_per_ms, overhead_ms;
} slosched_row;

/* run() P:src/simulator.cpp:49-74: per-instance schedules concatenated (inst_nb[i] batches each);
 * records in the report's order (instance by instance). */
int slosched_run(const slosched_workload* w, const double* coeffs8, const slosched_fleet* fleet, const int32_t* ids,
                 const int32_t* sizes, const int32_t* inst_nb, const slosched_sim_config* sim, double overhead_ms,
                 slosched_record* records, slosched_report* report);
/* run_fcfs() P:src/simulator.cpp:76-123: the FCFS plans (per instance, concatenated) and the report. */
int slosched_run_fcfs(const slosched_workload* w, const double* coeffs8, const slosched_fleet* fleet,
                      const slosched_sim_config* sim, int32_t* out_ids, int32_t* out_sizes, int32_t* inst_nb,
                      slosched_record* records, slosched_report* report);
/* One instance clock of the replay (realize_batches): records appended in dispatch order. */
int slosched_realize_batches(const slosched_workload* w, const double* coeffs8, const int32_t* ids,
                             const int32_t* sizes, int32_t nb, double clock0, double first_gap, double gap,
                             double until, double noise_pct, uint64_t seed, int32_t from_arrival,
                             slosched_record* records, double* clock, int32_t* batches_started);
/* Estimator P:src/output_estimator.cpp: classes with priors (kind 0 none, 1 Gaussian (a = mean,
 * b = std), 2 range (a = low, b = high)); observe n_obs (class, length) pairs in order, then predict
 * n_pred lengths with Rng(seed); the models' (count, mean, m2) after the observations. */
int slosched_estimator(int32_t n_classes, const int32_t* class_id, const int32_t* prior_kind, const double* prior_a,
                       const double* prior_b, int32_t n_obs, const int32_t* obs_cls, const int32_t* obs_len,
                       int32_t n_pred, const int32_t* pred_cls, uint64_t seed, int32_t* pred_out,
                       int64_t* model_count, double* model_mean, double* model_m2);
/* compare() P:src/simulator.cpp:148-220: rows (n_pol x n_seeds, policy-major) and medians (n_pol). */
int slosched_compare(const slosched_workload* w, const double* coeffs8, const slosched_fleet* fleet, int32_t n_pol,
                     const int32_t* policies, int32_t n_seeds, const uint64_t* seeds, const slosched_anneal_config* cfg,
                     const slosched_sim_config* sim, int32_t exhaustive_cap, slosched_row* rows, slosched_row* medians);
/* sweep / perturb drivers (P:tools/slosched.cpp:335-448) over the CLI's synthetic workload per seed
 * (generate_mixed(n, seed) + estimator priors when predict_mode = 1). sweep rows: (t0-major,
 * iter, seed); perturb rows: (param-major, factor, seed). */
int slosched_sweep(int32_t n_requests, int32_t predict_mode, int32_t n_seeds, const uint64_t* seeds,
                   const slosched_fleet* fleet, const double* coeffs8, const slosched_anneal_config* cfg, int32_t n_t0,
                   const double* t0_grid, int32_t n_iter, const int32_t* iter_grid, double* g_out);
int slosched_perturb(int32_t n_requests, int32_t predict_mode, int32_t n_seeds, const uint64_t* seeds,
                     const slosched_fleet* fleet, const double* truth8, const slosched_anneal_config* cfg,
                     const slosched_sim_config* sim, int32_t n_params, const char* const* params, int32_t n_factors,
                     const double* factors, double* g_out, double* baseline_out, double* degradation_out);
/* n / t / g of n_sched schedules over the same requests (ids: n_sched x n; inst-style batch counts
 * nb[s]; sizes concatenated) in one launch of the bit-exact evaluator (K1). */
int slosched_evaluate_batch(const slosched_workload* w, const double* coeffs8, int32_t n_sched, int32_t n,
                            const int32_t* ids, const int32_t* sizes, const int32_t* nb, int32_t max_batch,
                            int32_t* n_met, double* t, double* g);

/* run_online (include/slosched_b200.hpp "online rescheduling"): the stream as arrays (arrival
 * order), the result and up to overhead_cap per-window planning times (ms). policy: 0 SA, 2 FCFS. */
typedef struct {
    int32_t policy, n_instances;
    double window_ms;
    int32_t max_batch;
    double budget_ms;
    int32_t chains, chains_per_request, chains_min;
    uint64_t seed;
    double dispatch_gap_ms;
    int32_t n_devices;
    const int32_t* devices;
    int32_t n_scale_ladder;
    const double* scale_ladder;
    double t0, tau;
    int32_t iter, deadline_start, max_windows;
} slosched_online_config;

typedef struct {
    int32_t n, n_met;
    double total_latency_ms;
    int32_t windows, decisions;
    uint64_t proposals;
} slosched_online_result;

int slosched_run_online(int32_t n, const double* arrival_ms, const int32_t* cls, const int32_t* input_len,
                        const int32_t* true_out, const int32_t* pred_out, const double* coeffs8,
                        const slosched_online_config* cfg, slosched_online_result* out, double* overhead_ms,
                        int32_t overhead_cap);

#ifdef __cplusplus
}
#endif

#endif
