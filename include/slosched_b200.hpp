// slosched_b200.hpp -- C++ entry points of the B200 SLO-aware scheduler.
//
// Drop-in for the reference's scheduling path: the same namespace, type names, member
// names and function signatures as the reference headers (P: = /root/reference/proj/):
//   domain types            P:include/slosched/core.hpp:15-170
//   Rng                     P:include/slosched/rng.hpp:14-100
//   latency model           P:include/slosched/latency_model.hpp:41-59
//   objective               P:include/slosched/objective.hpp:13-38
//   priority mapper         P:include/slosched/priority_mapper.hpp:16-82
//   scheduler               P:include/slosched/scheduler.hpp:16-59
//   synthetic workload      P:include/slosched/workload.hpp:23-55 (generator subset)
//   estimator (cold start)  P:include/slosched/output_estimator.hpp:10-56 (subset)
// so code written against slosched::anneal / schedule_all / evaluate compiles against
// this header and runs the annealing loop on the GPU (include/slosched_gpu.h).
//
// Extensions (all defaulted so reference call sites are unchanged) live in
// AnnealConfig::engine and AnnealStats; see DESIGN.md.
#ifndef SLOSCHED_B200_HPP
#define SLOSCHED_B200_HPP

#include <cstdint>
#include <deque>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <variant>
#include <vector>

struct slo_ctx;  // include/slosched_gpu.h

namespace slosched {

// ---------------------------------------------------------------- errors
class DataError : public std::runtime_error {
public:
    explicit DataError(const std::string& w) : std::runtime_error(w) {}
};
class CapacityError : public std::runtime_error {
public:
    explicit CapacityError(const std::string& w) : std::runtime_error(w) {}
};
// CUDA / engine failures: there is no CPU fallback.
class EngineError : public std::runtime_error {
public:
    explicit EngineError(const std::string& w) : std::runtime_error(w) {}
};

// ---------------------------------------------------------------- domain
enum class SloKind { E2E, TTFT_TPOT };

struct SloSpec {
    SloKind kind = SloKind::E2E;
    std::optional<double> e2e_ms, ttft_ms, tpot_ms;
    static SloSpec e2e(double ms);
    static SloSpec ttft_tpot(double ttft_ms, double tpot_ms);
    void validate() const;
};

struct GaussianPrior {
    double mean_tokens = 0.0, std_tokens = 0.0;
};
struct RangePrior {
    int low = 1, high = 1;
};
using OutputPrior = std::variant<std::monostate, GaussianPrior, RangePrior>;

struct TaskClass {
    int id = 0;
    std::string name;
    SloSpec slo;
    OutputPrior output_prior;
    void validate() const;
};

struct Request {
    int id = 0;
    int task_class_id = 0;
    int input_len = 1;
    int true_output_len = 1;
    std::optional<int> predicted_output_len;
    double arrival_time_ms = 0.0;
    void validate() const;
};

struct LatencyCoefficients {
    double alpha_p = 0.0, beta_p = 0.0, gamma_p = 0.0, delta_p = 0.0;
    double alpha_d = 0.0, beta_d = 0.0, gamma_d = 0.0, delta_d = 0.0;
    void validate() const;
};

using Batch = std::vector<int>;

struct Schedule {
    std::vector<Batch> batches;
    std::size_t request_count() const;
    std::vector<int> flatten() const;
    std::unordered_map<int, std::pair<int, int>> positions() const;
    bool is_partition_of(const std::vector<int>& ids, int max_batch) const;
};

struct InstanceState {
    int id = 0;
    std::uint64_t total_mem = 0, remaining_mem = 0;
    double mem_utility = 0.9, bytes_per_token = 1.0;
    int max_batch_size = 1;
    void validate() const;
};

struct RequestMetrics {
    int request_id = 0;
    double wait_ms = 0.0, exec_ms = 0.0, e2e_ms = 0.0, ttft_ms = 0.0, tpot_ms = 0.0;
    bool slo_met = false;
    bool extrapolated = false;
};

struct EvaluatedSchedule {
    Schedule schedule;
    std::vector<RequestMetrics> per_request;
    int n = 0;
    double t_ms = 0.0;
    double g = 0.0;
};

struct Workload {
    std::vector<TaskClass> classes;
    std::vector<Request> requests;
    const TaskClass& class_of(const Request& r) const;
    const TaskClass* find_class(int class_id) const;
    const Request* find_request(int request_id) const;

private:
    friend Workload validate_workload(std::vector<Request>, std::vector<TaskClass>);
    std::unordered_map<int, std::size_t> class_index_, request_index_;
    // request ids spanning a small range (the common case) index a flat table instead of the
    // hash map: position + 1 at id - dense_lo_, 0 where no request has that id
    long long dense_lo_ = 0;
    std::vector<std::uint32_t> dense_;
};

Workload validate_workload(std::vector<Request> requests, std::vector<TaskClass> classes);

// ---------------------------------------------------------------- rng
// xoshiro256++ seeded by splitmix64; same streams as the reference Rng.
class Rng {
public:
    explicit Rng(std::uint64_t seed);
    std::uint64_t next_u64();
    double uniform();
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    std::uint64_t uniform_index(std::uint64_t n);
    long long uniform_int(long long lo, long long hi) {
        return lo + static_cast<long long>(uniform_index(static_cast<std::uint64_t>(hi - lo + 1)));
    }
    double normal();
    double normal(double mean, double sd) { return mean + sd * normal(); }
    template <typename T>
    void shuffle(std::vector<T>& v) {
        for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[uniform_index(i)]);
    }
    static std::uint64_t derive(std::uint64_t seed, std::uint64_t stream);

private:
    std::uint64_t s_[4];
};

// ---------------------------------------------------------------- latency model
double predict_prefill(const LatencyCoefficients& c, int b, int input_len);
double predict_per_token_decode(const LatencyCoefficients& c, int b, int accumulated_len);
double predict_decode_total(const LatencyCoefficients& c, int b, int input_len, int output_len);
double predict_exec(const LatencyCoefficients& c, int b, int input_len, int output_len);
double predict_tpot(const LatencyCoefficients& c, int b, int input_len, int output_len);
constexpr int kValidatedMaxLen = 2047;
inline bool is_extrapolated(int input_len, int output_len) { return input_len + output_len > kValidatedMaxLen; }
LatencyCoefficients table_coefficients();

// ---------------------------------------------------------------- objective
struct ExecProfile {
    int request_id = 0;
    double exec_ms = 0.0, prefill_ms = 0.0, tpot_ms = 0.0;
    bool extrapolated = false;
};
std::vector<ExecProfile> batch_exec_profile(const Schedule&, const LatencyCoefficients&, const Workload&);
std::vector<double> waiting_times(const Schedule&, const std::vector<ExecProfile>&);
bool meets_slo(const SloSpec& slo, double e2e_ms, double ttft_ms, double tpot_ms);
EvaluatedSchedule evaluate(const Schedule&, const LatencyCoefficients&, const Workload&);

// ---------------------------------------------------------------- priority mapper
enum class SearchMode {
    Chains,  // thousands of independent Philox chains on the GPU, best-of-chains (default)
    Replay,  // one chain driven by the reference's xoshiro stream: bit-identical to the reference
};

struct EngineOptions {
    SearchMode mode = SearchMode::Chains;
    int chains = 4096;                  // Chains mode: total chains
    double budget_ms = 0.0;             // > 0: stop the ladder after this much device time
    std::vector<double> scale_ladder;   // per-chain objective_scale multipliers (chain c uses [c % size])
    int device = -1;                    // -1: SLOSCHED_DEVICE env or 0
    int chain_begin = 0, chain_end = -1;  // slice of [0, chains) run by this call (multi-GPU sharding)
    int max_blocks = 0;                 // > 0: cap the chain grid (concurrent launches share the GPU)
    bool concurrent_instances = true;   // schedule_all: anneal the instances concurrently (Chains mode)
    bool deadline_start = true;         // Chains mode: the deadline-first candidate joins the two starts
    // multi-GPU (Chains mode; see include/slosched_gpu.h). The chains [chain_begin, chain_end) of
    // one call shard across devices and one device-side exchange picks the job-wide best:
    std::vector<int> devices;           // > 1 entry: this process drives all of them (slo_group, NCCL);
                                        //   1 entry: that device (overrides `device`)
    ::slo_ctx* comm_ctx = nullptr;      // one rank of a multi-process job: a context with an NCCL
                                        //   communicator (slo_ctx_comm_init); chain_end < 0 runs this
                                        //   rank's balanced share of `chains`
};

struct AnnealConfig {
    double t0 = 500.0;
    double t_thres = 20.0;
    int iter = 100;
    double tau = 0.95;
    std::uint64_t seed = 0;
    std::optional<double> objective_scale;
    EngineOptions engine;
    void validate() const;
};

struct AnnealStats {
    std::uint64_t proposals = 0;
    std::uint64_t accepted = 0;
    bool shortcut = false;
    double g_sorted_start = 0.0;
    double g_input_start = 0.0;
    double objective_scale_used = 1.0;
    // engine extensions
    int chains_run = 0;
    int levels_run = 0;
    int best_chain = -1;
    double engine_g = 0.0;    // best score as computed on the device
    double engine_t = 0.0;    // its summed latency (tie-break of the best-of-chains argmax)
    double kernel_ms = 0.0;   // device time of the annealing launch
    double g_deadline_start = 0.0;  // G of the deadline-first candidate (Chains mode; 0 if not built)
    double exchange_ms = 0.0; // multi-GPU: device time from the chain kernel's end to the job-wide winner
    int devices = 1;          // devices whose chains the result covers
};

struct AnnealResult {
    EvaluatedSchedule best;
    AnnealStats stats;
};

std::pair<Schedule, Schedule> initial_candidates(const Workload&, const std::vector<int>& request_ids,
                                                 const LatencyCoefficients&, int max_batch);
// Engine extension: a third start for the chains. Requests are taken in order of their latest
// feasible start (full batches); a request joins the kept set -- held in ascending exec order and
// cut into batches of max_batch -- when every kept request still starts in time, otherwise the
// longest kept request is dropped (Moore-Hodgson with batching). Kept batches run first, the
// rest follow shortest first.
Schedule deadline_first_candidate(const Workload&, const std::vector<int>& request_ids, const LatencyCoefficients&,
                                  int max_batch);
std::optional<EvaluatedSchedule> shortcut_check(const Schedule& sorted_schedule, const LatencyCoefficients&,
                                                const Workload&);
Schedule neighbor(const Schedule& schedule, Rng& rng, int max_batch);
AnnealResult anneal(const Workload&, const std::vector<int>& request_ids, const LatencyCoefficients&,
                    const AnnealConfig&, int max_batch);

struct ExhaustiveResult {
    EvaluatedSchedule best;
    std::uint64_t schedules_evaluated = 0;
};

// Small-n oracle on the GPU: every permutation x every ordered batch-size composition with
// parts <= max_batch; ties broken by lower t, then lexicographic request order, then batch-size
// sequence (P:include/slosched/priority_mapper.hpp:74-82). CapacityError when n > n_cap.
ExhaustiveResult exhaustive(const Workload& workload, const std::vector<int>& request_ids,
                            const LatencyCoefficients& coeffs, int max_batch, int n_cap = 10);

// Largest d with fl(d + c) <= s (the deadline convention of include/slosched_gpu.h).
double latest_start(double s, double c);

// The engine tables for a request set: exec[(b-1)*n + i] and deadline[(b-1)*n + i] for
// dense index i = rank of the id among `ids` (CostModel, P:src/priority_mapper.cpp:205-231).
void cost_tables(const Workload& w, const std::vector<int>& ids, const LatencyCoefficients& c, int max_batch,
                 std::vector<double>& exec, std::vector<double>& deadline);

// ---------------------------------------------------------------- scheduler
long long token_capacity(std::uint64_t remaining_mem_bytes, double mu, double sigma);

struct AssignmentResult {
    std::vector<std::vector<int>> per_instance;
    int epochs = 1;
};
AssignmentResult assign_instances(const Workload&, const std::vector<InstanceState>&, const LatencyCoefficients&);

enum class Policy { SA, EXHAUSTIVE, FCFS };

struct InstanceQueue {
    std::deque<Batch> pending;
};
std::optional<Batch> dispatch(InstanceQueue& queue, bool instance_ready);

struct ScheduleAllResult {
    AssignmentResult assignment;
    std::vector<EvaluatedSchedule> per_instance;
    std::vector<AnnealStats> stats;
    std::vector<InstanceQueue> queues;
    double overhead_ms = 0.0;
};
ScheduleAllResult schedule_all(const Workload&, const std::vector<InstanceState>&, const LatencyCoefficients&,
                               const AnnealConfig&, Policy policy = Policy::SA, int exhaustive_cap = 10);

// ---------------------------------------------------------------- output-length estimator
// (P:include/slosched/output_estimator.hpp:10-56) Welford running Gaussian per task class; the
// scheduler consumes its predictions as Request::predicted_output_len.
constexpr int kDefaultOutputLen = 256;

struct LengthModel {
    int task_class_id = 0;
    long long count = 0;
    double mean = 0.0;
    double m2 = 0.0;  // sum of squared deviations from the running mean
    OutputPrior prior;
    double sample_variance() const;
    double sample_std() const;
};
void observe(LengthModel& model, int actual_len);
int predict_len(const LengthModel& model, Rng& rng);
int simulate_predictor_error(int true_len, double error_pct, Rng& rng);

class Estimator {
public:
    explicit Estimator(const std::vector<TaskClass>& classes);
    LengthModel& model_for(int task_class_id);
    const std::vector<LengthModel>& models() const { return models_; }
    void observe_output(int task_class_id, int actual_len);
    int predict(int task_class_id, Rng& rng);

private:
    std::vector<LengthModel> models_;
};
void assign_predicted_lengths(std::vector<Request>& requests, Estimator& estimator, Rng& rng);

// ---------------------------------------------------------------- evaluation harness
// (P:include/slosched/core.hpp:139-150, P:include/slosched/simulator.hpp:13-72,
//  P:tools/slosched.cpp:297-448) The realized-attainment replay, the FCFS baseline and the
// compare / sweep / perturb drivers, with the annealing on the GPU (schedule_all) and the
// sweep's scoring batched through the bit-exact evaluator (K1).
struct MetricsReport {
    double slo_attainment = 0.0;
    double avg_latency_ms = 0.0;
    double g = 0.0;
    double scheduling_overhead_ms = 0.0;
    std::vector<RequestMetrics> per_request;
    int n_met = 0;
    double total_latency_ms = 0.0;
    static MetricsReport from_records(std::vector<RequestMetrics> records, double overhead_ms);
};

struct SimConfig {
    double noise_pct = 0.0;        // uniform multiplicative execution noise
    double dispatch_gap_ms = 0.1;  // interval between consecutive batch dispatches
    std::uint64_t seed = 0;
};

MetricsReport run(const std::vector<Schedule>& schedules, const Workload& workload,
                  const std::vector<InstanceState>& instances, const LatencyCoefficients& coeffs,
                  const SimConfig& sim_cfg, double scheduling_overhead_ms = 0.0);

struct FcfsResult {
    MetricsReport report;
    std::vector<Schedule> schedules;
};
FcfsResult run_fcfs(const Workload& workload, const std::vector<InstanceState>& instances,
                    const LatencyCoefficients& coeffs, const SimConfig& sim_cfg);

struct ComparisonRow {
    std::string policy;
    std::uint64_t seed = 0;
    int n_requests = 0;
    int max_batch = 0;
    double attainment = 0.0;
    double avg_latency_ms = 0.0;
    double g_req_per_ms = 0.0;
    double overhead_ms = 0.0;
};
struct ComparisonTable {
    std::vector<ComparisonRow> rows;
    std::vector<ComparisonRow> medians;
};
double median(std::vector<double> values);
std::string policy_name(Policy p);
Policy parse_policy(const std::string& name);
ComparisonTable compare(const Workload& workload, const std::vector<InstanceState>& instances,
                        const LatencyCoefficients& coeffs, const std::vector<Policy>& policies,
                        const std::vector<std::uint64_t>& seeds, const AnnealConfig& anneal_cfg,
                        const SimConfig& sim_cfg, int exhaustive_cap = 10);

// One instance clock of the replay: batch 0 starts at clock0 + first_gap, batch j > 0 at the
// previous batch's end + gap; no batch starts once the clock (before its gap) has reached `until`.
// Records (wait = start - arrival when from_arrival, else start) are appended; returns the clock
// and the number of batches started. run() is this from clock 0 with no first gap and no bound;
// the online driver replays each window with it.
struct ReplayResult {
    double clock = 0.0;
    int batches_started = 0;
};
ReplayResult realize_batches(const std::vector<Batch>& batches, const Workload& workload,
                             const LatencyCoefficients& coeffs, double clock0, double first_gap, double gap,
                             double until,
                             double noise_pct, Rng& rng, std::vector<RequestMetrics>& records,
                             bool from_arrival = false);

// Engine extension: n / t / g of many schedules over the same request set in one launch of the
// bit-exact evaluator (K1; == evaluate() bit for bit).
struct ScheduleScore {
    int n = 0;
    double t_ms = 0.0, g = 0.0;
};
std::vector<ScheduleScore> evaluate_batch(const std::vector<Schedule>& schedules, const LatencyCoefficients& coeffs,
                                          const Workload& workload, int max_batch, int device = -1);

// sweep / perturb drivers (P:tools/slosched.cpp:335-448): one workload per seed. Every cell's
// schedule_all runs concurrently on the GPU (a share of the SMs each; chain results do not depend
// on the grid, so the rows equal one-after-another runs).
struct SweepRow {
    double t0 = 0.0;
    int iter = 0;
    std::uint64_t seed = 0;
    double g_req_per_ms = 0.0;
};
std::vector<SweepRow> sweep(const std::vector<Workload>& per_seed, const std::vector<std::uint64_t>& seeds,
                            const std::vector<InstanceState>& instances, const LatencyCoefficients& coeffs,
                            const AnnealConfig& base_cfg, const std::vector<double>& t0_grid,
                            const std::vector<int>& iter_grid);
struct PerturbRow {
    std::string param;
    double factor = 1.0;
    std::uint64_t seed = 0;
    double g_req_per_ms = 0.0, baseline_g = 0.0, degradation_pct = 0.0;
};
std::vector<PerturbRow> perturb(const std::vector<Workload>& per_seed, const std::vector<std::uint64_t>& seeds,
                                const std::vector<InstanceState>& instances, const LatencyCoefficients& truth,
                                const AnnealConfig& base_cfg, const SimConfig& sim_cfg,
                                const std::vector<std::string>& params, const std::vector<double>& factors);

// ---------------------------------------------------------------- online rescheduling
// (engine extension, BASELINE configs[4]; the reference has no online mode) A request
// stream (arrival order) served by n_instances instances: arrivals join the least-loaded
// instance, every window_ms each instance's queue is re-planned -- GPU chains under the window's
// budget (SLOs less the time already waited), or FCFS -- and run on the replay until the next
// window boundary. Stream classes: 0 = code (E2E 30 s), 1 = chat (TTFT 10 s + TPOT 50 ms).
struct OnlineStream {
    std::vector<double> arrival_ms;
    std::vector<int> cls, input_len, true_out, pred_out;
};
struct OnlineConfig {
    Policy policy = Policy::SA;          // SA (GPU chains) or FCFS
    int n_instances = 8;
    double window_ms = 5000.0;
    int max_batch = 4;
    double budget_ms = 10.0;             // per window, all instances' planning together
    int chains = 4096;                   // per plan at most; in proportion to the queue:
    int chains_per_request = 64, chains_min = 256;
    std::uint64_t seed = 0;
    double dispatch_gap_ms = 0.1;
    std::vector<int> devices;            // instance i on devices[i % size] (empty: the default device)
    std::vector<double> scale_ladder = {1.0, 10.0, 100.0, 1000.0, 1e4, 1e5};
    double t0 = 500.0, tau = 0.7;
    int iter = 30;
    bool deadline_start = false;
    int max_windows = -1;                // < 0: until every request has started
};
struct OnlineResult {
    int n = 0, n_met = 0;
    double total_latency_ms = 0.0;
    int windows = 0, decisions = 0;
    std::uint64_t proposals = 0;
    std::vector<double> overhead_ms;     // wall time of each window's planning
};
OnlineResult run_online(const OnlineStream& stream, const LatencyCoefficients& coeffs, const OnlineConfig& cfg);

// ---------------------------------------------------------------- synthetic inputs
struct LengthDists {
    double code_input_median = 300.0, code_input_sigma = 0.5;
    double code_output_mean = 900.0, code_output_std = 300.0;
    double chat_input_median = 200.0, chat_input_sigma = 0.5;
    double chat_output_mean = 250.0, chat_output_std = 150.0;
};
std::pair<TaskClass, TaskClass> default_slo_classes();
std::pair<TaskClass, TaskClass> default_synth_classes(const LengthDists& dists = {});
std::vector<Request> generate_mixed(int n, std::uint64_t seed, const TaskClass& code_class,
                                    const TaskClass& chat_class, const LengthDists& dists = {});
// Estimator cold start: draw predicted_output_len from each class prior (Gaussian or
// range; 256 without a prior) for requests that lack one.
void assign_predicted_lengths_from_priors(std::vector<Request>& requests, const std::vector<TaskClass>& classes,
                                          Rng& rng);

}  // namespace slosched

#endif
