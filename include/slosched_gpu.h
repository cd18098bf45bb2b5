/* slosched_gpu.h -- C ABI of the B200 annealing engine (hand-written sm_100a CUDA).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * This is the layer the C++ scheduler entry point (include/slosched_b200.hpp,
 * slosched::anneal) calls into, and what an FFI binding (ctypes / cgo / JNI)
 * would bind directly. P: = reference tree /root/reference/proj/.
 *
 * What each entry point replaces in the reference:
 *   slo_problem_set     CostModel ctor, P:src/priority_mapper.cpp:205-231 (flat exec/prefill/
 *                       tpot tables per (dense index, batch size)); here the tables are
 *                       (exec, deadline) pairs in a structure-of-arrays HBM layout.
 *   slo_evaluate_batch  CostModel::score, P:src/priority_mapper.cpp:259-279 (identical operand
 *                       order to evaluate(), P:src/objective.cpp:55-82): one candidate per
 *                       thread, bit-exact n_met / t / g.
 *   slo_anneal_chains   the annealing loop of anneal(), P:src/priority_mapper.cpp:368-402:
 *                       SLO_RNG_XOSHIRO_REPLAY reproduces the reference walk bit-for-bit
 *                       (FlatSchedule moves :104-199, Rng P:include/slosched/rng.hpp:14-100);
 *                       SLO_RNG_PHILOX runs thousands of independent chains (one per warp),
 *                       each move scored from the batches it rebuilds on an integer tick
 *                       grid (slo_problem_tick_ms), plus a grid-wide best-of-chains argmax.
 *
 * Conventions: every function returns an slo_status; on failure slo_last_error()
 * (thread-local) holds the message. No exceptions cross the ABI. Output buffers are
 * caller-owned. A context is owned by one host thread at a time.
 *
 * Deadline convention (makes the SLO test one compare, bit-exact): for dense index i
 * and batch size b, deadline[b-1][i] is the largest double d such that a request whose
 * batch starts at elapsed = d meets its SLO under the reference arithmetic:
 *   E2E:       fl(d + exec) <= e2e_ms                       (P:src/priority_mapper.cpp:238)
 *   TTFT_TPOT: fl(d + prefill) <= ttft_ms, and -inf when tpot > tpot_ms   (:239-240)
 * fl(d + c) is monotone in d, so "met" == (elapsed <= deadline) exactly.
 */
#ifndef SLOSCHED_GPU_H
#define SLOSCHED_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLO_MAX_N 4096 /* 12-bit dense index per position */
#define SLO_MAX_MB 16  /* 4-bit batch-size field; moves touch <= 2*mb <= 32 positions */

typedef enum {
    SLO_OK = 0,
    SLO_ERR_DATA = 1,     /* reference DataError */
    SLO_ERR_CAPACITY = 2, /* reference CapacityError / size limits of this engine */
    SLO_ERR_CUDA = 3,
    SLO_ERR_COMM = 4,
    SLO_ERR_STATE = 5,    /* call order (e.g. no problem set) */
    SLO_ERR_ARG = 6       /* reference std::invalid_argument */
} slo_status;

typedef enum { SLO_RNG_PHILOX = 0, SLO_RNG_XOSHIRO_REPLAY = 1 } slo_rng_mode;

typedef struct slo_ctx slo_ctx;

const char* slo_last_error(void);
const char* slo_version(void);

/* One context per device; owns a stream, the device tables and chain buffers. */
int slo_ctx_create(int device, slo_ctx** out);
void slo_ctx_destroy(slo_ctx* ctx);
/* The cudaStream_t every launch of this context is enqueued on. */
void* slo_ctx_stream(slo_ctx* ctx);
int slo_ctx_sync(slo_ctx* ctx);
/* Number of streaming multiprocessors of the context's device. */
int slo_ctx_sm_count(slo_ctx* ctx);

/* Upload the per-(batch size, dense index) tables: exec[(b-1)*n + i], deadline[(b-1)*n + i].
 * 1 <= n <= SLO_MAX_N, 1 <= mb <= SLO_MAX_MB. */
int slo_problem_set(slo_ctx* ctx, int32_t n, int32_t mb, const double* exec, const double* deadline);

/* The chain kernel (K3) scores schedules exactly in integer "ticks" of 2^-k ms: exec times rounded
 * to that grid, deadlines compared on it. Returns the tick (ms) of the current problem, 0 if none. */
double slo_problem_tick_ms(slo_ctx* ctx);

/* Bit-exact objective of `count` candidate schedules. perms[c*n + p] = dense index at
 * position p; batch_end_bits[c*words + w] bit (p & 31) of word w = (p >> 5) set iff p is the
 * last position of its batch (words = ceil(n/32); bit n-1 must be set). Host buffers. */
int slo_evaluate_batch(slo_ctx* ctx, int32_t count, const uint16_t* perms,
                       const uint32_t* batch_end_bits, int32_t* n_met, double* t, double* g);

/* The chain kernel's own objective of `count` candidates (same layout as slo_evaluate_batch):
 * n_met bit-exact with CostModel::score -- the tick grid decides an SLO test only where its
 * rounding bound certifies it, the rest is re-summed in the reference's fp64 order -- and t (g)
 * on the grid, within 2^-26 relative of the reference's. exact_walks (may be NULL) receives
 * the number of 32-position units decided by the fp64 re-sum. Needs finite exec times
 * (negative ones are valid: the grid is offset, makespans start at 0 as in the reference). */
int slo_evaluate_batch_tick(slo_ctx* ctx, int32_t count, const uint16_t* perms,
                            const uint32_t* batch_end_bits, int32_t* n_met, double* t, double* g,
                            uint64_t* exact_walks);

typedef struct {
    double t0, t_thres; /* AnnealConfig (P:include/slosched/priority_mapper.hpp:16-28) */
    int32_t iter;
    double tau;
    uint64_t seed;
    double objective_scale;  /* resolved factor (reference :368-370 default t0 / G(start)) */
    int32_t rng_mode;        /* slo_rng_mode */
    int32_t chains;          /* total chains of the whole job (all devices) */
    int32_t chain_begin;     /* this call runs chain ids [chain_begin, chain_end) */
    int32_t chain_end;
    int64_t budget_ns;       /* 0 = run the whole ladder; else stop after this much device time */
    int32_t n_scale_mult;    /* optional per-chain scale ladder: chain c uses */
    const double* scale_mult;/*   objective_scale * scale_mult[c % n_scale_mult] */
    int32_t max_blocks;      /* > 0: cap the chain grid (share the GPU with concurrent launches) */
} slo_chain_params;

typedef struct {
    double g;            /* best score found (chain kernel: n_met exact, t on the 2^-k ms tick grid) */
    double t;            /* its summed latency (ticks x tick) */
    int32_t n_met;
    int32_t chain;       /* winning chain id (ties: lower t, then lower id) */
    uint64_t proposals;  /* summed over the chains run */
    uint64_t accepted;
    int32_t chains_run;  /* chains that started */
    int32_t levels_run;  /* temperature levels completed by the slowest chain */
    float kernel_ms;     /* device time of the annealing launches (CUDA events) */
    uint64_t positions_pass1; /* Philox mode: positions of the rebuilt batches scored */
    uint64_t positions_pass2; /*   and positions re-walked for SLO counts (replay: 0) */
    uint64_t exact_walks;     /* Philox mode: 32-position unit walks the tick grid could not certify,
                                 decided by the reference's fp64 arithmetic (n_met is always the
                                 reference's) */
    float exchange_ms;        /* multi-device: device time from the end of the chain kernel to the
                                 job-wide winner (argmax + slot pack + all-gather + pick); 0 otherwise */
    int32_t nranks;           /* devices whose chains the result covers (1 without an exchange) */
    uint64_t local_proposals; /* this device's share of proposals / positions_pass1 / positions_pass2 */
    uint64_t local_positions_pass1, local_positions_pass2;
} slo_chain_result;

/* Run chains from the start schedule (dense indices in position order + batch sizes) and
 * return the best schedule found, in the same form. Synchronous. */
int slo_anneal_chains(slo_ctx* ctx, const slo_chain_params* params, const int32_t* start_perm,
                      const int32_t* start_sizes, int32_t start_nb, int32_t* best_perm,
                      int32_t* best_sizes, int32_t* best_nb, slo_chain_result* result);

/* Split form for device-resident timing: prepare uploads the start state (H2D) and
 * parameters; launch only enqueues the annealing kernel and the argmax on the context
 * stream (no host synchronisation, no copies); fetch synchronises and copies the winner
 * back. slo_anneal_chains == prepare + launch + fetch. */
int slo_chains_prepare(slo_ctx* ctx, const slo_chain_params* params, const int32_t* start_perm,
                       const int32_t* start_sizes, int32_t start_nb);
int slo_chains_launch(slo_ctx* ctx);
int slo_chains_fetch(slo_ctx* ctx, int32_t* best_perm, int32_t* best_sizes, int32_t* best_nb,
                     slo_chain_result* result);

/* ---------------------------------------------------------------- multi-GPU
 * Chains shard across devices by global chain id (each chain's moves depend only on the seed and
 * its id, so the sharded job runs the same chains as one device would); after every device's
 * best-of-chains one device-side exchange -- an NCCL all-gather of one slot per device (header +
 * winner state), then an on-device pick in the k_argmax order -- leaves the job-wide winner on
 * every device. Nothing crosses the host between the chain kernel and the winner.
 * Replaces: nothing in the reference (one CPU chain per instance, P:src/scheduler.cpp:109-123). */
#define SLO_COMM_ID_BYTES 128

/* Multi-process (one rank per GPU): rank 0 creates the id, the launcher distributes it (e.g.
 * torch.distributed), every rank attaches it to its context (ncclCommInitRank; collective).
 * Afterwards slo_chains_launch also enqueues the exchange, slo_chains_fetch returns the job-wide
 * winner on every rank (chain ids global), and a rank may be given an empty slice
 * (chain_begin == chain_end). */
int slo_comm_unique_id(uint8_t id[SLO_COMM_ID_BYTES]);
int slo_ctx_comm_init(slo_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t id[SLO_COMM_ID_BYTES]);
int slo_ctx_comm_info(slo_ctx* ctx, int32_t* nranks, int32_t* rank);
/* A rank that cannot run its slice (an error before its launch) still takes part in the
 * exchange with an empty slot (n: the job's request count, which fixes the slot size), so the
 * other ranks are not left waiting in the collective. Collective. */
int slo_ctx_exchange_empty(slo_ctx* ctx, int32_t n);
/* ncclCommGetAsyncError of the attached communicator (SLO_ERR_COMM on a failed peer). */
int slo_comm_check(slo_ctx* ctx);

/* Single process, several devices: one context (stream) per listed device and one NCCL
 * communicator over them (ncclCommInitAll). A device listed twice cannot join an NCCL
 * communicator; such groups (and SLOSCHED_EXCHANGE=peer) gather the slots with peer copies
 * onto member 0 instead (transport "peer"). */
typedef struct slo_group slo_group;
int slo_group_create(int32_t ndev, const int32_t* devices, slo_group** out);
void slo_group_destroy(slo_group* group);
int32_t slo_group_size(slo_group* group);
slo_ctx* slo_group_ctx(slo_group* group, int32_t i);
const char* slo_group_transport(slo_group* group);  /* "nccl" or "peer" */
/* slo_problem_set on every member (host threads in parallel). */
int slo_group_problem_set(slo_group* group, int32_t n, int32_t mb, const double* exec, const double* deadline);
/* slo_anneal_chains over the group: chain ids [chain_begin, chain_end < 0 ? chains : chain_end)
 * split into contiguous balanced slices, one per member; Philox mode only. kernel_ms is the
 * slowest member's. Synchronous. */
int slo_group_anneal_chains(slo_group* group, const slo_chain_params* params, const int32_t* start_perm,
                            const int32_t* start_sizes, int32_t start_nb, int32_t* best_perm,
                            int32_t* best_sizes, int32_t* best_nb, slo_chain_result* result);

/* Exhaustive search of the current problem: every permutation x every ordered batch-size
 * composition with parts <= mb, one candidate stream per thread, best by the reference's order
 * (G desc, t asc, flattened ids, composition) -- P:src/priority_mapper.cpp:440-517. Fails with
 * SLO_ERR_CAPACITY when n > n_cap (reference message) or n > 16. Outputs the winner in dense
 * indices, its G and t, and the number of schedules evaluated (n! x compositions). */
int slo_exhaustive(slo_ctx* ctx, int32_t n_cap, int32_t* best_perm, int32_t* best_sizes, int32_t* best_nb,
                   double* g, double* t, uint64_t* evaluated);

/* Achievable shared-memory bandwidth of the device (GB/s): conflict-free 16-byte loads on
 * every SM -- the roofline denominator of the smem-bound chain kernel. */
int slo_probe_smem_bandwidth(slo_ctx* ctx, double* gbytes_per_s);

/* Philox4x32-10 (Random123 constants) -- the counter-based stream the chains draw from;
 * exported for known-answer tests. */
void slo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif

#endif
