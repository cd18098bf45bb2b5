// B200 annealing engine: hand-written sm_100a kernels behind include/slosched_gpu.h.
//
// Data layout:
//   * Tables: HBM structure-of-arrays exec[mb][n], deadline[mb][n] (uploaded by
//     slo_problem_set). One device pass (k_tables) derives the exact pair table
//     tab[mb][n] = {exec, deadline} (16 B, for K1, K2 and the exhaustive oracle) and the chain
//     kernel's tick tables: xt[mb][n] (u32 exec ticks | +inf-deadline flag, staged into shared
//     memory by every CTA of K3 with coalesced 16-byte loads) and dt[mb][n] (int64 deadline ticks).
//   * Chain state (one chain per warp, shared memory): 16-bit position entries
//     ent[q] = (batch_size-1) * n + dense_index (the table index itself), a linear batch-end
//     bitmask (bit q set iff q ends its batch) and two move-flag bitmasks (K3).
//
// Kernels:
//   k_eval_exact   K1: one candidate per thread, sequential reference arithmetic.
//   k_replay       K2: one chain per warp, xoshiro256++ and FlatSchedule moves, exact.
//   k_start<U>     K3 prologue: the shared start state's unit anchors and move flags.
//   k_chains<U>    K3: one chain per warp, Philox4x32-10 moves, tick-exact delta objective.
//   k_argmax       K4: best-of-chains (g desc, t asc, chain asc) + winner copy.
// P: = /root/reference/proj/.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "slosched_gpu.h"

namespace {

thread_local std::string g_err;

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t kTagMove = 0x5105c4edu;   // Philox counter word 3 for move draws

struct ChainRec {
    double g;      // best score of the chain (-1 = never started)
    double t;      // summed latency of the best
    double cur_f;  // current working score (multi-chain-per-warp state save)
    double best_f; // best working score (K3 state save; g is its exact counterpart)
    long long cur_tot;  // current total latency in ticks (K3 state save)
    int cur_A, cur_n;   // current +inf-deadline count and SLO count (K3 state save)
    int n_met;
    int levels;
    unsigned long long proposals;
    unsigned long long accepted;
    unsigned long long scan1, scan2;  // positions walked by pass 1 / pass 2 (roofline accounting)
};

struct ChainResult {
    double g, t;
    int n_met, chain;
    unsigned long long proposals, accepted;
    int chains_run, levels_min;
    unsigned long long scan1, scan2;
};

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Philox4x32-10, Random123 constants.
#ifndef SLO_PHILOX_ROUNDS
#define SLO_PHILOX_ROUNDS 10
#endif
// One round = two 32x32->64 products: written as one wide multiply each (IMAD.WIDE.U32: both
// halves from one instruction) instead of __umulhi + a low multiply (IMAD.HI + IMAD).
template <int R = 10>
__host__ __device__ __forceinline__ void philox_rounds(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        c[0] = n0, c[1] = (uint32_t)p1, c[2] = n2, c[3] = (uint32_t)p0;
        k0 += 0x9E3779B9u, k1 += 0xBB67AE85u;
    }
}

__device__ __forceinline__ uint32_t lemire32(uint32_t x, uint32_t n) { return __umulhi(x, n); }

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max

// first set bit at or after q (bit n-1 is always set, batches <= 16 long)
__device__ __forceinline__ int next_end(const uint32_t* bits, int q) {
    int w = q >> 5;
    uint32_t m = bits[w] & (FULL << (q & 31));
    while (!m) m = bits[++w];
    return (w << 5) + __ffs(m) - 1;
}

// last set bit strictly before q, or -1
__device__ __forceinline__ int prev_end(const uint32_t* bits, int q) {
    if (q <= 0) return -1;
    int w = q >> 5;
    uint32_t m = bits[w] & ((1u << (q & 31)) - 1u);
    while (!m && w > 0) m = bits[--w];
    return m ? (w << 5) + 31 - __clz(m) : -1;
}

// ================================================================ K1: exact evaluate
// Sequential CostModel::score (P:src/priority_mapper.cpp:259-279) per candidate.
// Candidates are validated here, not on the host: bit n-1 must end a batch, batches hold at most
// mb positions, indices are below n (error bits 1 / 2 / 4 in *err; the candidate is not scored).
__global__ void k_eval_exact(int count, int n, int mb, int words, const uint16_t* __restrict__ perms,
                             const uint32_t* __restrict__ bits, const double2* __restrict__ tab,
                             int* __restrict__ n_met, double* __restrict__ t_out, double* __restrict__ g_out,
                             int* __restrict__ err) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    const uint16_t* pr = perms + (size_t)c * n;
    const uint32_t* br = bits + (size_t)c * words;
    if (!((br[(n - 1) >> 5] >> ((n - 1) & 31)) & 1u)) {
        atomicOr(err, 1);
        return;
    }
    double elapsed = 0.0, total = 0.0;
    int met = 0, s = 0;
    while (s < n) {
        const int e = next_end(br, s);
        const int bidx = e - s;
        if (bidx >= mb) {
            atomicOr(err, 2);
            return;
        }
        double makespan = 0.0;
        for (int q = s; q <= e; ++q) {
            const int i = pr[q];
            if (i >= n) {
                atomicOr(err, 4);
                return;
            }
            const double2 v = __ldg(&tab[bidx * n + i]);
            const double e2e = elapsed + v.x;
            total += e2e;
            met += elapsed <= v.y;
            makespan = dmax(makespan, v.x);
        }
        elapsed += makespan;
        s = e + 1;
    }
    n_met[c] = met;
    t_out[c] = total;
    g_out[c] = total > 0.0 ? (double)met / total : 0.0;
}

// ================================================================ K3: chains
#include "chains.cuh"

// ================================================================ K5: chains, short queues
#include "chains_small.cuh"

// ================================================================ K2: exact replay
#include "replay.cuh"

// ================================================================ exhaustive oracle
#include "exhaustive.cuh"

// ================================================================ K4: argmax
__device__ __forceinline__ bool better(double g, double t, int c, double bg, double bt, int bc) {
    if (g != bg) return g > bg;
    if (t != bt) return t < bt;
    return c < bc;
}

__global__ void k_argmax(int chain_count, const ChainRec* __restrict__ rec, ChainResult* out, int ent_words,
                         int bit_words, const uint16_t* best_ent, const uint32_t* best_bits, uint16_t* win_ent,
                         uint32_t* win_bits) {
    __shared__ double sg[512], st[512];
    __shared__ int sc[512], slev[512], sn[512];
    __shared__ unsigned long long sp[512], sa[512], s1[512], s2[512];
    const int tid = threadIdx.x;
    double bg = -2.0, bt = 0.0;
    int bc = 0x7fffffff, lev = 0x7fffffff, started = 0;
    unsigned long long props = 0, accs = 0, sc1 = 0, sc2 = 0;
    for (int c = tid; c < chain_count; c += blockDim.x) {
        const ChainRec r = rec[c];
        if (r.levels > 0) {  // chain started (budget may stop chains before level 0)
            ++started;
            lev = min(lev, r.levels);
            props += r.proposals, accs += r.accepted, sc1 += r.scan1, sc2 += r.scan2;
            if (better(r.g, r.t, c, bg, bt, bc)) bg = r.g, bt = r.t, bc = c;
        }
    }
    sg[tid] = bg, st[tid] = bt, sc[tid] = bc, slev[tid] = lev, sn[tid] = started, sp[tid] = props, sa[tid] = accs;
    s1[tid] = sc1, s2[tid] = sc2;
    __syncthreads();
    for (int s = blockDim.x >> 1; s; s >>= 1) {
        if (tid < s) {
            const int o = tid + s;
            if (better(sg[o], st[o], sc[o], sg[tid], st[tid], sc[tid])) sg[tid] = sg[o], st[tid] = st[o], sc[tid] = sc[o];
            slev[tid] = min(slev[tid], slev[o]);
            sn[tid] += sn[o], sp[tid] += sp[o], sa[tid] += sa[o], s1[tid] += s1[o], s2[tid] += s2[o];
        }
        __syncthreads();
    }
    const int win = sc[0];
    if (win >= chain_count) {
        if (tid == 0) out->chain = -1, out->chains_run = 0, out->proposals = 0;
        return;
    }
    if (tid == 0) {
        out->g = sg[0], out->t = st[0], out->chain = win, out->n_met = rec[win].n_met;
        out->proposals = sp[0], out->accepted = sa[0], out->chains_run = sn[0];
        out->levels_min = slev[0] == 0x7fffffff ? 0 : slev[0];
        out->scan1 = s1[0], out->scan2 = s2[0];
    }
    for (int i = tid; i < ent_words; i += blockDim.x) win_ent[i] = best_ent[(size_t)win * ent_words + i];
    for (int i = tid; i < bit_words; i += blockDim.x) win_bits[i] = best_bits[(size_t)win * bit_words + i];
}

// shared-memory bandwidth probe: conflict-free 16-byte loads (4 wavefronts per warp load)
__global__ void __launch_bounds__(1024) k_smem_probe(int iters, uint4* sink) {
    extern __shared__ uint4 sbuf[];
    constexpr int kVec = 4096;  // 64 KiB
    for (int i = threadIdx.x; i < kVec; i += blockDim.x) sbuf[i] = make_uint4(i, i * 3, i * 5, i * 7);
    __syncthreads();
    uint4 acc = make_uint4(0, 0, 0, 0);
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int k = 0; k < 8; ++k) {
            const uint4 v = sbuf[(idx + k * 128) & (kVec - 1)];
            acc.x ^= v.x, acc.y ^= v.y, acc.z ^= v.z, acc.w ^= v.w;
        }
        idx += 1024;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9e3779b9u) sink[threadIdx.x] = acc;
}

// interleave the SoA tables into {exec, deadline} pairs (K1, K2, exhaustive) and build the
// tick tables of K3: exec rounded to the 2^-k ms grid (| kAlways where the deadline is +inf) and
// deadline ticks floor(D * 2^k) (-1 where no elapsed time >= 0 meets it)
__global__ void k_tables(int total, const double* exec, const double* dl, double scale, int cofs, double2* tab,
                         uint32_t* xt, long long* dt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const double e = exec[i], d = dl[i];
    tab[i] = make_double2(e, d);
    const bool always = d == INFINITY;
    xt[i] = (uint32_t)(__double2ll_rn(e * scale) + cofs) | (always ? kAlways : 0u);
    dt[i] = always || !(d >= 0.0) ? -1ll : (long long)fmin(floor(d * scale), 0x1.0p62);
}

// ------------------------------------------------------------------ host side
#define CK(call)                                                                  \
    do {                                                                          \
        cudaError_t e_ = (call);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            g_err = std::string(#call) + ": " + cudaGetErrorString(e_);           \
            return SLO_ERR_CUDA;                                                  \
        }                                                                         \
    } while (0)

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// units of 32 positions per lane: 1 (n <= 1024), 2 (<= 2048), 4 (<= 4096)
int pick_upl(int n) {
    const int units = (n + 31) / 32;
    return units <= 32 ? 1 : (units <= 64 ? 2 : 4);
}

// exchange.cuh
void comm_destroy(void* comm);
int ex_reserve(slo_ctx* c, int nslots);
int ex_pack(slo_ctx* c);
int ex_allgather(slo_ctx* c);
int ex_pick(slo_ctx* c, int nslots);
int ex_local_counts(slo_ctx* c, unsigned long long out[3]);  // async D2H on the stream

}  // namespace

struct slo_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int sm_count = 0;
    size_t smem_optin = 0;
    int n = 0, mb = 0;
    DevBuf tab, exec_soa, dl_soa, xt, dt;
    double tick = 1.0;   // K3 grid: 2^-k ms
    long long dg = -1;   // K3: largest finite deadline in ticks
    long long marg = 0;  // K3: ticks within which the grid cannot certify an SLO test
    bool exec_finite = true;
    int cofs = 0;        // K3: exec tick offset (> 0 only when some exec is negative)
    // chains
    DevBuf st_ent, st_bits, st_sum, best_ent, best_bits, rec, start_ent, start_bits, start_sum, start_obj, scale_mult,
        result, win_ent, win_bits, exact_count;
    // K1 (and the K3 evaluator)
    DevBuf e_perms, e_bits, e_n, e_t, e_g, e_err, e_cnt;
    bool prepared = false;
    slo_chain_params prm{};
    int UPL = 1, grid = 0, block = 0, levels = 0, chain_count = 0;
    size_t smem = 0;
    bool smem_tab = false;
    bool small = false;  // K5 (n <= 32) instead of K3
    double replay_scale = 0.0;
    int start_nb = 0;
    ChainParams kp{};
    ReplayParams rp{};
    // cross-device exchange (exchange.cuh)
    void* comm = nullptr;        // ncclComm_t: slo_ctx_comm_init (multi-process) or slo_group_create
    bool own_comm = false;
    int nranks = 1, rank = 0;
    slo_group* group = nullptr;  // member of a single-process group (the group drives the exchange)
    DevBuf ex_slot, ex_gather;
    size_t ex_slot_bytes = 0;
    bool exchanged = false;      // result / win_* hold the job-wide winner (global chain id)
    bool empty_slice = false;    // this rank runs no chain (fewer chains than ranks)
    cudaEvent_t ev2 = nullptr, ev_pack = nullptr;
};

extern "C" {

const char* slo_last_error(void) { return g_err.c_str(); }
const char* slo_version(void) { return "slosched_b200 engine 0.1 (sm_100a)"; }

void slo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    philox_rounds<10>(c, key[0], key[1]);
    for (int i = 0; i < 4; ++i) out[i] = c[i];
}

}  // extern "C"
namespace {
void prewarm_kernels(slo_ctx* c);
}
extern "C" {

int slo_ctx_create(int device, slo_ctx** out) {
    if (!out) return fail(SLO_ERR_ARG, "slo_ctx_create: null out");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(SLO_ERR_ARG, "slo_ctx_create: no such device");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(SLO_ERR_CUDA, std::string("slo_ctx_create: need an sm_100 device, got ") + prop.name);
    auto* c = new slo_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev2);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        delete c;
        return fail(SLO_ERR_CUDA, std::string("slo_ctx_create: ") + cudaGetErrorString(e));
    }
    prewarm_kernels(c);
    *out = c;
    return SLO_OK;
}

void slo_ctx_destroy(slo_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->comm && c->own_comm) comm_destroy(c->comm);
    cudaEventDestroy(c->ev0);
    cudaEventDestroy(c->ev1);
    cudaEventDestroy(c->ev2);
    cudaEventDestroy(c->ev_pack);
    cudaStreamDestroy(c->stream);
    delete c;
}

void* slo_ctx_stream(slo_ctx* c) { return c ? (void*)c->stream : nullptr; }
int slo_ctx_sm_count(slo_ctx* c) { return c ? c->sm_count : 0; }

int slo_ctx_sync(slo_ctx* c) {
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->stream));
    return SLO_OK;
}

int slo_problem_set(slo_ctx* c, int32_t n, int32_t mb, const double* exec, const double* deadline) {
    if (!c) return fail(SLO_ERR_ARG, "slo_problem_set: null context");
    if (n < 1 || n > SLO_MAX_N) return fail(SLO_ERR_CAPACITY, "slo_problem_set: n must be in [1, 4096]");
    if (mb < 1) return fail(SLO_ERR_DATA, "slo_problem_set: max_batch must be >= 1");
    if (mb > SLO_MAX_MB) return fail(SLO_ERR_CAPACITY, "slo_problem_set: max_batch must be <= 16");
    CK(cudaSetDevice(c->device));
    const size_t total = (size_t)n * mb;
    CK(c->tab.reserve(total * sizeof(double2)));
    CK(c->exec_soa.reserve(total * sizeof(double)));
    CK(c->dl_soa.reserve(total * sizeof(double)));
    CK(c->xt.reserve(total * sizeof(uint32_t)));
    CK(c->dt.reserve(total * sizeof(long long)));
    // K3 tick grid: the largest power of two 2^k with (max exec - min(min exec, 0)) * 2^k below
    // kTickMask (negative execs are stored offset by cofs ticks, chains.cuh mkspan)
    double emax = 0.0, emin = 0.0, dmax_fin = -1.0;
    bool finite = true;
    for (size_t i = 0; i < total; ++i) {
        if (!std::isfinite(exec[i])) finite = false;
        else emax = std::max(emax, exec[i]), emin = std::min(emin, exec[i]);
        if (std::isfinite(deadline[i]) && deadline[i] >= 0.0) dmax_fin = std::max(dmax_fin, deadline[i]);
    }
    const double range = emax - emin;
    int k = 40;
    if (range > 0.0) {
        k = 0;
        while (k < 60 && std::ldexp(range, k + 1) <= (double)kTickMask - 1.0) ++k;
        while (k > -60 && std::ldexp(range, k) > (double)kTickMask - 1.0) --k;
    }
    c->tick = std::ldexp(1.0, -k);
    c->cofs = emin < 0.0 ? (int)-std::nearbyint(std::ldexp(emin, k)) : 0;
    c->dg = dmax_fin >= 0.0 ? (long long)std::fmin(std::floor(std::ldexp(dmax_fin, k)), 0x1.0p61) : -1;
    c->marg = n / 2 + 2;  // chains.cuh cert_margin(n): no batch start drifts further from the reference
    c->exec_finite = finite;
    CK(cudaMemcpyAsync(c->exec_soa.p, exec, total * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->dl_soa.p, deadline, total * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    k_tables<<<(unsigned)((total + 255) / 256), 256, 0, c->stream>>>((int)total, c->exec_soa.as<double>(),
                                                                       c->dl_soa.as<double>(), std::ldexp(1.0, k), c->cofs,
                                                                       c->tab.as<double2>(), c->xt.as<uint32_t>(),
                                                                       c->dt.as<long long>());
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    c->n = n;
    c->mb = mb;
    c->prepared = false;
    return SLO_OK;
}

double slo_problem_tick_ms(slo_ctx* c) { return c && c->n > 0 ? c->tick : 0.0; }

int slo_evaluate_batch(slo_ctx* c, int32_t count, const uint16_t* perms, const uint32_t* bits, int32_t* n_met,
                       double* t, double* g) {
    if (!c) return fail(SLO_ERR_ARG, "slo_evaluate_batch: null context");
    if (c->n == 0) return fail(SLO_ERR_STATE, "slo_evaluate_batch: no problem set");
    if (count <= 0) return SLO_OK;
    const int n = c->n, words = (n + 31) / 32;
    CK(cudaSetDevice(c->device));
    CK(c->e_perms.reserve((size_t)count * n * sizeof(uint16_t)));
    CK(c->e_bits.reserve((size_t)count * words * sizeof(uint32_t)));
    CK(c->e_n.reserve((size_t)count * sizeof(int)));
    CK(c->e_t.reserve((size_t)count * sizeof(double)));
    CK(c->e_g.reserve((size_t)count * sizeof(double)));
    CK(c->e_err.reserve(sizeof(int)));
    CK(cudaMemsetAsync(c->e_err.p, 0, sizeof(int), c->stream));
    CK(cudaMemcpyAsync(c->e_perms.p, perms, (size_t)count * n * sizeof(uint16_t), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->e_bits.p, bits, (size_t)count * words * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    k_eval_exact<<<(count + 127) / 128, 128, 0, c->stream>>>(count, n, c->mb, words, c->e_perms.as<uint16_t>(),
                                                               c->e_bits.as<uint32_t>(), c->tab.as<double2>(),
                                                               c->e_n.as<int>(), c->e_t.as<double>(), c->e_g.as<double>(),
                                                               c->e_err.as<int>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(n_met, c->e_n.p, (size_t)count * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(t, c->e_t.p, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(g, c->e_g.p, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    int err = 0;
    CK(cudaMemcpyAsync(&err, c->e_err.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (err & 1) return fail(SLO_ERR_DATA, "slo_evaluate_batch: last position must end a batch");
    if (err & 2) return fail(SLO_ERR_DATA, "slo_evaluate_batch: batch larger than max_batch");
    if (err & 4) return fail(SLO_ERR_DATA, "slo_evaluate_batch: dense index out of range");
    return SLO_OK;
}

}  // extern "C"

namespace {
template <int UPL, bool NEG>
void launch_eval_tick(slo_ctx* c, const ChainParams& kp, int count, int words) {
    constexpr size_t slot = eval_slot_bytes<UPL>();
    const int warps = 8;
    const int grid = std::min((count + warps - 1) / warps, c->sm_count * 8);
    static_assert(8 * slot <= 227 * 1024, "evaluator slots exceed shared memory");
    cudaFuncSetAttribute(k_eval_tick<UPL, NEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(warps * slot));
    k_eval_tick<UPL, NEG><<<grid, warps * 32, warps * slot, c->stream>>>(
        kp, count, words, c->e_perms.as<uint16_t>(), c->e_bits.as<uint32_t>(), c->e_n.as<int>(), c->e_t.as<double>(),
        c->e_g.as<double>(), c->e_err.as<int>());
}
}  // namespace

extern "C" {

int slo_evaluate_batch_tick(slo_ctx* c, int32_t count, const uint16_t* perms, const uint32_t* bits, int32_t* n_met,
                            double* t, double* g, uint64_t* exact_walks) {
    if (!c) return fail(SLO_ERR_ARG, "slo_evaluate_batch_tick: null context");
    if (c->n == 0) return fail(SLO_ERR_STATE, "slo_evaluate_batch_tick: no problem set");
    if (!c->exec_finite) return fail(SLO_ERR_DATA, "slo_evaluate_batch_tick: the tick grid needs finite exec times");
    if (count <= 0) return SLO_OK;
    const int n = c->n, words = (n + 31) / 32;
    CK(cudaSetDevice(c->device));
    CK(c->e_perms.reserve((size_t)count * n * sizeof(uint16_t)));
    CK(c->e_bits.reserve((size_t)count * words * sizeof(uint32_t)));
    CK(c->e_n.reserve((size_t)count * sizeof(int)));
    CK(c->e_t.reserve((size_t)count * sizeof(double)));
    CK(c->e_g.reserve((size_t)count * sizeof(double)));
    CK(c->e_err.reserve(sizeof(int)));
    CK(c->e_cnt.reserve(sizeof(unsigned long long)));
    CK(cudaMemsetAsync(c->e_err.p, 0, sizeof(int), c->stream));
    CK(cudaMemsetAsync(c->e_cnt.p, 0, sizeof(unsigned long long), c->stream));
    CK(cudaMemcpyAsync(c->e_perms.p, perms, (size_t)count * n * sizeof(uint16_t), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->e_bits.p, bits, (size_t)count * words * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    ChainParams kp{};
    kp.n = n, kp.mb = c->mb, kp.xt = c->xt.as<uint32_t>(), kp.dt = c->dt.as<long long>(), kp.tick = c->tick;
    kp.dg = c->dg >= 0 ? c->dg + c->marg : -1, kp.tab64 = c->tab.as<double2>();
    kp.exact_count = c->e_cnt.as<unsigned long long>();
    kp.cofs = c->cofs;
    const bool neg = c->cofs > 0;
    switch (pick_upl(n)) {
        case 1: neg ? launch_eval_tick<1, true>(c, kp, count, words) : launch_eval_tick<1, false>(c, kp, count, words); break;
        case 2: neg ? launch_eval_tick<2, true>(c, kp, count, words) : launch_eval_tick<2, false>(c, kp, count, words); break;
        default: neg ? launch_eval_tick<4, true>(c, kp, count, words) : launch_eval_tick<4, false>(c, kp, count, words); break;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(n_met, c->e_n.p, (size_t)count * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(t, c->e_t.p, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(g, c->e_g.p, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    int err = 0;
    unsigned long long cnt = 0;
    CK(cudaMemcpyAsync(&err, c->e_err.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&cnt, c->e_cnt.p, sizeof cnt, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (exact_walks) *exact_walks = cnt;
    if (err & 1) return fail(SLO_ERR_DATA, "slo_evaluate_batch_tick: last position must end a batch");
    if (err & 2) return fail(SLO_ERR_DATA, "slo_evaluate_batch_tick: batch larger than max_batch");
    if (err & 4) return fail(SLO_ERR_DATA, "slo_evaluate_batch_tick: dense index out of range");
    return SLO_OK;
}

}  // extern "C"

namespace {

int count_levels(double t0, double t_thres, double tau) {
    int L = 0;
    for (double t = t0; t >= t_thres; t *= tau) ++L;  // identical FP sequence to the device loop
    return L;
}

// The max-dynamic-smem attribute is per function and device (process-wide). Raise it to the
// device maximum once: concurrent contexts then never race on it, and no call blocks behind a
// running instance of the kernel (setting it while the kernel runs serialises the callers).
// (The device maximum less the kernel's static shared memory, s_xr.)
template <void (*K)(ChainParams)>
cudaError_t ensure_smem_attr(int device, size_t dyn_max) {
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> g(mu);
    if (device >= 0 && device < 64 && done[device]) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max);
    if (e == cudaSuccess && device >= 0 && device < 64) done[device] = true;
    return e;
}

// dynamic shared memory a block of K may use: the opt-in maximum less K's static allocation
template <void (*K)(ChainParams)>
size_t dyn_smem_max(const slo_ctx* c) {
    cudaFuncAttributes a{};
    if (cudaFuncGetAttributes(&a, K) != cudaSuccess) return c->smem_optin - 64;
    return c->smem_optin - a.sharedSizeBytes;
}

// W warps per block (bounded by max_w and shared memory), cpw chains per warp
template <void (*K)(ChainParams)>
int configure_kernel(slo_ctx* c, size_t base, size_t warp_bytes, int max_w, int cpw) {
    const size_t dyn_max = dyn_smem_max<K>(c);
    int W = (int)std::min<size_t>(max_w, (dyn_max - base) / warp_bytes);
    W = std::max(1, std::min(W, (c->chain_count + cpw - 1) / cpw));
    c->smem = base + (size_t)W * warp_bytes;
    CK(ensure_smem_attr<K>(c->device, dyn_max));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K, W * 32, c->smem));
    if (occ < 1) return fail(SLO_ERR_CAPACITY, "slo_anneal_chains: chain kernel does not fit on an SM");
    c->block = W * 32;
    c->grid = std::min((c->chain_count + W * cpw - 1) / (W * cpw), c->sm_count * occ);
    if (c->prm.max_blocks > 0) c->grid = std::min(c->grid, c->prm.max_blocks);
    return SLO_OK;
}

template <int UPL>
int configure_chains(slo_ctx* c) {
    const size_t tab_bytes = (size_t)c->n * c->mb * sizeof(uint32_t);
    const size_t tab_smem = (tab_bytes + 15) & ~(size_t)15;
    const size_t slot = slot_bytes<UPL>();
    const int max_w = chain_threads<UPL>() / 32;
    // the exec-tick table is staged in shared memory only when the block keeps its full warp
    // count beside it: where it would cost resident warps (N = 4096, mb = 4: 14 of 16) the chains
    // read it through L1 instead (measured: 1.27e9 vs 1.16e9 proposals/s there)
    const size_t full = (size_t)max_w * slot;
    if (c->cofs > 0) {  // negative execs (rare inputs): one variant, table through L1
        c->smem_tab = false;
        return configure_kernel<k_chains<UPL, false, true>>(c, 0, slot, max_w, 1);
    }
#ifdef SLO_TABLE_SMEM_IF_FITS
    c->smem_tab = tab_smem + slot <= dyn_smem_max<k_chains<UPL, true, false>>(c);
#else
    c->smem_tab = tab_smem + full <= dyn_smem_max<k_chains<UPL, true, false>>(c);
#endif
    return c->smem_tab ? configure_kernel<k_chains<UPL, true, false>>(c, tab_smem, slot, max_w, 1)
                       : configure_kernel<k_chains<UPL, false, false>>(c, 0, slot, max_w, 1);
}

template <int UPL>
void launch_t(slo_ctx* c) {
    const size_t ss = 32 * (size_t)UPL * 12 + 1024 * (size_t)UPL * 2 + 16 + 32 * (size_t)UPL * 4 + 16;
    if (c->cofs > 0) {
        k_start<UPL, true><<<1, 32, ss, c->stream>>>(c->kp);
        k_chains<UPL, false, true><<<c->grid, c->block, c->smem, c->stream>>>(c->kp);
        return;
    }
    k_start<UPL, false><<<1, 32, ss, c->stream>>>(c->kp);
    if (c->smem_tab) k_chains<UPL, true, false><<<c->grid, c->block, c->smem, c->stream>>>(c->kp);
    else k_chains<UPL, false, false><<<c->grid, c->block, c->smem, c->stream>>>(c->kp);
}

// K5: one chain per warp spread over as many SMs as the launch may use (a short queue's chain is
// latency-bound: fewer warps per scheduler is faster), the block's tables in shared memory
template <bool NEG, int MB>
int configure_small_t(slo_ctx* c) {
    constexpr auto K = k_chains_small<NEG, MB>;
    const size_t tab = ((size_t)c->n * c->mb * 12 + 15) & ~(size_t)15;
    int avail = c->sm_count;
    if (c->prm.max_blocks > 0) avail = std::min(avail, c->prm.max_blocks);
    const int W = std::max(1, std::min(kSmallThreads / 32, (c->chain_count + avail - 1) / avail));
    c->smem = tab + (size_t)W * small_warp_bytes();
    CK(ensure_smem_attr<K>(c->device, dyn_smem_max<K>(c)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K, W * 32, c->smem));
    if (occ < 1) return fail(SLO_ERR_CAPACITY, "slo_anneal_chains: short-queue kernel does not fit on an SM");
    c->block = W * 32;
    c->grid = std::min((c->chain_count + W - 1) / W, c->sm_count * occ);
    if (c->prm.max_blocks > 0) c->grid = std::min(c->grid, c->prm.max_blocks);
    return SLO_OK;
}

template <bool NEG, int MB>
void launch_small_t(slo_ctx* c) {
    const size_t ss = 32 * 12 + 1024 * 2 + 16 + 32 * 4 + 16;
    k_start<1, NEG><<<1, 32, ss, c->stream>>>(c->kp);
    k_chains_small<NEG, MB><<<c->grid, c->block, c->smem, c->stream>>>(c->kp);
}

// the segmented-max depth: the power of two >= mb
template <bool NEG, template <bool, int> class F, typename R = int>
R small_dispatch(slo_ctx* c) {
    const int mb = c->mb;
    if (mb <= 1) return F<NEG, 1>::run(c);
    if (mb <= 2) return F<NEG, 2>::run(c);
    if (mb <= 4) return F<NEG, 4>::run(c);
    if (mb <= 8) return F<NEG, 8>::run(c);
    return F<NEG, 16>::run(c);
}
template <bool NEG, int MB>
struct SmallConfigure {
    static int run(slo_ctx* c) { return configure_small_t<NEG, MB>(c); }
};
template <bool NEG, int MB>
struct SmallLaunch {
    static int run(slo_ctx* c) {
        launch_small_t<NEG, MB>(c);
        return 0;
    }
};

// prologue (start-state summaries, one warp) then the chain kernel
int launch_chains_U(slo_ctx* c) {
    if (c->small) {
        if (c->cofs > 0) small_dispatch<true, SmallLaunch>(c);
        else small_dispatch<false, SmallLaunch>(c);
        CK(cudaGetLastError());
        return SLO_OK;
    }
    switch (c->UPL) {
        case 1: launch_t<1>(c); break;
        case 2: launch_t<2>(c); break;
        case 4: launch_t<4>(c); break;
        default: return fail(SLO_ERR_CAPACITY, "bad units-per-lane");
    }
    CK(cudaGetLastError());
    return SLO_OK;
}

size_t chain_state_bytes(int upl) {
    return upl == 1 ? sizeof(LaneState<1>) : (upl == 2 ? sizeof(LaneState<2>) : sizeof(LaneState<4>));
}

int configure_U(slo_ctx* c) {
    if (c->small)
        return c->cofs > 0 ? small_dispatch<true, SmallConfigure>(c) : small_dispatch<false, SmallConfigure>(c);
    switch (c->UPL) {
        case 1: return configure_chains<1>(c);
        case 2: return configure_chains<2>(c);
        case 4: return configure_chains<4>(c);
    }
    return fail(SLO_ERR_CAPACITY, "bad units-per-lane");
}

// Load every kernel of the annealing path (and raise its shared-memory limit) once per device when
// the first context is created: with lazy module loading the first launch of each kernel otherwise
// pays for its load inside a timed decision (online windows: one-off 10-35 ms planning outliers
// the first time a queue size needs another kernel variant).
template <void (*K)(ChainParams)>
void warm_chain_kernel(slo_ctx* c) {
    ensure_smem_attr<K>(c->device, dyn_smem_max<K>(c));
}
template <typename F>
void warm_fn(F* f) {
    cudaFuncAttributes a{};
    cudaFuncGetAttributes(&a, f);
}
void prewarm_kernels(slo_ctx* c) {
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> g(mu);
    if (c->device < 0 || c->device >= 64 || done[c->device]) return;
    done[c->device] = true;
    warm_chain_kernel<k_chains<1, true, false>>(c), warm_chain_kernel<k_chains<1, false, false>>(c);
    warm_chain_kernel<k_chains<1, false, true>>(c), warm_chain_kernel<k_chains<2, true, false>>(c);
    warm_chain_kernel<k_chains<2, false, false>>(c), warm_chain_kernel<k_chains<2, false, true>>(c);
    warm_chain_kernel<k_chains<4, true, false>>(c), warm_chain_kernel<k_chains<4, false, false>>(c);
    warm_chain_kernel<k_chains<4, false, true>>(c);
    warm_chain_kernel<k_chains_small<false, 1>>(c), warm_chain_kernel<k_chains_small<false, 2>>(c);
    warm_chain_kernel<k_chains_small<false, 4>>(c), warm_chain_kernel<k_chains_small<false, 8>>(c);
    warm_chain_kernel<k_chains_small<false, 16>>(c), warm_chain_kernel<k_chains_small<true, 1>>(c);
    warm_chain_kernel<k_chains_small<true, 2>>(c), warm_chain_kernel<k_chains_small<true, 4>>(c);
    warm_chain_kernel<k_chains_small<true, 8>>(c), warm_chain_kernel<k_chains_small<true, 16>>(c);
    warm_fn(k_start<1, false>), warm_fn(k_start<1, true>), warm_fn(k_start<2, false>), warm_fn(k_start<2, true>);
    warm_fn(k_start<4, false>), warm_fn(k_start<4, true>), warm_fn(k_argmax), warm_fn(k_tables);
    cudaGetLastError();  // (a failure here surfaces again, with its message, at the launch)
}

}  // namespace

extern "C" {

int slo_chains_prepare(slo_ctx* c, const slo_chain_params* prm, const int32_t* start_perm,
                       const int32_t* start_sizes, int32_t start_nb) {
    if (!c || !prm) return fail(SLO_ERR_ARG, "slo_chains_prepare: null argument");
    if (c->n == 0) return fail(SLO_ERR_STATE, "slo_chains_prepare: no problem set");
    if (!(prm->t0 > prm->t_thres) || !(prm->t_thres > 0.0) || prm->iter < 1 || !(prm->tau > 0.0) || !(prm->tau < 1.0))
        return fail(SLO_ERR_DATA, "AnnealConfig: requires t0 > t_thres > 0, iter >= 1, tau in (0,1)");
    if (!(prm->objective_scale >= 0.0)) return fail(SLO_ERR_DATA, "AnnealConfig: objective_scale must be >= 0");
    const int n = c->n;
    const int cb = prm->chain_begin, ce = prm->chain_end;
    // a rank with a communicator may run no chain (fewer chains than ranks): it still takes part
    // in the exchange with an empty slot
    const bool empty = ce == cb && c->comm && prm->rng_mode == SLO_RNG_PHILOX;
    if (cb < 0 || (ce <= cb && !empty) || ce > prm->chains) return fail(SLO_ERR_ARG, "slo_chains_prepare: bad chain slice");
    // validate the start schedule
    {
        std::vector<char> seen(n, 0);
        int pos = 0;
        for (int k = 0; k < start_nb; ++k) {
            if (start_sizes[k] < 1 || start_sizes[k] > c->mb) return fail(SLO_ERR_DATA, "start schedule: bad batch size");
            pos += start_sizes[k];
        }
        if (pos != n) return fail(SLO_ERR_DATA, "start schedule: sizes do not cover n");
        for (int q = 0; q < n; ++q) {
            if (start_perm[q] < 0 || start_perm[q] >= n || seen[start_perm[q]]) return fail(SLO_ERR_DATA, "start schedule: not a permutation");
            seen[start_perm[q]] = 1;
        }
    }
    CK(cudaSetDevice(c->device));
    c->prm = *prm;
    c->prm.scale_mult = nullptr;
    c->chain_count = ce - cb;
    c->levels = count_levels(prm->t0, prm->t_thres, prm->tau);
    c->start_nb = start_nb;
    c->prepared = false;
    c->exchanged = false;
    c->empty_slice = empty;

    if (prm->rng_mode == SLO_RNG_XOSHIRO_REPLAY) {  // K2: one warp per chain, state in shared memory
        const int chains = c->chain_count;
        const int npad = (n + 31) & ~31;
        std::vector<uint16_t> ent(npad, 0);
        std::vector<uint32_t> bits(npad / 32, 0);
        int pos = 0;
        for (int k = 0; k < start_nb; ++k) {
            for (int j = 0; j < start_sizes[k]; ++j, ++pos) ent[pos] = (uint16_t)(start_perm[pos] + (start_sizes[k] - 1) * n);
            bits[(pos - 1) >> 5] |= 1u << ((pos - 1) & 31);
        }
        CK(c->start_ent.reserve((size_t)npad * sizeof(uint16_t)));
        CK(c->start_bits.reserve((size_t)(npad / 32) * sizeof(uint32_t)));
        CK(c->best_ent.reserve((size_t)chains * npad * sizeof(uint16_t)));
        CK(c->best_bits.reserve((size_t)chains * (npad / 32) * sizeof(uint32_t)));
        CK(c->rec.reserve((size_t)chains * sizeof(ChainRec)));
        CK(c->result.reserve(sizeof(ChainResult)));
        CK(c->win_ent.reserve((size_t)npad * sizeof(uint16_t)));
        CK(c->win_bits.reserve((size_t)(npad / 32) * sizeof(uint32_t)));
        CK(cudaMemcpyAsync(c->start_ent.p, ent.data(), (size_t)npad * sizeof(uint16_t), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->start_bits.p, bits.data(), bits.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const size_t slot = replay_slot_bytes(npad);
        if (slot > c->smem_optin) return fail(SLO_ERR_CAPACITY, "replay: schedule too large for shared memory");
        // one warp per block: the rest of the SM's 256 KB stays L1 for the table gathers
        c->block = 32;
        c->smem = (size_t)(c->block / 32) * slot;
        c->grid = (chains + c->block / 32 - 1) / (c->block / 32);
        CK(cudaFuncSetAttribute(k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_optin));
        // carve out only the shared memory the resident chains need (one warp each, as many per SM
        // as there are chains per SM, up to what fits): the rest of the SM's 256 KB stays L1, which
        // holds the (exec, deadline) table for the per-proposal gathers. A single chain is
        // latency-bound (one warp), so co-resident chains multiply throughput.
        const size_t per_sm = std::max<size_t>(1, std::min<size_t>((chains + c->sm_count - 1) / c->sm_count,
                                                                   c->smem_optin / c->smem));
        CK(cudaFuncSetAttribute(k_replay, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)std::min<size_t>(100, (per_sm * c->smem * 100 + c->smem_optin - 1) / c->smem_optin + 1)));
        c->UPL = npad / 32;  // words of the state, for fetch
        ReplayParams& rp = c->rp;
        rp.n = n, rp.mb = c->mb, rp.chains = chains, rp.magic = (1ull << 32) / (uint64_t)n + 1;
        rp.tab = c->tab.as<double2>();
        rp.t0 = prm->t0, rp.t_thres = prm->t_thres, rp.tau = prm->tau, rp.scale = prm->objective_scale;
        rp.iter = prm->iter, rp.seed = prm->seed + (uint64_t)cb;
        rp.start_ent = c->start_ent.as<uint16_t>(), rp.start_bits = c->start_bits.as<uint32_t>();
        rp.best_ent = c->best_ent.as<uint16_t>(), rp.best_bits = c->best_bits.as<uint32_t>();
        rp.rec = c->rec.as<ChainRec>(), rp.npad = npad;
        c->prepared = true;
        return SLO_OK;
    }
    if (prm->rng_mode != SLO_RNG_PHILOX) return fail(SLO_ERR_ARG, "slo_chains_prepare: unknown rng_mode");
    if (!c->exec_finite) return fail(SLO_ERR_DATA, "slo_chains_prepare: the chain kernel needs finite exec times");

    const int UPL = pick_upl(n);
    c->UPL = UPL;
    {  // K5 for short queues (SLOSCHED_SMALL_KERNEL=0 keeps K3: the equivalence tests run both)
        const char* ev = std::getenv("SLOSCHED_SMALL_KERNEL");
        c->small = n <= kSmallMaxN && c->mb <= 16 && !(ev && ev[0] == '0');
    }
    const size_t ent_words = 1024 * (size_t)UPL, bit_words = 32 * (size_t)UPL;
    if (empty) {  // only the exchange buffers: the slot says "no chain"
        CK(c->result.reserve(sizeof(ChainResult)));
        CK(c->win_ent.reserve(ent_words * sizeof(uint16_t)));
        CK(c->win_bits.reserve(bit_words * sizeof(uint32_t)));
        CK(c->exact_count.reserve(sizeof(unsigned long long)));
        if (int rc = ex_reserve(c, c->nranks)) return rc;
        c->prepared = true;
        return SLO_OK;
    }
    // start state: linear entries (batch_size-1)*n + dense index, linear batch-end bitmask
    std::vector<uint16_t> ent(ent_words, 0);
    std::vector<uint32_t> bits(bit_words, 0);
    {
        int pos = 0;
        for (int k = 0; k < start_nb; ++k) {
            for (int j = 0; j < start_sizes[k]; ++j, ++pos)
                ent[pos] = (uint16_t)(start_perm[pos] + (start_sizes[k] - 1) * n);
            bits[(pos - 1) >> 5] |= 1u << ((pos - 1) & 31);
        }
    }
    const size_t cc = c->chain_count;
    CK(c->start_ent.reserve(ent_words * sizeof(uint16_t)));
    CK(c->start_bits.reserve(3 * bit_words * sizeof(uint32_t)));  // + move flags (k_start)
    CK(c->best_ent.reserve(cc * ent_words * sizeof(uint16_t)));
    CK(c->best_bits.reserve(cc * bit_words * sizeof(uint32_t)));
    CK(c->rec.reserve(cc * sizeof(ChainRec)));
    CK(c->result.reserve(sizeof(ChainResult)));
    CK(c->win_ent.reserve(ent_words * sizeof(uint16_t)));
    CK(c->win_bits.reserve(bit_words * sizeof(uint32_t)));
    CK(c->scale_mult.reserve(std::max<size_t>(1, prm->n_scale_mult) * sizeof(double)));
    if (int rc = configure_U(c)) return rc;
    const int TW = c->grid * (c->block / 32);
    const bool multi = (int)cc > TW;
    const size_t csb = chain_state_bytes(UPL);
    CK(c->start_sum.reserve(32 * csb));
    CK(c->start_obj.reserve(4 * sizeof(double)));
    if (multi) {
        CK(c->st_ent.reserve(cc * ent_words * sizeof(uint16_t)));
        CK(c->st_bits.reserve(cc * 3 * bit_words * sizeof(uint32_t)));
        CK(c->st_sum.reserve(cc * 32 * csb));
    }
    // (LaneState has no padding and parked anchors are written before they are read: no memset)
    CK(cudaMemcpyAsync(c->start_ent.p, ent.data(), ent_words * sizeof(uint16_t), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->start_bits.p, bits.data(), bit_words * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    if (prm->n_scale_mult > 0)
        CK(cudaMemcpyAsync(c->scale_mult.p, prm->scale_mult, prm->n_scale_mult * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));  // host staging vectors go out of scope

    ChainParams& kp = c->kp;
    kp.n = n, kp.mb = c->mb, kp.smem_tab = c->smem_tab ? 1 : 0;
    kp.xt = c->xt.as<uint32_t>(), kp.dt = c->dt.as<long long>(), kp.tick = c->tick, kp.cofs = c->cofs;
    kp.dg = c->dg >= 0 ? c->dg + c->marg : -1, kp.tab64 = c->tab.as<double2>();
    kp.magic = n >= 2 ? (uint32_t)((1ull << 32) / (uint64_t)n + 1) : 0u;
    kp.t0 = prm->t0, kp.tau = prm->tau, kp.scale = prm->objective_scale;
    kp.iter = prm->iter, kp.levels = c->levels;
    kp.scale_mult = c->scale_mult.as<double>(), kp.n_mult = prm->n_scale_mult;
    kp.key0 = (uint32_t)prm->seed, kp.key1 = (uint32_t)(prm->seed >> 32);
    kp.chain_begin = cb, kp.chain_count = (int)cc;
    kp.budget_ns = prm->budget_ns;
    kp.start_ent = c->start_ent.as<uint16_t>(), kp.start_bits = c->start_bits.as<uint32_t>();
    kp.st_ent = multi ? c->st_ent.as<uint16_t>() : nullptr, kp.st_bits = multi ? c->st_bits.as<uint32_t>() : nullptr;
    kp.st_lane = multi ? c->st_sum.p : nullptr;
    kp.start_lane = c->start_sum.p, kp.start_obj = c->start_obj.as<long long>();
    kp.best_ent = c->best_ent.as<uint16_t>(), kp.best_bits = c->best_bits.as<uint32_t>();
    kp.rec = c->rec.as<ChainRec>();
    CK(c->exact_count.reserve(sizeof(unsigned long long)));
    kp.exact_count = c->exact_count.as<unsigned long long>();
    if (c->comm && !c->group)
        if (int rc = ex_reserve(c, c->nranks)) return rc;
    c->prepared = true;
    return SLO_OK;
}

}  // extern "C"

namespace {
// this device's chains and best-of-chains (no exchange)
int launch_local(slo_ctx* c) {
    const size_t cc = c->chain_count;
    c->exchanged = false;
    if (c->empty_slice) {
        CK(cudaEventRecord(c->ev0, c->stream));
        CK(cudaEventRecord(c->ev1, c->stream));
        return SLO_OK;
    }
    CK(cudaMemsetAsync(c->rec.p, 0, cc * sizeof(ChainRec), c->stream));
    if (c->prm.rng_mode != SLO_RNG_XOSHIRO_REPLAY)
        CK(cudaMemsetAsync(c->exact_count.p, 0, sizeof(unsigned long long), c->stream));
    CK(cudaEventRecord(c->ev0, c->stream));
    if (c->prm.rng_mode == SLO_RNG_XOSHIRO_REPLAY) {
        k_replay<<<c->grid, c->block, c->smem, c->stream>>>(c->rp);
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->ev1, c->stream));
        k_argmax<<<1, 512, 0, c->stream>>>((int)cc, c->rec.as<ChainRec>(), c->result.as<ChainResult>(), c->rp.npad,
                                            c->rp.npad / 32, c->best_ent.as<uint16_t>(), c->best_bits.as<uint32_t>(),
                                            c->win_ent.as<uint16_t>(), c->win_bits.as<uint32_t>());
        CK(cudaGetLastError());
        return SLO_OK;
    }
    int rc = launch_chains_U(c);
    if (rc) return rc;
    CK(cudaEventRecord(c->ev1, c->stream));
    k_argmax<<<1, 512, 0, c->stream>>>((int)cc, c->rec.as<ChainRec>(), c->result.as<ChainResult>(), 1024 * c->UPL, 32 * c->UPL,
                                        c->best_ent.as<uint16_t>(), c->best_bits.as<uint32_t>(),
                                        c->win_ent.as<uint16_t>(), c->win_bits.as<uint32_t>());
    CK(cudaGetLastError());
    return SLO_OK;
}
}  // namespace

extern "C" {

int slo_chains_launch(slo_ctx* c) {
    if (!c || !c->prepared) return fail(SLO_ERR_STATE, "slo_chains_launch: not prepared");
    if (c->group) return fail(SLO_ERR_STATE, "slo_chains_launch: the context belongs to a group (slo_group_anneal_chains)");
    CK(cudaSetDevice(c->device));
    if (int rc = launch_local(c)) return rc;
    // multi-process: the job-wide winner on every rank, enqueued behind the local argmax
    if (c->comm && c->prm.rng_mode == SLO_RNG_PHILOX) {
        if (int rc = ex_pack(c)) return rc;
        if (int rc = ex_allgather(c)) return rc;
        if (int rc = ex_pick(c, c->nranks)) return rc;
        CK(cudaEventRecord(c->ev2, c->stream));
    }
    return SLO_OK;
}

int slo_chains_fetch(slo_ctx* c, int32_t* best_perm, int32_t* best_sizes, int32_t* best_nb, slo_chain_result* out) {
    if (!c || !c->prepared) return fail(SLO_ERR_STATE, "slo_chains_fetch: not prepared");
    CK(cudaSetDevice(c->device));
    ChainResult r;
    unsigned long long exact = 0;
    CK(cudaMemcpyAsync(&r, c->result.p, sizeof r, cudaMemcpyDeviceToHost, c->stream));
    if (c->prm.rng_mode != SLO_RNG_XOSHIRO_REPLAY)
        CK(cudaMemcpyAsync(&exact, c->exact_count.p, sizeof exact, cudaMemcpyDeviceToHost, c->stream));
    if (c->empty_slice && !c->exchanged) return fail(SLO_ERR_STATE, "slo_chains_fetch: this rank ran no chain");
    unsigned long long local[3] = {0, 0, 0};
    if (c->exchanged)
        if (int rc = ex_local_counts(c, local)) return rc;
    const int n = c->n;
    std::vector<uint16_t> ent;
    std::vector<uint32_t> bits;
    const bool replay = c->prm.rng_mode == SLO_RNG_XOSHIRO_REPLAY;
    // winner entries: npad words for replay, 1024 * UPL for the chain kernel
    const size_t ent_n = replay ? (size_t)c->rp.npad : 1024 * (size_t)c->UPL;
    ent.resize(ent_n);
    bits.resize(replay ? (size_t)c->rp.npad / 32 : 32 * (size_t)c->UPL);
    CK(cudaMemcpyAsync(ent.data(), c->win_ent.p, ent.size() * sizeof(uint16_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(bits.data(), c->win_bits.p, bits.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f, xms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (c->exchanged) CK(cudaEventElapsedTime(&xms, c->ev1, c->ev2));
    if (r.chain < 0) return fail(SLO_ERR_STATE, "slo_chains_fetch: no chain ran (budget too small?)");
    {
        int nb = 0, run = 0;
        for (int q = 0; q < n; ++q) {
            best_perm[q] = ent[q] % n;
            ++run;
            if ((bits[q >> 5] >> (q & 31)) & 1u) best_sizes[nb++] = run, run = 0;
        }
        *best_nb = nb;
    }
    if (out) {
        out->g = r.g, out->t = r.t, out->n_met = r.n_met;
        out->chain = c->exchanged ? r.chain : c->prm.chain_begin + r.chain;
        out->proposals = r.proposals, out->accepted = r.accepted;
        out->chains_run = r.chains_run, out->levels_run = r.levels_min;
        out->kernel_ms = ms;
        out->positions_pass1 = r.scan1;
        out->positions_pass2 = r.scan2;
        out->exact_walks = exact;
        out->exchange_ms = xms;
        if (c->exchanged) out->local_proposals = local[0], out->local_positions_pass1 = local[1], out->local_positions_pass2 = local[2];
        else out->local_proposals = r.proposals, out->local_positions_pass1 = r.scan1, out->local_positions_pass2 = r.scan2;
        out->nranks = c->exchanged ? (c->group ? (int)slo_group_size(c->group) : c->nranks) : 1;
    }
    return SLO_OK;
}

int slo_exhaustive(slo_ctx* c, int32_t n_cap, int32_t* best_perm, int32_t* best_sizes, int32_t* best_nb,
                   double* g, double* t, uint64_t* evaluated) {
    if (!c) return fail(SLO_ERR_ARG, "slo_exhaustive: null context");
    if (c->n == 0) return fail(SLO_ERR_STATE, "slo_exhaustive: no problem set");
    const int n = c->n, mb = c->mb;
    if (n > n_cap)
        return fail(SLO_ERR_CAPACITY, "exhaustive: " + std::to_string(n) + " requests exceed cap of " +
                                          std::to_string(n_cap) + " (search space is O(N! * 2^N))");
    if (n > kExMaxN) return fail(SLO_ERR_CAPACITY, "exhaustive: the engine enumerates at most 16 requests");
    // ordered compositions of n with parts <= mb, lexicographic (P:src/priority_mapper.cpp:416-436)
    std::vector<uint8_t> comps, lens;
    std::vector<uint8_t> cur;
    auto rec = [&](auto&& self, int remaining) -> void {
        if (remaining == 0) {
            std::vector<uint8_t> row(kExMaxN, 0);
            std::copy(cur.begin(), cur.end(), row.begin());
            comps.insert(comps.end(), row.begin(), row.end());
            lens.push_back((uint8_t)cur.size());
            return;
        }
        for (int part = 1; part <= std::min(remaining, mb); ++part) {
            cur.push_back((uint8_t)part);
            self(self, remaining - part);
            cur.pop_back();
        }
    };
    rec(rec, n);
    const int n_comps = (int)lens.size();
    unsigned long long nfact = 1;
    for (int i = 2; i <= n; ++i) nfact *= (unsigned long long)i;
    const unsigned long long target = (unsigned long long)c->sm_count * 2048ull * 4ull;
    const unsigned long long total = nfact * (unsigned long long)n_comps;
    const unsigned long long chunk = std::max<unsigned long long>(1ull, (total + target - 1) / target);
    const unsigned long long cpc = (nfact + chunk - 1) / chunk;
    const unsigned long long items = cpc * (unsigned long long)n_comps;
    const unsigned long long blocks = (items + 255) / 256;
    if (blocks > 0x7fffffffull) return fail(SLO_ERR_CAPACITY, "exhaustive: search space too large");
    CK(cudaSetDevice(c->device));
    DevBuf d_comps, d_lens, d_best, d_out;
    CK(d_comps.reserve(comps.size()));
    CK(d_lens.reserve(lens.size()));
    CK(d_best.reserve(blocks * sizeof(ExKey)));
    CK(d_out.reserve(sizeof(ExKey)));
    CK(cudaMemcpyAsync(d_comps.p, comps.data(), comps.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(d_lens.p, lens.data(), lens.size(), cudaMemcpyHostToDevice, c->stream));
    k_exhaustive<<<(unsigned)blocks, 256, 0, c->stream>>>(n, c->tab.as<double2>(), n_comps, d_comps.as<uint8_t>(),
                                                           d_lens.as<uint8_t>(), nfact, chunk, cpc, d_best.as<ExKey>());
    CK(cudaGetLastError());
    k_exhaustive_reduce<<<1, 1024, 0, c->stream>>>((int)blocks, d_best.as<ExKey>(), d_out.as<ExKey>());
    CK(cudaGetLastError());
    ExKey best;
    CK(cudaMemcpyAsync(&best, d_out.p, sizeof best, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (!best.valid) return fail(SLO_ERR_STATE, "slo_exhaustive: no candidate evaluated");
    // unrank the winning permutation (lexicographic order over dense indices)
    std::vector<int> avail(n);
    for (int i = 0; i < n; ++i) avail[i] = i;
    unsigned long long r = best.prank, f = nfact;
    for (int i = 0; i < n; ++i) {
        f /= (unsigned long long)(n - i);
        const int d = (int)(r / f);
        r -= (unsigned long long)d * f;
        best_perm[i] = avail[d];
        avail.erase(avail.begin() + d);
    }
    *best_nb = lens[best.comp];
    for (int k = 0; k < lens[best.comp]; ++k) best_sizes[k] = comps[(size_t)best.comp * kExMaxN + k];
    *g = best.g;
    *t = best.t;
    *evaluated = total;
    return SLO_OK;
}

int slo_probe_smem_bandwidth(slo_ctx* c, double* gbytes_per_s) {
    if (!c || !gbytes_per_s) return fail(SLO_ERR_ARG, "slo_probe_smem_bandwidth: null argument");
    CK(cudaSetDevice(c->device));
    const size_t smem = 4096 * sizeof(uint4);
    CK(cudaFuncSetAttribute(k_smem_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DevBuf sink;
    CK(sink.reserve(1024 * sizeof(uint4)));
    const int grid = c->sm_count * 2, block = 1024, iters = 4096;
    k_smem_probe<<<grid, block, smem, c->stream>>>(64, sink.as<uint4>());  // warm-up
    CK(cudaGetLastError());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(c->ev0, c->stream));
        k_smem_probe<<<grid, block, smem, c->stream>>>(iters, sink.as<uint4>());
        CK(cudaEventRecord(c->ev1, c->stream));
        CK(cudaEventSynchronize(c->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        best = std::min(best, ms);
    }
    const double bytes = (double)grid * block * iters * 8 * sizeof(uint4);
    *gbytes_per_s = bytes / (best * 1e-3) / 1e9;
    CK(cudaStreamSynchronize(c->stream));
    return SLO_OK;
}

int slo_anneal_chains(slo_ctx* c, const slo_chain_params* prm, const int32_t* start_perm, const int32_t* start_sizes,
                      int32_t start_nb, int32_t* best_perm, int32_t* best_sizes, int32_t* best_nb,
                      slo_chain_result* result) {
    int rc = slo_chains_prepare(c, prm, start_perm, start_sizes, start_nb);
    if (rc) return rc;
    rc = slo_chains_launch(c);
    if (rc) return rc;
    return slo_chains_fetch(c, best_perm, best_sizes, best_nb, result);
}

}  // extern "C"

#include "exchange.cuh"

namespace {
void comm_destroy(void* comm) {
    if (nccl_api().ok) nccl_api().CommDestroy((ncclComm_t)comm);
}
}  // namespace
