// Cross-device best-of-chains: the one data-path exchange of the path.
//
// Every device runs its slice of the global chain ids (k_chains), reduces it to its best chain
// (k_argmax) and packs that chain into a fixed-size slot: a 128-byte header (G, t, global chain
// id, summed counters) followed by the winner's position entries and batch-end bitmask. The
// slots are exchanged on the device -- no host round trip, nothing between the kernels and the
// collective but stream order -- and k_pick applies the argmax order of k_argmax (G desc, t asc,
// global chain id asc) to them, so every device ends up holding the job-wide winner:
//
//   multi-process (one rank per GPU, torchrun):  slo_ctx_comm_init attaches an NCCL communicator
//       (ncclCommInitRank); slo_chains_launch enqueues pack -> ncclAllGather -> pick.
//   single process, several devices:             slo_group_create (ncclCommInitAll, one context
//       per device); slo_group_anneal_chains launches every device, then one grouped
//       ncclAllGather, then pick. Devices listed twice (two contexts on one GPU) cannot share an
//       NCCL communicator: such groups gather the slots with peer copies onto member 0 instead.
//
// One all-gather of (#devices x slot) bytes replaces "all-reduce(MAX) on a packed key + broadcast
// of the winner": the winner is known on every device without the host learning the root, and
// ties resolve exactly (a packed 64-bit key cannot hold G, t and the chain id).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"; in a process that already mapped torch's
// NCCL the same library is reused), so the engine links no NCCL and single-device callers never
// touch it.
//
// The reference has no counterpart: it anneals one chain per instance on one CPU thread
// (P:src/scheduler.cpp:109-123, P:src/priority_mapper.cpp:340-411).
#include <dlfcn.h>
#include <nccl.h>

#include <thread>

namespace {

struct ExHead {                     // 128 bytes at the start of every slot
    double g, t;
    long long chain;                // global chain id, -1: no chain ran on this device
    unsigned long long proposals, accepted, scan1, scan2, exact;
    int n_met, chains_run, levels_min, pad;
    unsigned long long reserved[6];
};
static_assert(sizeof(ExHead) == 128, "slot header");

size_t ex_slot_bytes(size_t ent_words, size_t bit_words) {
    return ((sizeof(ExHead) + ent_words * 2 + bit_words * 4) + 127) & ~(size_t)127;
}

__global__ void k_pack(const ChainResult* __restrict__ r, int chain_begin, int empty,
                       const unsigned long long* __restrict__ exact, const uint16_t* __restrict__ win_ent,
                       const uint32_t* __restrict__ win_bits, int ent_words, int bit_words, uint8_t* slot) {
    ExHead* h = reinterpret_cast<ExHead*>(slot);
    if (threadIdx.x == 0) {
        ExHead o{};
        if (empty || r->chain < 0) {
            o.chain = -1, o.g = -2.0;
        } else {
            o.g = r->g, o.t = r->t, o.chain = (long long)chain_begin + r->chain, o.n_met = r->n_met;
            o.proposals = r->proposals, o.accepted = r->accepted, o.scan1 = r->scan1, o.scan2 = r->scan2;
            o.exact = exact ? *exact : 0ull;
            o.chains_run = r->chains_run, o.levels_min = r->levels_min;
        }
        *h = o;
    }
    if (empty) return;
    uint16_t* e = reinterpret_cast<uint16_t*>(slot + sizeof(ExHead));
    uint32_t* b = reinterpret_cast<uint32_t*>(slot + sizeof(ExHead) + (size_t)ent_words * 2);
    for (int i = threadIdx.x; i < ent_words; i += blockDim.x) e[i] = win_ent[i];
    for (int i = threadIdx.x; i < bit_words; i += blockDim.x) b[i] = win_bits[i];
}

// job-wide winner of `nslots` gathered slots (the k_argmax order over global chain ids)
__global__ void k_pick(int nslots, const uint8_t* __restrict__ gather, size_t slot_bytes, int ent_words,
                       int bit_words, ChainResult* out, unsigned long long* exact_out, uint16_t* win_ent,
                       uint32_t* win_bits) {
    __shared__ int s_win;
    if (threadIdx.x == 0) {
        int w = -1;
        double bg = 0.0, bt = 0.0;
        long long bc = 0;
        unsigned long long props = 0, accs = 0, sc1 = 0, sc2 = 0, ex = 0;
        int run = 0, lev = 0x7fffffff;
        for (int s = 0; s < nslots; ++s) {
            const ExHead* h = reinterpret_cast<const ExHead*>(gather + (size_t)s * slot_bytes);
            if (h->chain < 0) continue;
            props += h->proposals, accs += h->accepted, sc1 += h->scan1, sc2 += h->scan2, ex += h->exact;
            run += h->chains_run, lev = min(lev, h->levels_min);
            const bool b = w < 0 || h->g > bg || (h->g == bg && (h->t < bt || (h->t == bt && h->chain < bc)));
            if (b) w = s, bg = h->g, bt = h->t, bc = h->chain;
        }
        ChainResult r{};
        if (w < 0) {
            r.chain = -1;
        } else {
            const ExHead* h = reinterpret_cast<const ExHead*>(gather + (size_t)w * slot_bytes);
            r.g = h->g, r.t = h->t, r.n_met = h->n_met, r.chain = (int)h->chain;
            r.proposals = props, r.accepted = accs, r.scan1 = sc1, r.scan2 = sc2;
            r.chains_run = run, r.levels_min = lev == 0x7fffffff ? 0 : lev;
        }
        *out = r;
        if (exact_out) *exact_out = ex;
        s_win = w;
    }
    __syncthreads();
    const int w = s_win;
    if (w < 0) return;
    const uint8_t* slot = gather + (size_t)w * slot_bytes;
    const uint16_t* e = reinterpret_cast<const uint16_t*>(slot + sizeof(ExHead));
    const uint32_t* b = reinterpret_cast<const uint32_t*>(slot + sizeof(ExHead) + (size_t)ent_words * 2);
    for (int i = threadIdx.x; i < ent_words; i += blockDim.x) win_ent[i] = e[i];
    for (int i = threadIdx.x; i < bit_words; i += blockDim.x) win_bits[i] = b[i];
}

// ------------------------------------------------------------------ NCCL, loaded on first use
struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        const char* env = getenv("SLOSCHED_NCCL_LIB");
        void* h = nullptr;
        for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
            if (name && *name && (h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
        }
        if (!h) {
            const char* why = dlerror();
            a.err = std::string("NCCL not found (libnccl.so.2): ") + (why ? why : "");
            return a;
        }
        bool all = true;
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp) all = false;
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommInitAll, "ncclCommInitAll");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(a.AllGather, "ncclAllGather");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        sym(a.GetVersion, "ncclGetVersion");
        if (!all) a.err = "NCCL library lacks an entry point the exchange needs";
        a.ok = all;
        return a;
    }();
    return api;
}

#define NCK(call)                                                                          \
    do {                                                                                   \
        const NcclApi& a_ = nccl_api();                                                    \
        if (!a_.ok) return fail(SLO_ERR_COMM, a_.err);                                     \
        ncclResult_t r_ = (call);                                                          \
        if (r_ != ncclSuccess) return fail(SLO_ERR_COMM, std::string(#call) + ": " + a_.GetErrorString(r_)); \
    } while (0)

// the slot buffers of a context for its current chain configuration (Philox mode)
int ex_reserve(slo_ctx* c, int nslots) {
    const size_t ew = 1024 * (size_t)c->UPL, bw = 32 * (size_t)c->UPL;
    c->ex_slot_bytes = ex_slot_bytes(ew, bw);
    CK(c->ex_slot.reserve(c->ex_slot_bytes));
    CK(c->ex_gather.reserve(c->ex_slot_bytes * (size_t)nslots));
    return SLO_OK;
}

int ex_pack(slo_ctx* c) {
    k_pack<<<1, 256, 0, c->stream>>>(c->result.as<ChainResult>(), c->prm.chain_begin, c->empty_slice ? 1 : 0,
                                     c->exact_count.as<unsigned long long>(), c->win_ent.as<uint16_t>(),
                                     c->win_bits.as<uint32_t>(), 1024 * c->UPL, 32 * c->UPL, c->ex_slot.as<uint8_t>());
    CK(cudaGetLastError());
    return SLO_OK;
}

int ex_pick(slo_ctx* c, int nslots) {
    k_pick<<<1, 256, 0, c->stream>>>(nslots, c->ex_gather.as<uint8_t>(), c->ex_slot_bytes, 1024 * c->UPL, 32 * c->UPL,
                                     c->result.as<ChainResult>(), c->exact_count.as<unsigned long long>(),
                                     c->win_ent.as<uint16_t>(), c->win_bits.as<uint32_t>());
    CK(cudaGetLastError());
    c->exchanged = true;
    return SLO_OK;
}

// this device's own counters: its slot header in the gathered buffer (group member i = slot i)
int ex_local_counts(slo_ctx* c, unsigned long long out[3]) {
    const int me = c->rank;
    const uint8_t* h = c->ex_gather.as<uint8_t>() + (size_t)me * c->ex_slot_bytes;
    CK(cudaMemcpyAsync(&out[0], h + offsetof(ExHead, proposals), 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&out[1], h + offsetof(ExHead, scan1), 16, cudaMemcpyDeviceToHost, c->stream));
    return SLO_OK;
}

int ex_allgather(slo_ctx* c) {
    NCK(nccl_api().AllGather(c->ex_slot.p, c->ex_gather.p, c->ex_slot_bytes, ncclUint8, (ncclComm_t)c->comm,
                             c->stream));
    return SLO_OK;
}

// every contiguous balanced slice [b, e) of [lo, hi) for member i of k
void split_slice(int lo, int hi, int i, int k, int* b, int* e) {
    const int total = hi - lo, base = total / k, extra = total % k;
    *b = lo + i * base + std::min(i, extra);
    *e = *b + base + (i < extra ? 1 : 0);
}

}  // namespace

struct slo_group {
    std::vector<slo_ctx*> m;
    std::vector<int> devs;
    bool nccl = false;
};

extern "C" {

int slo_comm_unique_id(uint8_t* out) {
    if (!out) return fail(SLO_ERR_ARG, "slo_comm_unique_id: null out");
    ncclUniqueId id;
    NCK(nccl_api().GetUniqueId(&id));
    std::memcpy(out, id.internal, SLO_COMM_ID_BYTES);
    return SLO_OK;
}

int slo_ctx_comm_init(slo_ctx* c, int32_t nranks, int32_t rank, const uint8_t* id) {
    if (!c || !id) return fail(SLO_ERR_ARG, "slo_ctx_comm_init: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SLO_ERR_ARG, "slo_ctx_comm_init: bad rank / nranks");
    if (c->comm || c->group) return fail(SLO_ERR_STATE, "slo_ctx_comm_init: context already has a communicator");
    CK(cudaSetDevice(c->device));
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, SLO_COMM_ID_BYTES);
    ncclComm_t comm = nullptr;
    NCK(nccl_api().CommInitRank(&comm, nranks, uid, rank));
    c->comm = comm, c->own_comm = true, c->nranks = nranks, c->rank = rank;
    return SLO_OK;
}

int slo_ctx_exchange_empty(slo_ctx* c, int32_t n) {
    if (!c || !c->comm || c->group) return fail(SLO_ERR_ARG, "slo_ctx_exchange_empty: needs a rank context");
    if (n < 1 || n > SLO_MAX_N) return fail(SLO_ERR_ARG, "slo_ctx_exchange_empty: bad n");
    CK(cudaSetDevice(c->device));
    c->UPL = pick_upl(n);
    const size_t ew = 1024 * (size_t)c->UPL, bw = 32 * (size_t)c->UPL;
    CK(c->result.reserve(sizeof(ChainResult)));
    CK(c->win_ent.reserve(ew * sizeof(uint16_t)));
    CK(c->win_bits.reserve(bw * sizeof(uint32_t)));
    CK(c->exact_count.reserve(sizeof(unsigned long long)));
    if (int rc = ex_reserve(c, c->nranks)) return rc;
    c->empty_slice = true;
    c->prm.chain_begin = 0;
    if (int rc = ex_pack(c)) return rc;
    if (int rc = ex_allgather(c)) return rc;
    if (int rc = ex_pick(c, c->nranks)) return rc;
    CK(cudaStreamSynchronize(c->stream));
    c->prepared = false;
    return SLO_OK;
}

int slo_ctx_comm_info(slo_ctx* c, int32_t* nranks, int32_t* rank) {
    if (!c) return fail(SLO_ERR_ARG, "slo_ctx_comm_info: null context");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    return SLO_OK;
}

int slo_comm_check(slo_ctx* c) {
    if (!c) return fail(SLO_ERR_ARG, "slo_comm_check: null context");
    if (!c->comm) return SLO_OK;
    ncclResult_t st = ncclSuccess;
    NCK(nccl_api().CommGetAsyncError((ncclComm_t)c->comm, &st));
    if (st != ncclSuccess && st != ncclInProgress)
        return fail(SLO_ERR_COMM, std::string("NCCL async error: ") + nccl_api().GetErrorString(st));
    return SLO_OK;
}

int slo_group_create(int32_t ndev, const int32_t* devices, slo_group** out) {
    if (!out || !devices || ndev < 1) return fail(SLO_ERR_ARG, "slo_group_create: need >= 1 device");
    auto* g = new slo_group();
    for (int i = 0; i < ndev; ++i) {
        slo_ctx* c = nullptr;
        if (int rc = slo_ctx_create(devices[i], &c)) {
            slo_group_destroy(g);
            return rc;
        }
        c->group = g, c->rank = i, c->nranks = ndev;
        g->m.push_back(c);
        g->devs.push_back(devices[i]);
    }
    std::vector<int> sorted = g->devs;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const char* force = getenv("SLOSCHED_EXCHANGE");
    g->nccl = distinct && !(force && std::string(force) == "peer");
    if (g->nccl) {
        std::vector<ncclComm_t> comms(ndev);
        const NcclApi& a = nccl_api();
        ncclResult_t r = a.ok ? a.CommInitAll(comms.data(), ndev, g->devs.data()) : ncclSystemError;
        if (!a.ok || r != ncclSuccess) {
            const std::string msg = a.ok ? std::string("ncclCommInitAll: ") + a.GetErrorString(r) : a.err;
            slo_group_destroy(g);
            return fail(SLO_ERR_COMM, msg);
        }
        for (int i = 0; i < ndev; ++i) g->m[i]->comm = comms[i], g->m[i]->own_comm = true;
    }
    *out = g;
    return SLO_OK;
}

void slo_group_destroy(slo_group* g) {
    if (!g) return;
    for (slo_ctx* c : g->m) {
        c->group = nullptr;
        slo_ctx_destroy(c);
    }
    delete g;
}

int32_t slo_group_size(slo_group* g) { return g ? (int32_t)g->m.size() : 0; }
slo_ctx* slo_group_ctx(slo_group* g, int32_t i) {
    return g && i >= 0 && i < (int32_t)g->m.size() ? g->m[i] : nullptr;
}
const char* slo_group_transport(slo_group* g) { return !g ? "" : (g->nccl ? "nccl" : "peer"); }

int slo_group_problem_set(slo_group* g, int32_t n, int32_t mb, const double* exec, const double* deadline) {
    if (!g) return fail(SLO_ERR_ARG, "slo_group_problem_set: null group");
    const int k = (int)g->m.size();
    std::vector<int> rc(k, SLO_OK);
    std::vector<std::string> err(k);
    std::vector<std::thread> th;
    for (int i = 1; i < k; ++i)
        th.emplace_back([&, i] {
            rc[i] = slo_problem_set(g->m[i], n, mb, exec, deadline);
            if (rc[i]) err[i] = g_err;
        });
    rc[0] = slo_problem_set(g->m[0], n, mb, exec, deadline);
    if (rc[0]) err[0] = g_err;
    for (auto& t : th) t.join();
    for (int i = 0; i < k; ++i)
        if (rc[i]) return fail(rc[i], err[i]);
    return SLO_OK;
}

int slo_group_anneal_chains(slo_group* g, const slo_chain_params* prm, const int32_t* start_perm,
                            const int32_t* start_sizes, int32_t start_nb, int32_t* best_perm, int32_t* best_sizes,
                            int32_t* best_nb, slo_chain_result* result) {
    if (!g || !prm) return fail(SLO_ERR_ARG, "slo_group_anneal_chains: null argument");
    if (prm->rng_mode != SLO_RNG_PHILOX) return fail(SLO_ERR_ARG, "slo_group_anneal_chains: chains (Philox) mode only");
    const int k = (int)g->m.size();
    const int lo = prm->chain_begin, hi = prm->chain_end < 0 ? prm->chains : prm->chain_end;
    if (lo < 0 || hi > prm->chains || hi - lo < 1) return fail(SLO_ERR_ARG, "slo_group_anneal_chains: bad chain range");
    // phase 1: every member uploads its start state and slice (parallel host threads); a failure
    // anywhere stops the call before any collective is enqueued
    std::vector<int> rc(k, SLO_OK);
    std::vector<std::string> err(k);
    auto prep = [&](int i) {
        slo_chain_params p = *prm;
        int b, e;
        split_slice(lo, hi, i, k, &b, &e);
        p.chain_begin = b, p.chain_end = e;
        rc[i] = slo_chains_prepare(g->m[i], &p, start_perm, start_sizes, start_nb);
        if (!rc[i]) rc[i] = ex_reserve(g->m[i], k);
        if (rc[i]) err[i] = g_err;
    };
    {
        std::vector<std::thread> th;
        for (int i = 1; i < k; ++i) th.emplace_back(prep, i);
        prep(0);
        for (auto& t : th) t.join();
        for (int i = 0; i < k; ++i)
            if (rc[i]) return fail(rc[i], err[i]);
    }
    // phase 2 (this thread): every device's chains, argmax and slot, then the exchange
    for (slo_ctx* c : g->m) {
        CK(cudaSetDevice(c->device));
        if (int r = launch_local(c)) return r;
        if (int r = ex_pack(c)) return r;
    }
    if (g->nccl) {
        NCK(nccl_api().GroupStart());
        for (slo_ctx* c : g->m) {
            CK(cudaSetDevice(c->device));
            ncclResult_t r = nccl_api().AllGather(c->ex_slot.p, c->ex_gather.p, c->ex_slot_bytes, ncclUint8,
                                                  (ncclComm_t)c->comm, c->stream);
            if (r != ncclSuccess) {
                nccl_api().GroupEnd();
                return fail(SLO_ERR_COMM, std::string("ncclAllGather: ") + nccl_api().GetErrorString(r));
            }
        }
        NCK(nccl_api().GroupEnd());
    } else {  // peer copies of every slot onto member 0, ordered after each member's pack
        slo_ctx* c0 = g->m[0];
        for (int i = 0; i < k; ++i) {
            slo_ctx* c = g->m[i];
            CK(cudaSetDevice(c->device));
            CK(cudaEventRecord(c->ev_pack, c->stream));
            CK(cudaSetDevice(c0->device));
            CK(cudaStreamWaitEvent(c0->stream, c->ev_pack, 0));
            CK(cudaMemcpyPeerAsync(c0->ex_gather.as<uint8_t>() + (size_t)i * c0->ex_slot_bytes, c0->device, c->ex_slot.p,
                                   c->device, c0->ex_slot_bytes, c0->stream));
        }
    }
    const int pick_members = g->nccl ? k : 1;
    for (int i = 0; i < pick_members; ++i) {
        slo_ctx* c = g->m[i];
        CK(cudaSetDevice(c->device));
        if (int r = ex_pick(c, k)) return r;
        CK(cudaEventRecord(c->ev2, c->stream));
    }
    // the job-wide winner from member 0; device time = the slowest member's kernel
    if (int r = slo_chains_fetch(g->m[0], best_perm, best_sizes, best_nb, result)) return r;
    float kmax = result ? result->kernel_ms : 0.f;
    for (int i = 1; i < k; ++i) {
        slo_ctx* c = g->m[i];
        CK(cudaSetDevice(c->device));
        CK(cudaEventSynchronize(c->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        kmax = std::max(kmax, ms);
    }
    if (result) result->kernel_ms = kmax;
    for (int i = 1; i < k; ++i) g->m[i]->exchanged = false;
    return SLO_OK;
}

}  // extern "C"
