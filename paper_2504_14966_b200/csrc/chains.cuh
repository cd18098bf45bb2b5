// K3: one annealing chain per warp (Philox4x32-10 moves, incremental objective).
// Included by engine.cu inside its anonymous namespace.
//
// Chain state (shared memory, per warp):
//   ent[q]   u16, q = position: combined table index (batch_size-1) * n + dense_index, so the
//            table gather needs no index arithmetic and every entry carries its batch size
//   bits[w]  u32 linear batch-end bitmask (bit q set iff q is the last position of a batch)
//   rnd      the Philox words of the next 32 proposals, drawn lane-parallel
// Objective: the schedule is cut into units of 32 consecutive positions. Each unit has a
// content-only summary (its batches' makespans, latency moments, deadline bound) computed
// cooperatively by the 32 lanes. A warp-wide scan over the unit summaries gives every
// unit's start time E and the makespan fmk of the batch open at its start; a unit's summed
// latency is then closed-form (cnt*E + fmk*A + bs), and the SLO test walks only "live" units
// (E <= an upper bound of the unit's deadlines) -- at N=1024 the first one or two. After a
// move only the (<= 2) dirty units are re-summarised.

#define kNegInf (-static_cast<double>(INFINITY))
#ifndef SLO_CHAIN_THREADS
#define SLO_CHAIN_THREADS 768  // k_chains<1> block size: 24 warps, 80 registers per thread
#endif
constexpr int kPreAttempts = 6;                      // move attempts drawn ahead (3 words each)
constexpr int kRndWords = 3 * kPreAttempts + 2;      // + the acceptance uniform (2 words)
static_assert(kRndWords % 4 == 0, "Philox block rows are stored as uint4");

struct UnitSum {
    double hm;    // max exec from the unit start through its first batch end (whole unit if none)
    double tm;    // max exec after the unit's last batch end
    double inner; // summed makespans of batches that start and end inside the unit
    double bs;    // sum of exec over the unit + sum over inner batches of makespan * positions after it
    float dmax;   // upper bound of the unit's deadlines (rounded up; -inf if none)
    int fe;       // unit contains a batch end
    int cnt;      // positions in the unit
    int A;        // positions after the first batch end
    int always;   // positions whose deadline is +inf (met in every schedule; excluded from dmax)
};

template <int UPL>
struct __align__(16) ChainState {  // per-lane registers: this lane's unit summaries + SLO-walk cache
    UnitSum s[UPL];
    double wE[UPL], wF[UPL];
    int wN[UPL];
};

struct ChainParams {
    int n, mb;
    uint64_t magic;      // floor(2^32 / n) + 1: (e * magic) >> 32 == e / n exactly for e < 65536
    const double2* tab;  // global [mb][n] (exec, deadline)
    int smem_tab;
    double t0, tau, scale;
    int iter, levels;
    const double* scale_mult;
    int n_mult;
    uint32_t key0, key1;
    int chain_begin, chain_count;
    long long budget_ns;
    const uint16_t* start_ent;   // [1024*UPL]
    const uint32_t* start_bits;  // [32*UPL]
    const void* start_sum;       // ChainState<UPL>[32]: the start state's summaries (k_start)
    const double* start_obj;     // {f, total, n_met} of the start state (k_start)
    uint16_t* st_ent;            // [chain_count][1024*UPL]  parked chains (several chains per warp)
    uint32_t* st_bits;           // [chain_count][32*UPL]
    void* st_sum;                // [chain_count][32] ChainState<UPL>
    uint16_t* best_ent;          // [chain_count][1024*UPL]
    uint32_t* best_bits;         // [chain_count][32*UPL]
    ChainRec* rec;
};

// The (exec, deadline) table: staged in shared memory (s = its 32-bit shared address) or read
// from global memory (g). A compile-time choice, so the gather is an LDS.128 / LDG.128 rather
// than a generic load.
struct TabRef {
    const double2* g;
    uint32_t s;
};

template <bool SMEM>
__device__ __forceinline__ double2 tab_ld(const TabRef& t, uint32_t i) {
    if constexpr (SMEM) {
        double2 v;
        asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(t.s + i * 16u));
        return v;
    } else {
        return __ldg(t.g + i);
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    return v;
}

// order-preserving map float -> u32 (for REDUX max)
__device__ __forceinline__ uint32_t f2key(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// segmented inclusive max over the 32 positions of a unit; segments restart after an end bit
// (and at the unit start) and are at most mb long, so log2(mb) shuffle steps suffice. The
// segment start comes from the bitmask, so only the value is shuffled.
__device__ __forceinline__ double seg_max(double e, uint32_t w, int lane, int mb) {
    double m = dmax(e, 0.0);  // makespans start at 0 (reference P:src/priority_mapper.cpp:266)
    const uint32_t below = w & ((1u << lane) - 1u);
    const int span = lane - (below ? 32 - __clz(below) : 0);  // positions before lane in its segment
    for (int d = 1; d < mb; d <<= 1) {
        const double mu = __shfl_up_sync(FULL, m, d);
        if (d <= span) m = dmax(m, mu);
    }
    return m;
}

// cooperative summary of unit u (all 32 lanes; every lane receives the result)
template <bool SMEM>
__device__ __forceinline__ UnitSum unit_summary(const uint16_t* ent, const uint32_t* bits, const TabRef& tab, int n,
                                                int mb, int u, int lane) {
    UnitSum s;
    const int q0 = u << 5;
    const int cnt = min(32, n - q0);
    const uint32_t w = bits[u];
    double e = 0.0, D = kNegInf;
    if (lane < cnt) {
        const double2 v = tab_ld<SMEM>(tab, ent[q0 + lane]);
        e = v.x, D = v.y;
    }
    const double m = seg_max(e, w, lane, mb);
    const int f = w ? __ffs(w) - 1 : -1;
    const int la = w ? 31 - __clz(w) : -1;
    const double m_last = __shfl_sync(FULL, m, cnt - 1);
    const double m_first = __shfl_sync(FULL, m, f < 0 ? cnt - 1 : f);
    const bool inner_end = ((w >> lane) & 1u) && lane != f;
    const double mk = inner_end ? m : 0.0;
    double inner = mk, bs = e + mk * (double)(cnt - 1 - lane);
#pragma unroll
    for (int d = 16; d; d >>= 1) {  // two interleaved butterfly reductions
        inner += __shfl_xor_sync(FULL, inner, d);
        bs += __shfl_xor_sync(FULL, bs, d);
    }
    s.fe = w != 0;
    s.cnt = cnt;
    s.A = w ? cnt - 1 - f : 0;
    s.hm = m_first;
    s.tm = (w == 0 || la < cnt - 1) ? m_last : 0.0;
    s.inner = inner;
    s.bs = bs;
    const bool inf = D == INFINITY;  // host marks deadlines no schedule can miss as +inf
    s.always = __popc(__ballot_sync(FULL, inf));
    s.dmax = key2f(__reduce_max_sync(FULL, f2key(__double2float_ru(inf ? kNegInf : D))));
    return s;
}

// cooperative SLO count of unit u whose first position starts at elapsed E, the batch open at
// the unit start having makespan fmk. Rare (live units whose inputs changed): kept out of line.
template <bool SMEM>
__device__ __noinline__ int unit_met(const uint16_t* ent, const uint32_t* bits, TabRef tab, int n, int mb, int u,
                                     int lane, double E, double fmk) {
    const int q0 = u << 5;
    const int cnt = min(32, n - q0);
    const uint32_t w = bits[u];
    double e = 0.0, D = kNegInf;
    if (lane < cnt) {
        const double2 v = tab_ld<SMEM>(tab, ent[q0 + lane]);
        e = v.x, D = v.y;
    }
    const double m = seg_max(e, w, lane, mb);
    const int f = w ? __ffs(w) - 1 : -1;
    double v = ((w >> lane) & 1u) ? (lane == f ? fmk : m) : 0.0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {  // inclusive prefix of closed makespans
        const double up = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += up;
    }
    double off = __shfl_up_sync(FULL, v, 1);
    if (lane == 0) off = 0.0;
    const bool met = lane < cnt && E + off <= D;
    return __popc(__ballot_sync(FULL, met));
}

// Philox words of (proposal, chain, attempt) -- out of line: only retries >= kPreAttempts need it
__device__ __noinline__ uint4 philox_draw(uint32_t prop, uint32_t cid, uint32_t attempt, uint32_t k0, uint32_t k1) {
    uint32_t r[4] = {prop, cid, attempt, kTagMove};
    philox10(r, k0, k1);
    return make_uint4(r[0], r[1], r[2], r[3]);
}

struct Move {
    int kind;        // 0 none, 1 range (squeeze/delay), 2 swap
    int lo, hi, split, sz1, sz2;
    int ra, rb, dir; // rotation on [ra, rb]; dir +1 right, -1 left
    int clr, set;    // bitmask edits (-1 = none)
    int a, b;        // swap positions
};

// The reference's proposal discipline (P:src/priority_mapper.cpp:184-198) over the entry /
// bitmask representation: batch sizes come from the entries, batch starts from one bit search.
// Attempts < kPreAttempts read the lane-parallel Philox block; later retries draw directly.
// Counter = (proposal, chain, attempt, tag): results do not depend on the launch geometry.
__device__ __forceinline__ Move draw_move(const uint16_t* ent, const uint32_t* bits, int n, int mb, uint32_t nn,
                                          uint64_t magic, uint32_t prop, uint32_t cid, uint32_t k0, uint32_t k1,
                                          const uint32_t* rw) {
    auto size_at = [&](int q) { return (int)(((uint64_t)ent[q] * magic) >> 32) + 1; };
    Move mv;
    mv.kind = 0;
    if (n == 0) return mv;
    for (int attempt = 0; attempt <= 8; ++attempt) {
        uint32_t r0, r1, r2;
        if (attempt < kPreAttempts) {
            r0 = rw[3 * attempt], r1 = rw[3 * attempt + 1], r2 = rw[3 * attempt + 2];
        } else {
            const uint4 r = philox_draw(prop, cid, (uint32_t)attempt, k0, k1);
            r0 = r.x, r1 = r.y, r2 = r.z;
        }
        const uint32_t op = attempt < 8 ? lemire32(r0, 3) : 2u;  // forced swap after 8 misses
        if (op == 0) {  // squeeze (:141-153)
            const int first = size_at(0);
            if (first >= n) continue;
            const int pos = first + (int)lemire32(r1, (uint32_t)(n - first));
            const int sk = prev_end(bits, pos) + 1;
            const int prev_size = size_at(sk - 1);
            if (prev_size >= mb) continue;
            const int ek = sk + size_at(sk) - 1;
            mv.kind = 1;
            mv.lo = sk - prev_size, mv.hi = ek, mv.split = sk;
            mv.sz1 = prev_size + 1, mv.sz2 = ek - sk;
            mv.ra = sk, mv.rb = pos, mv.dir = 1;
            mv.clr = sk - 1, mv.set = sk;
            return mv;
        } else if (op == 1) {  // delay (:155-170)
            const int pos = (int)lemire32(r1, (uint32_t)n);
            const int sk = prev_end(bits, pos) + 1;
            const int ek = sk + size_at(pos) - 1;
            if (ek < n - 1) {
                const int next_size = size_at(ek + 1);
                if (next_size >= mb) continue;
                const int ek1 = ek + next_size;
                mv.kind = 1;
                mv.lo = sk, mv.hi = ek1, mv.split = ek - 1;
                mv.sz1 = ek - sk, mv.sz2 = next_size + 1;
                mv.ra = pos, mv.rb = ek1, mv.dir = -1;
                mv.clr = ek, mv.set = ek >= 1 ? ek - 1 : -1;
            } else {
                mv.kind = 1;
                mv.lo = sk, mv.hi = n - 1, mv.split = n - 2;
                mv.sz1 = n - 1 - sk, mv.sz2 = 1;
                mv.ra = pos, mv.rb = n - 1, mv.dir = -1;
                mv.clr = -1, mv.set = n >= 2 ? n - 2 : -1;
            }
            return mv;
        } else {  // swap (:172-180)
            if (n < 2) continue;
            const int a = (int)lemire32(r1, (uint32_t)n);
            int b = (int)lemire32(r2, (uint32_t)(n - 1));
            if (b >= a) ++b;
            mv.kind = 2;
            mv.a = a, mv.b = b;
            return mv;
        }
    }
    return mv;
}

// Warp-wide scan over unit summaries: E[k] (start elapsed) and fmk[k] for this lane's units.
// Batches hold at most 16 positions, so every non-empty unit of 32 contains a batch end (the
// last, partial unit ends at position n-1): the batch open at a unit's start is exactly the
// previous unit's tail, and only the elapsed times need a scan.
template <int UPL>
__device__ __forceinline__ void combine_units(const ChainState<UPL>& cs, int lane, double (&E)[UPL],
                                              double (&fmk)[UPL]) {
    double rest = cs.s[0].inner;
#pragma unroll
    for (int k = 1; k < UPL; ++k) rest = rest + dmax(cs.s[k - 1].tm, cs.s[k].hm), rest = rest + cs.s[k].inner;
    double carry = __shfl_up_sync(FULL, cs.s[UPL - 1].tm, 1);
    if (lane == 0) carry = 0.0;
    double S = cs.s[0].fe ? dmax(carry, cs.s[0].hm) + rest : 0.0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {  // sum scan of the makespans closed in each lane
        const double v = __shfl_up_sync(FULL, S, d);
        if (lane >= d) S += v;
    }
    double el = __shfl_up_sync(FULL, S, 1);
    if (lane == 0) el = 0.0;
    double cm = carry;
#pragma unroll
    for (int k = 0; k < UPL; ++k) {
        const UnitSum& s = cs.s[k];
        E[k] = el;
        fmk[k] = dmax(cm, s.hm);
        el = el + fmk[k], el = el + s.inner, cm = s.tm;
    }
}

// objective G = n / t (reference :278); the reciprocal form is used identically everywhere
__device__ __forceinline__ double objective(int nm, double tot) {
    return tot > 0.0 ? (double)nm * __drcp_rn(tot) : 0.0;
}

// Objective of the current state. full: re-summarise every unit and re-walk every live unit;
// otherwise only units du0/du1 (-1 = none). Outputs the total latency, the SLO count and the
// per-unit (E, fmk, walk result) to commit when the state is accepted.
template <int UPL, bool SMEM>
__device__ __forceinline__ void evaluate_chain(ChainState<UPL>& cs, const uint16_t* ent, const uint32_t* bits,
                                               const TabRef& tab, int n, int mb, int lane, bool full, int du0,
                                               int du1, double& tot_out, int& nm_out, double (&E)[UPL],
                                               double (&fmk)[UPL], int (&nN)[UPL], unsigned long long& sc1,
                                               unsigned long long& sc2) {
    const int U = (n + 31) >> 5;
    const int todo = full ? 32 * UPL : (du0 < 0 ? 0 : (du1 >= 0 && du1 != du0 ? 2 : 1));
    for (int i = 0; i < todo; ++i) {  // one inlined copy of the unit summary
        const int u = full ? i : (i == 0 ? du0 : du1);
        UnitSum v{0.0, 0.0, 0.0, 0.0, -INFINITY, 0, 0, 0, 0};
        if (u < U) v = unit_summary<SMEM>(ent, bits, tab, n, mb, u, lane), sc1 += lane == 0 ? 32 : 0;
        if (lane == u / UPL) {
#pragma unroll
            for (int k = 0; k < UPL; ++k)
                if (k == u % UPL) cs.s[k] = v;
        }
    }
    combine_units<UPL>(cs, lane, E, fmk);
    double tot = 0.0;
    int nm = 0;
#pragma unroll
    for (int k = 0; k < UPL; ++k) {
        const UnitSum& s = cs.s[k];
        const int u = lane * UPL + k;
        // summed latency of the unit's positions, closed form
        tot += (double)s.cnt * E[k] + (s.fe ? fmk[k] * (double)s.A : 0.0) + s.bs;
        const bool live = E[k] <= (double)s.dmax;
        const bool dirty = full || u == du0 || u == du1;
        const bool need = live && (dirty || E[k] != cs.wE[k] || fmk[k] != cs.wF[k]);
        nN[k] = live ? cs.wN[k] : s.always;
        unsigned mask = __ballot_sync(FULL, need);
        while (mask) {  // cooperative SLO walks of the units that need one
            const int ln = __ffs(mask) - 1;
            mask &= mask - 1;
            const double Eu = __shfl_sync(FULL, E[k], ln);
            const double Fu = __shfl_sync(FULL, fmk[k], ln);
            const int cntm = unit_met<SMEM>(ent, bits, tab, n, mb, ln * UPL + k, lane, Eu, Fu);
            if (lane == ln) nN[k] = cntm;
            sc2 += lane == 0 ? 32 : 0;
        }
        nm += nN[k];
    }
    tot_out = warp_sum(tot);
    nm_out = __reduce_add_sync(FULL, nm);
}

template <int UPL>
__host__ __device__ constexpr int slot_bytes() {
    // entries + bitmask + two parked unit summaries + Philox block (32 proposals)
    return 1024 * UPL * 2 + 32 * UPL * 4 + 2 * (int)sizeof(UnitSum) + 32 * kRndWords * 4;
}

template <int UPL>
__device__ __forceinline__ void copy_state(uint16_t* de, uint32_t* db, const uint16_t* se, const uint32_t* sb,
                                           int lane) {
    constexpr int kEnt = 1024 * UPL, kBits = 32 * UPL;
    for (int i = lane; i < kEnt / 8; i += 32) reinterpret_cast<uint4*>(de)[i] = reinterpret_cast<const uint4*>(se)[i];
    for (int i = lane; i < kBits; i += 32) db[i] = sb[i];
}

// Prologue: one warp evaluates the start schedule shared by every chain and publishes its
// unit summaries, so the chains start without a full evaluation each.
template <int UPL>
__global__ void __launch_bounds__(32) k_start(const ChainParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    uint16_t* ent = reinterpret_cast<uint16_t*>(smem);
    uint32_t* bits = reinterpret_cast<uint32_t*>(smem + 1024 * UPL * 2);
    copy_state<UPL>(ent, bits, p.start_ent, p.start_bits, lane);
    __syncwarp();
    ChainState<UPL> cs;
#pragma unroll
    for (int k = 0; k < UPL; ++k) cs.wE[k] = 0.0, cs.wF[k] = 0.0, cs.wN[k] = 0;
    double tot, E[UPL], fmk[UPL];
    int nm, nN[UPL];
    unsigned long long sc1 = 0, sc2 = 0;
    const TabRef tab{p.tab, 0u};
    evaluate_chain<UPL, false>(cs, ent, bits, tab, p.n, p.mb, lane, true, -1, -1, tot, nm, E, fmk, nN, sc1, sc2);
#pragma unroll
    for (int k = 0; k < UPL; ++k) cs.wE[k] = E[k], cs.wF[k] = fmk[k], cs.wN[k] = nN[k];
    reinterpret_cast<ChainState<UPL>*>(const_cast<void*>(p.start_sum))[lane] = cs;
    if (lane == 0) {
        double* o = const_cast<double*>(p.start_obj);
        o[0] = objective(nm, tot), o[1] = tot, o[2] = (double)nm;
    }
}

template <int UPL, bool SMEM>
__global__ void __launch_bounds__(UPL == 1 ? SLO_CHAIN_THREADS : 512, 1) k_chains(const ChainParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int n = p.n, mb = p.mb;

    TabRef tab{p.tab, 0u};
    size_t off = 0;
    if constexpr (SMEM) {  // stage the (exec, deadline) table once per block: coalesced 16 B loads
        double2* st = reinterpret_cast<double2*>(smem);
        const int total = mb * n;
        for (int i = threadIdx.x; i < total; i += blockDim.x) st[i] = p.tab[i];
        __syncthreads();
        tab.s = (uint32_t)__cvta_generic_to_shared(st);
        off = ((size_t)total * sizeof(double2) + 15) & ~(size_t)15;
    }
    constexpr int kEnt = 1024 * UPL, kBits = 32 * UPL;
    unsigned char* slot = smem + off + (size_t)wid * slot_bytes<UPL>();
    uint16_t* ent = reinterpret_cast<uint16_t*>(slot);
    uint32_t* bits = reinterpret_cast<uint32_t*>(slot + kEnt * 2);
    UnitSum* saved = reinterpret_cast<UnitSum*>(slot + kEnt * 2 + kBits * 4);
    uint32_t* rnd = reinterpret_cast<uint32_t*>(slot + kEnt * 2 + kBits * 4 + 2 * sizeof(UnitSum));

    const int gw = blockIdx.x * W + wid, TW = gridDim.x * W;
    if (gw >= p.chain_count) return;
    const int n_my = (p.chain_count - gw + TW - 1) / TW;

    uint64_t deadline = ~0ull;
    if (p.budget_ns > 0) deadline = __shfl_sync(FULL, gtimer(), 0) + (uint64_t)p.budget_ns;

    ChainState<UPL> cs;
    double f = 0.0, best_f = 0.0;
    unsigned long long props = 0, accs = 0;
    int stop = 0;
    const uint32_t nn = (uint32_t)n;
    const uint64_t magic = p.magic;
    auto* parked = reinterpret_cast<ChainState<UPL>*>(p.st_sum);

    double t = p.t0;
    for (int lev = 0; lev < p.levels && !stop; ++lev, t *= p.tau) {
        const double inv_t = 1.0 / t;
        for (int k = 0; k < n_my; ++k) {
            if (p.budget_ns > 0 && __shfl_sync(FULL, gtimer() > deadline ? 1 : 0, 0)) {
                stop = 1;
                break;
            }
            const int c = gw + k * TW;
            const uint32_t cid = (uint32_t)(p.chain_begin + c);
            ChainRec* rc = p.rec + c;
            unsigned long long sc1 = 0, sc2 = 0;
            if (lev == 0) {  // every chain starts from the shared start state
                copy_state<UPL>(ent, bits, p.start_ent, p.start_bits, lane);
                cs = reinterpret_cast<const ChainState<UPL>*>(p.start_sum)[lane];
                f = best_f = p.start_obj[0], props = 0, accs = 0;
                __syncwarp();
                copy_state<UPL>(p.best_ent + (size_t)c * kEnt, p.best_bits + (size_t)c * kBits, ent, bits, lane);
                if (lane == 0) rc->g = f, rc->t = p.start_obj[1], rc->n_met = (int)p.start_obj[2];
            } else if (n_my > 1) {  // resume a parked chain
                copy_state<UPL>(ent, bits, p.st_ent + (size_t)c * kEnt, p.st_bits + (size_t)c * kBits, lane);
                cs = parked[(size_t)c * 32 + lane];
                f = rc->cur_f, best_f = rc->g, props = rc->proposals, accs = rc->accepted;
                __syncwarp();
            }
            const double scale = p.n_mult > 0 ? p.scale * p.scale_mult[cid % (uint32_t)p.n_mult] : p.scale;

            for (int it = 0; it < p.iter; ++it) {
                // the device budget is checked every 8 proposals (warp-uniform), so a launch
                // overruns it by at most ~8 proposal latencies; the chain is parked as usual
                if (p.budget_ns > 0 && (it & 7) == 7 && __shfl_sync(FULL, gtimer() > deadline ? 1 : 0, 0)) {
                    stop = 1;
                    break;
                }
                const uint32_t prop = (uint32_t)(lev * p.iter + it);
                if ((it & 31) == 0) {  // lane j draws proposal prop + j: attempts 0..5 and acceptance
                    __syncwarp();      // every lane is done reading the previous block
                    uint4* dst = reinterpret_cast<uint4*>(rnd + kRndWords * lane);
                    uint32_t w[kRndWords];
#pragma unroll
                    for (int a = 0; a < kPreAttempts; ++a) {
                        uint32_t r[4] = {prop + (uint32_t)lane, cid, (uint32_t)a, kTagMove};
                        philox10(r, p.key0, p.key1);
                        w[3 * a] = r[0], w[3 * a + 1] = r[1], w[3 * a + 2] = r[2];
                    }
                    uint32_t r[4] = {prop + (uint32_t)lane, cid, (uint32_t)kAcceptAttempt, kTagMove};
                    philox10(r, p.key0, p.key1);
                    w[3 * kPreAttempts] = r[0], w[3 * kPreAttempts + 1] = r[1];
#pragma unroll
                    for (int v = 0; v < kRndWords / 4; ++v)
                        dst[v] = make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
                    __syncwarp();
                }
                const uint32_t* rw = rnd + kRndWords * (it & 31);
                const Move mv = draw_move(ent, bits, n, mb, nn, magic, prop, cid, p.key0, p.key1, rw);

                // ---- apply in place (undo on reject)
                int q = 0;
                uint16_t old_q = 0;
                uint32_t ow0 = 0, ow1 = 0;
                int w0 = 0, w1 = 0, du0 = -1, du1 = -1;
                if (mv.kind == 1) {
                    q = mv.lo + lane;
                    const bool act = q <= mv.hi;
                    uint16_t nw = 0;
                    if (act) {
                        int s = q;
                        if (mv.dir > 0) s = q == mv.ra ? mv.rb : (q > mv.ra && q <= mv.rb ? q - 1 : q);
                        else s = q == mv.rb ? mv.ra : (q >= mv.ra && q < mv.rb ? q + 1 : q);
                        old_q = ent[q];
                        const uint32_t se = ent[s];
                        const uint32_t idx = se - (uint32_t)(((uint64_t)se * magic) >> 32) * nn;
                        const int sz = q <= mv.split ? mv.sz1 : mv.sz2;
                        nw = (uint16_t)(idx + (uint32_t)(sz - 1) * nn);
                    }
                    w0 = mv.clr >= 0 ? mv.clr >> 5 : 0;
                    w1 = mv.set >= 0 ? mv.set >> 5 : 0;
                    ow0 = bits[w0], ow1 = bits[w1];
                    __syncwarp();
                    if (act) ent[q] = nw;
                    if (lane == 0) {
                        if (mv.clr >= 0) bits[mv.clr >> 5] &= ~(1u << (mv.clr & 31));
                        if (mv.set >= 0) bits[mv.set >> 5] |= 1u << (mv.set & 31);
                    }
                    __syncwarp();
                    du0 = mv.lo >> 5, du1 = mv.hi >> 5;
                } else if (mv.kind == 2) {
                    const uint32_t ea = ent[mv.a], eb = ent[mv.b];
                    ow0 = ea, ow1 = eb;
                    const uint32_t ba = (uint32_t)(((uint64_t)ea * magic) >> 32) * nn;
                    const uint32_t bb = (uint32_t)(((uint64_t)eb * magic) >> 32) * nn;
                    __syncwarp();
                    if (lane == 0) ent[mv.a] = (uint16_t)(ba + (eb - bb)), ent[mv.b] = (uint16_t)(bb + (ea - ba));
                    __syncwarp();
                    du0 = mv.a >> 5, du1 = mv.b >> 5;
                }
                // owners park the summaries of the dirty units (restored on reject)
#pragma unroll
                for (int kk = 0; kk < UPL; ++kk) {
                    if (du0 >= 0 && lane == du0 / UPL && kk == du0 % UPL) saved[0] = cs.s[kk];
                    if (du1 >= 0 && du1 != du0 && lane == du1 / UPL && kk == du1 % UPL) saved[1] = cs.s[kk];
                }
                double tot, E[UPL], fmk[UPL];
                int nm, nN[UPL];
                evaluate_chain<UPL, SMEM>(cs, ent, bits, tab, n, mb, lane, false, du0, du1, tot, nm, E, fmk, nN, sc1,
                                          sc2);
                const double f_new = objective(nm, tot);
                ++props;
                bool accept = f_new > f;  // Metropolis (P:src/priority_mapper.cpp:385-391)
                if (!accept) {
                    // x = (f - f_new) * scale / t; the test u < exp(-x) runs on the SFU in fp32
                    // (relative error ~1e-7 on the acceptance probability)
                    const double x = (f - f_new) * scale * inv_t;
                    const uint32_t* ru = rw + 3 * kPreAttempts;
                    const double u = (double)((((uint64_t)ru[0] << 32) | ru[1]) >> 11) * 0x1.0p-53;
                    accept = x < 38.0 ? (float)u < __expf(-(float)x) : u == 0.0;
                }
                if (accept) {
                    ++accs;
#pragma unroll
                    for (int kk = 0; kk < UPL; ++kk) cs.wE[kk] = E[kk], cs.wF[kk] = fmk[kk], cs.wN[kk] = nN[kk];
                    f = f_new;
                    if (f > best_f) {
                        best_f = f;
                        copy_state<UPL>(p.best_ent + (size_t)c * kEnt, p.best_bits + (size_t)c * kBits, ent, bits,
                                        lane);
                        if (lane == 0) rc->g = f, rc->t = tot, rc->n_met = nm;
                    }
                } else {
                    if (mv.kind == 1) {
                        if (q <= mv.hi) ent[q] = old_q;
                        if (lane == 0) bits[w1] = ow1, bits[w0] = ow0;
                    } else if (mv.kind == 2) {
                        if (lane == 0) ent[mv.a] = (uint16_t)ow0, ent[mv.b] = (uint16_t)ow1;
                    }
#pragma unroll
                    for (int kk = 0; kk < UPL; ++kk) {
                        if (du0 >= 0 && lane == du0 / UPL && kk == du0 % UPL) cs.s[kk] = saved[0];
                        if (du1 >= 0 && du1 != du0 && lane == du1 / UPL && kk == du1 % UPL) cs.s[kk] = saved[1];
                    }
                    __syncwarp();
                }
            }
            if (n_my > 1) {  // park the chain (state + summaries) until the next level
                copy_state<UPL>(p.st_ent + (size_t)c * kEnt, p.st_bits + (size_t)c * kBits, ent, bits, lane);
                parked[(size_t)c * 32 + lane] = cs;
                __syncwarp();
            }
            if (lane == 0) {
                rc->proposals = props, rc->accepted = accs, rc->levels = lev + 1, rc->cur_f = f;
                rc->scan1 += sc1, rc->scan2 += sc2;
            }
            if (stop) break;
        }
    }
}
