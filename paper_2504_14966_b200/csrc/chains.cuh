// K3: one annealing chain per warp (Philox4x32-10 moves) over a tick-exact incremental objective.
// Included by engine.cu inside its anonymous namespace.
//
// Objective arithmetic. Exec times are rounded once to a power-of-two grid of 2^-k ms ("ticks",
// k chosen per problem so every exec is < 2^27 ticks) and every sum is an integer: total latency
// and elapsed times are int64 (bounded by n^2 * 2^27 < 2^51 at n = 4096), so the objective is an
// exact function of the schedule, independent of summation order. That is what lets a move be
// scored from the few positions it touches: the result is bit-identical to a full re-evaluation
// (no drift, chains park and resume exactly). Deadlines compare exactly on the same grid:
// elapsed_ms <= D  <=>  elapsed_ticks <= floor(D * 2^k). The returned schedule is always
// re-scored by the exact reference arithmetic on the host (P:src/priority_mapper.cpp:404-410).
//
// Chain state (shared memory, per warp):
//   ent[q]   u16, q = position: combined table index (batch_size-1) * n + dense_index
//   bits[w]  u32 batch-end bitmask (bit q set iff q is the last position of a batch)
//   rnd      the Philox words of the next 32 proposals, drawn lane-parallel
// Per lane (registers): the anchors of its units of 32 positions -- E, the elapsed time at the
// start of the batch holding the unit's first position; F, that batch's makespan; W, the unit's
// met finite-deadline SLOs (kept while the unit is live, i.e. E <= the largest finite deadline).
// Chain scalars: total latency (ticks) and A, the number of positions whose deadline is +inf
// (met in every schedule). n_met = A + sum of W over live units.
//
// total = sum_q exec_q + sum_batches makespan_B * (positions after B)   (from e2e = elapsed + exec,
// P:src/priority_mapper.cpp:266-276), so a move changes the total only through the batches it
// rebuilds: a squeeze/delay rewrites two adjacent batches, a swap two batches. One warp pass over
// those positions (REDUX max per batch, REDUX sum of execs) gives the new total and the elapsed
// shift of every later batch; each lane then shifts its units' anchors, and only live units whose
// anchors or contents changed are re-walked (at N=1024 the first one or two units).

#ifndef SLO_CHAIN_THREADS
#define SLO_CHAIN_THREADS 896  // k_chains<1> block size (28 warps, 72 registers; 768 and 1024 measured slower)
#endif
#ifndef SLO_CHAIN_THREADS2
#define SLO_CHAIN_THREADS2 768  // 20-word rows let 25 warps fit; 24 balance 16384 chains better (8.8e9 vs 6.1e9)
#endif
#ifndef SLO_CHAIN_THREADS4
#define SLO_CHAIN_THREADS4 448  // 14 warps: the 64 KiB tick table keeps more L1 beside their slots (512: -3 %)
#endif
// block-size bound per units-per-lane (N <= 1024 / 2048 / 4096): more resident warps hide the
// dependent-latency stalls until registers spill (measured with tools/prof_chains.py --bench:
// UPL 2 896 > 768 > 640 > 512, UPL 4 448 > 512 ~ 384 > 416). 16384 chains over 148 x 28 warps is 3.95
// chains per warp, so 896 also balances; 832 and 960 leave a fifth/fourth round partly empty.
template <int UPL>
__host__ __device__ constexpr int chain_threads() {
    return UPL == 1 ? SLO_CHAIN_THREADS : (UPL == 2 ? SLO_CHAIN_THREADS2 : SLO_CHAIN_THREADS4);
}
// A proposal's row of Philox words: word 0 holds the ops of the 8 random attempts (U[0, 3^8) by
// one multiply-high, op j = its base-3 digit j: each op exactly uniform); attempt j reads its
// positions from words 1 + 2j (squeeze / delay position, first swap position) and 2 + 2j (second
// swap position); words 17, 18 are the forced swap's (attempt 8), word 19 the acceptance uniform.
constexpr int kAttempts = 9;                         // 8 random move attempts + the forced swap
constexpr int kOpsWord = 0;
constexpr int kAccWord = 1 + 2 * kAttempts;          // 19
constexpr int kRndWords = kAccWord + 1;              // 20 words = 5 Philox blocks
constexpr int kRndBlocks = kRndWords / 4;
static_assert(4 * kRndBlocks == kRndWords, "Philox row");
__device__ __forceinline__ uint32_t pos_word(int j) { return 1 + 2 * j; }
#ifndef SLO_PHILOX_UNROLL
#define SLO_PHILOX_UNROLL 1  // rolled: the kernel is instruction-fetch bound (N=1024: 1.31e10 unrolled, 1.47e10 rolled)
#endif
constexpr int kPhiloxUnroll = SLO_PHILOX_UNROLL;  // Philox blocks unrolled per row refill
#ifndef SLO_DECODE_UNROLL
#define SLO_DECODE_UNROLL 2  // code size: N=1024 1.48e10 at 8, 1.53e10 at 2
#endif
constexpr int kDecodeUnroll = SLO_DECODE_UNROLL;  // move attempts unrolled in the speculative decode
constexpr uint32_t kAlways = 0x80000000u;            // exec-tick flag: deadline +inf at this batch size
constexpr uint32_t kTickMask = 0x07ffffffu;          // exec ticks < 2^27: 32 of them sum in a u32
constexpr long long kPadE = 1ll << 62;               // anchor of units past the end (never live)

// Negative exec times (fitted coefficients with negative intercepts are valid reference inputs,
// P:src/core.cpp:55-62): the tick table then holds exec + cofs >= 0, and a makespan -- the
// reference's max starting at 0.0 (P:src/priority_mapper.cpp:267-273) -- is max(m - cofs, 0) of
// the offset maximum m. Exec sums over the same positions cancel the offset. NEG is a template
// flag so the common non-negative case compiles exactly as before.
template <bool NEG>
__device__ __forceinline__ uint32_t mkspan(uint32_t m, int cofs) {
    if constexpr (NEG) return (uint32_t)max((int)m - cofs, 0);
    else return m;
}

template <int UPL>
struct __align__(16) LaneState {  // this lane's unit anchors
    long long E[UPL];  // elapsed (ticks) at the start of the batch holding the unit's first position
    uint32_t F[UPL];   // makespan (ticks) of that batch
    int W[UPL];        // met finite-deadline SLOs of the unit (valid while E <= dg)
};

struct ChainParams {
    int n, mb;
    uint32_t magic;      // floor(2^32 / n) + 1 (0 for n = 1, whose only entry is 0):
                         // umulhi(e, magic) == e / n exactly for e < 65536, 2 <= n <= 4096
    const uint32_t* xt;  // global [mb][n] exec ticks | kAlways
    const long long* dt; // global [mb][n] deadline ticks (-1: never met; unused where kAlways)
    long long dg;        // live bound (ticks): the largest finite deadline + cert_margin(n) (-1: none); units
                         // with E > dg are dead -- no SLO met there, certified (unit_walk)
    const double2* tab64; // global [mb][n] {exec, latest start} fp64: the reference's SLO test
    unsigned long long* exact_count;  // SLO tests the grid could not certify (exact_met)
    double tick;         // 2^-k ms
    int cofs;            // exec tick offset: xt holds exec + cofs >= 0 (cofs > 0 only with negative execs)
    int smem_tab;
    double t0, tau, scale;
    int iter, levels;
    const double* scale_mult;
    int n_mult;
    uint32_t key0, key1;
    int chain_begin, chain_count;
    long long budget_ns;
    const uint16_t* start_ent;   // [1024*UPL]
    uint32_t* start_bits;        // [3][32*UPL]: batch ends (host), move flags sqb, dlb (k_start)
    void* start_lane;            // LaneState<UPL>[32]: the start state's anchors (k_start)
    long long* start_obj;        // {total ticks, A, n_met} of the start state (k_start)
    uint16_t* st_ent;            // [chain_count][1024*UPL]  parked chains (several chains per warp)
    uint32_t* st_bits;           // [chain_count][3][32*UPL]
    void* st_lane;               // [chain_count][32] LaneState<UPL>
    uint16_t* best_ent;          // [chain_count][1024*UPL]
    uint32_t* best_bits;         // [chain_count][32*UPL]
    ChainRec* rec;
};

// The exec-tick table: staged in shared memory (s = its 32-bit shared address) or read from
// global memory (g). A compile-time choice, so the gather is an LDS rather than a generic load.
struct TabRef {
    const uint32_t* g;
    uint32_t s;
};

template <bool SMEM>
__device__ __forceinline__ uint32_t xt_ld(const TabRef& t, uint32_t i) {
    if constexpr (SMEM) {
        uint32_t v;
        asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(t.s + i * 4u));
        return v;
    } else {
        return __ldg(t.g + i);
    }
}

// Batch-end searches for batches of <= 16 positions: the answer lies within the 64-bit window of
// the word holding q and its neighbour, so no loop is needed.
// last set bit strictly before q, or -1
// (bits[-1] is a zero word in the chain slot)
__device__ __forceinline__ int prev_end16(const uint32_t* bits, int q) {
    const int w = q >> 5;
    const uint32_t lo = bits[w - 1];
    const uint32_t hi = bits[w] & ((1u << (q & 31)) - 1u);
    // branch-free over the 64-bit window: clz(hi:lo) picks hi's top bit, else lo's (lo = 0 only
    // when w = 0, where the max gives -1)
    const unsigned long long x = (unsigned long long)hi << 32 | lo;
    return max((w << 5) + 31 - __clzll(x), -1);
}
// first set bit at or after q (bit n-1 is always set; the word after the last one is never the
// answer, so reading past it is harmless)
__device__ __forceinline__ int next_end16(const uint32_t* bits, int q) {
    const int w = q >> 5;
    const unsigned long long x = (((unsigned long long)bits[w + 1] << 32) | bits[w]) >> (q & 31);
    return q + __ffsll(x) - 1;
}

__device__ __forceinline__ unsigned long long mulw(uint32_t a, uint32_t b) { return (unsigned long long)a * b; }

// segmented inclusive max over the 32 positions of a unit; segments restart after an end bit
// (and at the unit start) and are at most mb long, so log2(mb) shuffle steps suffice
__device__ __forceinline__ uint32_t seg_max(uint32_t x, uint32_t w, int lane, int mb) {
    uint32_t m = x;
    const uint32_t below = w & ((1u << lane) - 1u);
    const int span = lane - (below ? 32 - __clz(below) : 0);  // positions before lane in its segment
    for (int d = 1; d < mb; d <<= 1) {
        const uint32_t mu = __shfl_up_sync(FULL, m, d);
        if (d <= span) m = max(m, mu);
    }
    return m;
}

// ---- SLO tests: certified on the tick grid, the rest in the reference's fp64 arithmetic
//
// The reference's elapsed time at a batch start is a left-to-right fp64 sum of the makespans
// before it (P:src/priority_mapper.cpp:264-276); the grid's is an exact integer sum of the same
// makespans rounded to ticks. With j batches before position q (j <= q), the two differ by at most
// j/2 ticks of rounding plus j * 2^-14 ticks of fp64 rounding (elapsed < 2^39 ticks), and the
// deadline tick is floor(D * 2^k). So a test whose tick slack d = dt - elapsed has
// |d| > cert_margin(q) = q/2 + 2 is met in the reference iff d >= 0. The rest (rare: ~1e-4 walks
// per proposal at the bench shape) is decided by re-summing in fp64 (exact_chunk). n_met is the
// reference's, bit for bit.
__device__ __forceinline__ int cert_margin(int q) { return (q >> 1) + 2; }

struct ExactRef {
    const double2* tab;        // [mb][n] {exec, latest start} fp64
    unsigned long long* count; // units decided by exact_chunk (statistics; may be null)
};
// Per block (set once by the kernels that walk): kept out of the walks' register arguments, since
// only the rare exact path reads it.
__shared__ ExactRef s_xr;

// The reference's SLO tests of one 32-position chunk c (walk_units calls it for chunks 0..u): the
// elapsed time goes on in fp64 makespan by makespan (elapsed += max(0.0, exec...)) and each batch
// start is compared with the fp64 latest-start table (met <=> elapsed <= latest start). The
// chunk's makespans come from a segmented max (exact in any order); only the additions are
// sequential. Loop-free: a loop in any function the walk reaches costs the chain kernel registers.
struct ExactStep {
    double E;      // elapsed at the start of the batch open after the chunk (warp-uniform)
    double mc;     // that batch's running makespan (warp-uniform)
    unsigned met;  // finite-deadline positions of the chunk that meet their SLO
};

__device__ __noinline__ ExactStep exact_chunk(const uint16_t* ent, const uint32_t* bits, const double2* tab, int n,
                                              int mb, int c, int lane, double E, double mc) {
    const int q = (c << 5) + lane;
    const uint32_t w = bits[c];
    double2 v = make_double2(0.0, -INFINITY);
    if (q < n) v = __ldg(&tab[ent[q]]);
    const uint32_t below = w & ((1u << lane) - 1u);
    const int span = lane - (below ? 32 - __clz(below) : 0);
    double m = v.x;
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {  // batches <= 16
        const double mu = __shfl_up_sync(FULL, m, d);
        if (d < mb && d <= span) m = dmax(m, mu);
    }
    m = dmax(below ? 0.0 : mc, m);  // the open batch carries its partial makespan in
    double Ec = E, Es = E;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        const double mk = __shfl_sync(FULL, m, k);
        if ((w >> k) & 1u) {
            Ec = Ec + mk;
            if (lane > k) Es = Ec;
        }
    }
    const double mlast = __shfl_sync(FULL, m, 31);
    ExactStep r;
    r.E = Ec;
    r.mc = (w >> 31) & 1u ? 0.0 : mlast;
    r.met = __ballot_sync(FULL, q < n && v.y != INFINITY && Es <= v.y);
    return r;
}

// Cooperative count of the met finite-deadline SLOs of unit u, whose first batch started at
// elapsed E with makespan F, on the tick grid; -1 when some test is not certified.
template <bool SMEM, bool NEG>
__device__ __forceinline__ int unit_count(const uint16_t* ent, const uint32_t* bits, TabRef tab, const long long* dt,
                                          int n, int mb, int cofs, int u, int lane, long long E, uint32_t F) {
    const int q = (u << 5) + lane;
    const uint32_t w = bits[u];
    uint32_t x = 0;
    long long D = -1;
    if (q < n) {
        const uint32_t e = ent[q];
        const uint32_t v = xt_ld<SMEM>(tab, e);
        x = mkspan<NEG>(v & kTickMask, cofs);
        if (!(v & kAlways)) D = __ldg(dt + e);  // +inf deadlines are counted in A, not here
    }
    const uint32_t m = seg_max(x, w, lane, mb);
    const int f = w ? __ffs(w) - 1 : 32;
    const uint32_t v = ((w >> lane) & 1u) ? (lane == f ? F : m) : 0u;
    uint32_t s = v;  // closed makespans of the unit: < 32 * 2^27, no overflow
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t up = __shfl_up_sync(FULL, s, d);
        if (lane >= d) s += up;
    }
    // D < 0: no elapsed time >= 0 meets the deadline (the reference's elapsed is >= 0 too)
    const long long sl = D - (E + (long long)(s - v));
    const unsigned marg = (unsigned)cert_margin(q);
    const bool amb = D >= 0 && (unsigned long long)(sl + marg) <= 2ull * marg;
    const unsigned met = __ballot_sync(FULL, D >= 0 && sl >= 0);
    if (__any_sync(FULL, amb)) return -1;
    return __popc(met);
}

// -1: some test needs the reference arithmetic (walk_units then runs exact_chunk over the prefix)
template <bool SMEM, bool NEG>
__device__ __noinline__ int unit_walk(const uint16_t* ent, const uint32_t* bits, TabRef tab, const long long* dt,
                                      int n, int mb, int cofs, int u, int lane, long long E, uint32_t F) {
    return unit_count<SMEM, NEG>(ent, bits, tab, dt, n, mb, cofs, u, lane, E, F);
}

struct Move {         // also the move record of K2 (replay.cuh)
    int kind;        // 0 none, 1 range (squeeze/delay), 2 swap
    int lo, hi, split, sz1, sz2;
    int ra, rb, dir; // rotation on [ra, rb]; dir +1 right, -1 left
    int clr, set;    // bitmask edits (-1 = none)
    int a, b;        // swap positions
};

constexpr uint32_t kNoMove = 0xffffffffu;  // packed move: op << 30 | pos | b << 13

// the batch rebuild of a squeeze (op 0) or delay (op 1) of position pos: batch bounds from one
// bit search, sizes from the entries
#ifndef SLO_COLD
#define SLO_COLD __forceinline__  // code only the general path runs (tuning runs: __noinline__)
#endif
__device__ SLO_COLD Move range_move(const uint16_t* ent, const uint32_t* bits, int n, uint32_t magic,
                                           uint32_t op, int pos) {
    auto size_at = [&](int q) { return (int)__umulhi(ent[q], magic) + 1; };
    Move mv;
    mv.kind = 1;
    if (op == 0) {
        const int sk = prev_end16(bits, pos) + 1;
        const int prev_size = size_at(sk - 1);
        const int ek = sk + size_at(sk) - 1;
        mv.lo = sk - prev_size, mv.hi = ek, mv.split = sk;
        mv.sz1 = prev_size + 1, mv.sz2 = ek - sk;
        mv.ra = sk, mv.rb = pos, mv.dir = 1;
        mv.clr = sk - 1, mv.set = sk;
    } else {
        const int ek = next_end16(bits, pos);
        const int sk = ek - size_at(pos) + 1;
        mv.ra = pos, mv.dir = -1;
        if (ek < n - 1) {
            const int next_size = size_at(ek + 1);
            const int ek1 = ek + next_size;
            mv.lo = sk, mv.hi = ek1, mv.split = ek - 1;
            mv.sz1 = ek - sk, mv.sz2 = next_size + 1;
            mv.rb = ek1;
            mv.clr = ek, mv.set = ek >= 1 ? ek - 1 : -1;
        } else {
            mv.lo = sk, mv.hi = n - 1, mv.split = n - 2;
            mv.sz1 = n - 1 - sk, mv.sz2 = 1;
            mv.rb = n - 1;
            mv.clr = -1, mv.set = n >= 2 ? n - 2 : -1;
        }
    }
    return mv;
}

// objective G = n / t (reference :278); the reciprocal form is used identically everywhere a
// score is recorded (the winner's g is compared bit-for-bit in the tests)
__device__ __forceinline__ double objective(int nm, double tot) {
    return tot > 0.0 ? (double)nm * __drcp_rn(tot) : 0.0;
}

// the chain's working score: the same quotient from a hardware reciprocal estimate and two Newton
// steps (relative error ~1e-16), a pure function of (nm, tot) like the exact one; only the
// Metropolis comparisons use it, recorded scores use objective()
__device__ __forceinline__ double objective_fast(int nm, double tot) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(tot));
    double e = fma(-tot, r, 1.0);
    r = fma(r, e, r);
    e = fma(-tot, r, 1.0);
    r = fma(r, e, r);
    return tot > 0.0 ? (double)nm * r : 0.0;
}

#ifndef SLO_RND_ROWS2
#define SLO_RND_ROWS2 32
#endif
#ifndef SLO_RND_ROWS4
// 32 rows (one proposal per lane) since the incremental live-cache refresh: N=4096 6.59e9 ->
// 7.49e9 fixed-work over 16 rows scored by lane pairs (16 stays available: -DSLO_RND_ROWS4=16)
#define SLO_RND_ROWS4 32
#endif
#ifndef SLO_RND_STRIDE1
#define SLO_RND_STRIDE1 20  // 5 x 16 B: odd in 16-byte units, so the row stores stay conflict-free
#endif
#ifndef SLO_RND_STRIDE_WIDE
#define SLO_RND_STRIDE_WIDE 20
#endif
// Philox rows drawn per refill (one per lane): 32 proposals (16: a lane pair per proposal)
template <int UPL>
__host__ __device__ constexpr int rnd_rows() { return UPL == 1 ? 32 : (UPL == 2 ? SLO_RND_ROWS2 : SLO_RND_ROWS4); }

// row stride (words): a row is 20 words (5 Philox blocks); an odd number of 16-byte units puts
// the lanes' row stores on distinct bank groups (conflict-free uint4 stores); where shared memory
// bounds the resident warps (2-4 units per lane) the dense stride keeps one more warp per SM
template <int UPL>
__host__ __device__ constexpr int rnd_stride() { return UPL == 1 ? SLO_RND_STRIDE1 : SLO_RND_STRIDE_WIDE; }

// units at the head of the schedule whose per-position slacks and batch starts are cached: the
// live prefix at the bench shape is two to four units
#ifndef SLO_LIVE_CAP2
#define SLO_LIVE_CAP2 6
#endif
#ifndef SLO_LIVE_CAP4
#define SLO_LIVE_CAP4 10
#endif
#ifndef SLO_LIVE_CAP1
#define SLO_LIVE_CAP1 5  // mb = 8 at N = 1024: the live prefix is 4 units (3: 6.2e9, 5: 9.1e9 proposals/s)
#endif
template <int UPL>
__host__ __device__ constexpr int live_cap() { return UPL == 1 ? SLO_LIVE_CAP1 : (UPL == 2 ? SLO_LIVE_CAP2 : SLO_LIVE_CAP4); }

template <int UPL>
__host__ __device__ constexpr int slot_bytes() {
    // entries + a zero word (bits[-1]) and padding + batch-end bitmask + two move-flag bitmasks +
    // Philox rows (next_end16 may read one word past the bitmask: the first flag word) + the
    // slack and batch-start caches of the first kLiveCap units and their anchors
    return 1024 * UPL * 2 + 16 + 3 * 32 * UPL * 4 + rnd_rows<UPL>() * rnd_stride<UPL>() * 4 +
           ((2 * live_cap<UPL>() * 32 * 4 + 8 * live_cap<UPL>() + 15) & ~15);  // (slots stay 16-byte aligned)
}

// entries + BW words of bitmasks (the batch ends; with 3 * 32 * UPL also the move flags)
template <int UPL, int BW = 32 * UPL>
__device__ __forceinline__ void copy_state(uint16_t* de, uint32_t* db, const uint16_t* se, const uint32_t* sb,
                                           int lane) {
    constexpr int kEnt = 1024 * UPL;
    for (int i = lane; i < kEnt / 8; i += 32) reinterpret_cast<uint4*>(de)[i] = reinterpret_cast<const uint4*>(se)[i];
    for (int i = lane; i < BW; i += 32) db[i] = sb[i];
}

// Move flags, words [w0, w1] (all lanes): bit q of sqb set iff a squeeze of position q fails (the
// batch before q's batch is full), of dlb iff a delay of q fails (q's batch is not the last and
// the next one is full). They change only when an accepted squeeze/delay rebuilds batches, so the
// draw tests an attempt with one bit instead of a batch-bound search.
__device__ SLO_COLD void rebuild_flags(const uint16_t* ent, const uint32_t* bits, uint32_t* sqb, uint32_t* dlb,
                                              int n, int mb, uint32_t magic, int w0, int w1, int lane) {
    for (int w = w0; w <= w1; ++w) {
        const int q = (w << 5) + lane;
        bool sb = false, db = false;
        if (q < n) {
            const int s = prev_end16(bits, q) + 1, e = next_end16(bits, q);
            sb = s > 0 && (int)__umulhi(ent[s - 1], magic) + 1 >= mb;
            db = e < n - 1 && (int)__umulhi(ent[e + 1], magic) + 1 >= mb;
        }
        const unsigned a = __ballot_sync(FULL, sb), b = __ballot_sync(FULL, db);
        if (lane == 0) sqb[w] = a, dlb[w] = b;
    }
}

// Re-walk the live units flagged in `need` (per unit k of this lane); W receives the counts. A unit
// the tick grid cannot certify (unit_walk returns -1) is decided by exact_chunk over chunks 0..u,
// one chunk per trip of the same loop (a separate loop, anywhere on this path, costs the chain
// kernel registers on every walk).
template <int UPL, bool SMEM, bool NEG>
__device__ __forceinline__ void walk_units(const bool (&need)[UPL], LaneState<UPL>& ls, const uint16_t* ent,
                                           const uint32_t* bits, const TabRef& tab, const long long* dt,
                                           int n, int mb, int cofs, int lane, unsigned& sc2) {
#pragma unroll
    for (int k = 0; k < UPL; ++k) {
        unsigned mask = __ballot_sync(FULL, need[k]);
        int c = -1;  // -1: the tick walk of the next unit; >= 0: its exact chunk c
        ExactStep st{0.0, 0.0, 0u};
        while (mask) {
            const int ln = __ffs(mask) - 1;
            const int u = ln * UPL + k;
            int cnt = -1;
            if (c < 0) {
                const long long Eu = __shfl_sync(FULL, ls.E[k], ln);
                const uint32_t Fu = __shfl_sync(FULL, ls.F[k], ln);
                cnt = unit_walk<SMEM, NEG>(ent, bits, tab, dt, n, mb, cofs, u, lane, Eu, Fu);
#ifndef SLO_DIAG
                sc2 += 32;  // only lane 0's count is stored
#endif
                if (cnt < 0) {
                    c = 0, st = ExactStep{0.0, 0.0, 0u};
                    if (lane == 0 && s_xr.count) atomicAdd(s_xr.count, 1ull);
                }
            } else {
                st = exact_chunk(ent, bits, s_xr.tab, n, mb, c, lane, st.E, st.mc);
                if (c == u) cnt = __popc(st.met), c = -1;
                else ++c;
            }
            if (cnt >= 0) {
                if (lane == ln) ls.W[k] = cnt;
                mask &= mask - 1;
            }
        }
    }
}

template <int UPL>
__device__ __forceinline__ int live_met(const LaneState<UPL>& ls, long long dg) {
    int s = 0;
#pragma unroll
    for (int k = 0; k < UPL; ++k) s += ls.E[k] <= dg ? ls.W[k] : 0;
    return (int)__reduce_add_sync(FULL, (unsigned)s);
}

// One warp evaluates a schedule from scratch with the chain kernel's arithmetic (tick totals, the
// certified SLO walk): each lane owns its UPL units, sums their batches sequentially, one warp scan
// gives the anchors. Es/Fs: kU-entry scratch. Returns the lane's anchors; tot, A, nm warp-uniform.
template <int UPL, bool NEG>
__device__ void eval_schedule(const ChainParams& p, const uint16_t* ent, const uint32_t* bits, long long* Es,
                              uint32_t* Fs, int lane, LaneState<UPL>& ls, long long& tot_out, int& A_out,
                              int& nm_out) {
    constexpr int kU = 32 * UPL;
    const int n = p.n;
    for (int u = lane; u < kU; u += 32) Es[u] = kPadE, Fs[u] = 0;
    __syncwarp();
    // each lane owns positions [q0, q1) (its UPL units); every non-empty range holds a batch end
    // (ranges are >= 32 long, batches <= 16), so the batch open at a range start is closed in it
    const int q0 = lane * 32 * UPL, q1 = min(n, q0 + 32 * UPL);
    uint32_t hm = 0, tm = 0;  // max exec through the first end; after the last end
    long long inner = 0;      // makespans of the batches that start after the first end
    bool seen = false;
    for (int q = q0; q < q1; ++q) {
        const uint32_t x = mkspan<NEG>(__ldg(p.xt + ent[q]) & kTickMask, p.cofs);
        if (!seen) hm = max(hm, x);
        else tm = max(tm, x);
        if ((bits[q >> 5] >> (q & 31)) & 1u) {
            if (seen) inner += tm;
            seen = true, tm = 0;
        }
    }
    uint32_t tprev = __shfl_up_sync(FULL, tm, 1);
    if (lane == 0) tprev = 0;
    const long long S = q0 < q1 ? (long long)max(tprev, hm) + inner : 0ll;
    long long E = S;  // exclusive scan: elapsed at the start of the batch open at q0
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long up = __shfl_up_sync(FULL, E, d);
        if (lane >= d) E += up;
    }
    E -= S;
    long long tot = 0;
    int A = 0, pend = -1;
    uint32_t mk = tprev;
    for (int q = q0; q < q1; ++q) {
        if ((q & 31) == 0) Es[q >> 5] = E, pend = q >> 5;
        const uint32_t v = __ldg(p.xt + ent[q]);
        const uint32_t x = mkspan<NEG>(v & kTickMask, p.cofs);
        A += v >> 31;
        tot += E + ((long long)(v & kTickMask) - p.cofs);  // the exec itself may be negative
        mk = max(mk, x);
        if ((bits[q >> 5] >> (q & 31)) & 1u) {
            if (pend >= 0) Fs[pend] = mk, pend = -1;
            E += mk, mk = 0;
        }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) tot += __shfl_xor_sync(FULL, tot, d);
    A = (int)__reduce_add_sync(FULL, (unsigned)A);
    __syncwarp();
    bool need[UPL];
#pragma unroll
    for (int k = 0; k < UPL; ++k) {
        ls.E[k] = Es[lane * UPL + k], ls.F[k] = Fs[lane * UPL + k], ls.W[k] = 0;
        need[k] = ls.E[k] <= p.dg;
    }
    unsigned sc2 = 0;
    const TabRef tab{p.xt, 0u};
    walk_units<UPL, false, NEG>(need, ls, ent, bits, tab, p.dt, n, p.mb, p.cofs, lane, sc2);
    tot_out = tot, A_out = A, nm_out = A + live_met<UPL>(ls, p.dg);
    __syncwarp();
}

// Prologue: one warp evaluates the start schedule shared by every chain and publishes its unit
// anchors, so the chains start without a full evaluation each.
template <int UPL, bool NEG>
__global__ void __launch_bounds__(32) k_start(const ChainParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int kU = 32 * UPL;
    const int lane = threadIdx.x;
    long long* Es = reinterpret_cast<long long*>(smem);
    uint32_t* Fs = reinterpret_cast<uint32_t*>(smem + kU * 8);
    uint16_t* ent = reinterpret_cast<uint16_t*>(smem + kU * 12);
    uint32_t* bits = reinterpret_cast<uint32_t*>(smem + kU * 12 + 1024 * UPL * 2 + 16);  // bits[-1] = 0
    copy_state<UPL>(ent, bits, p.start_ent, p.start_bits, lane);
    if (lane == 0) bits[-1] = 0u, bits[kU] = 0u, s_xr = ExactRef{p.tab64, p.exact_count};
    __syncwarp();
    rebuild_flags(ent, bits, p.start_bits + kU, p.start_bits + 2 * kU, p.n, p.mb, p.magic, 0, kU - 1, lane);
    LaneState<UPL> ls;
    long long tot;
    int A, nm;
    eval_schedule<UPL, NEG>(p, ent, bits, Es, Fs, lane, ls, tot, A, nm);
    reinterpret_cast<LaneState<UPL>*>(p.start_lane)[lane] = ls;
    if (lane == 0) p.start_obj[0] = tot, p.start_obj[1] = A, p.start_obj[2] = nm;
}

template <int UPL>
__host__ __device__ constexpr int eval_slot_bytes() {
    return 32 * UPL * 12 + 1024 * UPL * 2 + 16 + (32 * UPL + 1) * 4 + 12;
}

// K3 evaluator (slo_evaluate_batch_tick): the chain kernel's objective of given schedules, one
// warp per candidate -- n_met exactly CostModel::score's (P:src/priority_mapper.cpp:259-279),
// the total on the tick grid. perms: [count][n] dense indices; bits: [count][words] batch ends.
// Invalid candidates set error bits 1 (last position not a batch end), 2 (batch > mb), 4 (index
// out of range) and are not scored.
template <int UPL, bool NEG>
__global__ void __launch_bounds__(256) k_eval_tick(const ChainParams p, int count, int words,
                                                   const uint16_t* __restrict__ perms,
                                                   const uint32_t* __restrict__ cbits, int* __restrict__ n_met,
                                                   double* __restrict__ t_out, double* __restrict__ g_out,
                                                   int* __restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int kU = 32 * UPL;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char* slot = smem + (size_t)wid * eval_slot_bytes<UPL>();
    long long* Es = reinterpret_cast<long long*>(slot);
    uint32_t* Fs = reinterpret_cast<uint32_t*>(slot + kU * 8);
    uint16_t* ent = reinterpret_cast<uint16_t*>(slot + kU * 12);
    uint32_t* bits = reinterpret_cast<uint32_t*>(slot + kU * 12 + 1024 * UPL * 2 + 16);
    const int n = p.n;
    if (threadIdx.x == 0) s_xr = ExactRef{p.tab64, p.exact_count};
    __syncthreads();
    for (int c = blockIdx.x * (blockDim.x >> 5) + wid; c < count; c += gridDim.x * (blockDim.x >> 5)) {
        const uint32_t* cb = cbits + (size_t)c * words;
        for (int w = lane; w <= kU; w += 32) bits[w] = w < words ? cb[w] : 0u;
        if (lane == 0) bits[-1] = 0u;
        __syncwarp();
        // validation: bit n-1 ends a batch; no batch longer than mb; indices below n
        bool bad1 = !((bits[(n - 1) >> 5] >> ((n - 1) & 31)) & 1u), bad2 = false, bad4 = false;
        if (!bad1) {
            for (int q = lane; q < n; q += 32) {
                if ((bits[q >> 5] >> (q & 31)) & 1u) {
                    int s = q - 1;  // previous end (linear search, at most mb + 1 steps when valid)
                    while (s >= 0 && s >= q - p.mb && !((bits[s >> 5] >> (s & 31)) & 1u)) --s;
                    if (q - s > p.mb) bad2 = true;
                }
            }
            // bits past n - 1 must be clear
            for (int w = lane; w < words; w += 32) {
                const int lo = w << 5;
                const uint32_t keep = lo + 32 <= n ? FULL : (lo >= n ? 0u : (1u << (n - lo)) - 1u);
                if (cb[w] & ~keep) bad1 = true;
            }
        }
        const bool fail_v = __any_sync(FULL, bad1 || bad2);
        if (!fail_v) {
            for (int q = lane; q < n; q += 32) {
                const uint32_t i = perms[(size_t)c * n + q];
                if (i >= (uint32_t)n) bad4 = true;
                const int sz = next_end16(bits, q) - prev_end16(bits, q);
                ent[q] = (uint16_t)((uint32_t)(sz - 1) * (uint32_t)n + min(i, (uint32_t)n - 1));
            }
        }
        const unsigned e = (__any_sync(FULL, bad1) ? 1u : 0u) | (__any_sync(FULL, bad2) ? 2u : 0u) |
                           (__any_sync(FULL, bad4) ? 4u : 0u);
        __syncwarp();
        if (e) {
            if (lane == 0) atomicOr(err, (int)e);
            continue;
        }
        LaneState<UPL> ls;
        long long tot;
        int A, nm;
        eval_schedule<UPL, NEG>(p, ent, bits, Es, Fs, lane, ls, tot, A, nm);
        if (lane == 0) {
            const double t = (double)tot * p.tick;
            n_met[c] = nm, t_out[c] = t, g_out[c] = objective(nm, t);
        }
    }
}

template <int UPL, bool SMEM, bool NEG>
__global__ void __launch_bounds__(chain_threads<UPL>(), 1) k_chains(const ChainParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int n = p.n, mb = p.mb;

    TabRef tab{p.xt, 0u};
    size_t off = 0;
    if constexpr (SMEM) {  // stage the exec-tick table once per block: coalesced 16 B loads
        const int total = mb * n;
        uint32_t* st = reinterpret_cast<uint32_t*>(smem);
        const int v4 = total >> 2;
        for (int i = threadIdx.x; i < v4; i += blockDim.x) reinterpret_cast<uint4*>(st)[i] = reinterpret_cast<const uint4*>(p.xt)[i];
        for (int i = (v4 << 2) + threadIdx.x; i < total; i += blockDim.x) st[i] = p.xt[i];
        __syncthreads();
        tab.s = (uint32_t)__cvta_generic_to_shared(st);
        off = ((size_t)total * sizeof(uint32_t) + 15) & ~(size_t)15;
    }
    constexpr int kEnt = 1024 * UPL, kBits = 32 * UPL;
    // the slot's shared address is pinned in a register: otherwise the compiler, short of registers,
    // re-derives it (S2R CgaCtaId, LEA, IMAD by the slot size...) before most shared accesses
    uint32_t slot_s = (uint32_t)__cvta_generic_to_shared(smem + off + (size_t)wid * slot_bytes<UPL>());
    if constexpr (UPL == 1) asm volatile("" : "+r"(slot_s));  // (UPL 2/4: measured slower pinned)
    unsigned char* slot = reinterpret_cast<unsigned char*>(__cvta_shared_to_generic(slot_s));
    uint16_t* ent = reinterpret_cast<uint16_t*>(slot);
    uint32_t* bits = reinterpret_cast<uint32_t*>(slot + kEnt * 2 + 16);
    uint32_t* sqb = bits + kBits;  // move flags (state: copied and parked with the bitmask)
    uint32_t* dlb = bits + 2 * kBits;
    uint32_t* rnd = reinterpret_cast<uint32_t*>(slot + kEnt * 2 + 16 + 3 * kBits * 4);
    // sig[q] (q < 32 * min(live units, kLiveCap)): deadline minus batch start of position q in the
    // committed state, clamped to int32 (INT_MIN: +inf deadline or past the end). A unit whose
    // contents and batch structure are unchanged and whose anchor moves by d meets exactly
    // #{q : sig[q] >= d} finite-deadline SLOs (|d| < 2^28), so its walk is a ballot (UPL 1).
    int* sig = reinterpret_cast<int*>(rnd + rnd_rows<UPL>() * rnd_stride<UPL>());
    // bst[q] (same positions): batch start of position q minus its unit's anchor cE[q >> 5], in the
    // committed state (the speculative stage's live-region bound reads both)
    constexpr int kLiveCap = live_cap<UPL>();
    uint32_t* bst = reinterpret_cast<uint32_t*>(sig + kLiveCap * 32);
    long long* cE = reinterpret_cast<long long*>(bst + kLiveCap * 32);
    constexpr int kRows = rnd_rows<UPL>();
    if (lane == 0) bits[-1] = 0u;  // prev_end16 reads it for positions < 32 (never written again)
    if (threadIdx.x == 0) s_xr = ExactRef{p.tab64, p.exact_count};
    __syncthreads();

    const int gw = blockIdx.x * W + wid, TW = gridDim.x * W;
    if (gw >= p.chain_count) return;
    const int n_my = (p.chain_count - gw + TW - 1) / TW;

    uint64_t deadline = ~0ull;
    if (p.budget_ns > 0) deadline = __shfl_sync(FULL, gtimer(), 0) + (uint64_t)p.budget_ns;

    LaneState<UPL> cur;  // committed anchors
    long long tot = 0;   // committed total (ticks)
    int A = 0, nm_cur = 0;
    double f = 0.0, best_f = 0.0;
    unsigned props = 0, accs = 0;  // per chain and launch (< 2^32: levels * iter)
    int stop = 0;
    const uint32_t nn = (uint32_t)n;
    const uint32_t magic = p.magic;
    const long long dg = p.dg;
    auto* parked = reinterpret_cast<LaneState<UPL>*>(p.st_lane);

    double t = p.t0;
    for (int lev = 0; lev < p.levels && !stop; ++lev, t *= p.tau) {
        const double inv_t = 1.0 / t;
        double sinv = 0.0;  // objective scale / t of the current chain
        for (int k = 0; k < n_my; ++k) {
            if (p.budget_ns > 0 && __shfl_sync(FULL, gtimer() > deadline ? 1 : 0, 0)) {
                stop = 1;
                break;
            }
            const int c = gw + k * TW;
            const uint32_t cid = (uint32_t)(p.chain_begin + c);
            ChainRec* rc = p.rec + c;
            unsigned sc1 = 0, sc2 = 0;
            if (lev == 0) {  // every chain starts from the shared start state
                copy_state<UPL, 3 * kBits>(ent, bits, p.start_ent, p.start_bits, lane);
                cur = reinterpret_cast<const LaneState<UPL>*>(p.start_lane)[lane];
                tot = p.start_obj[0], A = (int)p.start_obj[1], nm_cur = (int)p.start_obj[2];
                f = best_f = objective_fast(nm_cur, (double)tot * p.tick), props = 0, accs = 0;
                __syncwarp();
                copy_state<UPL>(p.best_ent + (size_t)c * kEnt, p.best_bits + (size_t)c * kBits, ent, bits, lane);
                if (lane == 0) rc->g = objective(nm_cur, (double)tot * p.tick), rc->t = (double)tot * p.tick, rc->n_met = nm_cur;
            } else if (n_my > 1) {  // resume a parked chain
                copy_state<UPL, 3 * kBits>(ent, bits, p.st_ent + (size_t)c * kEnt, p.st_bits + (size_t)c * 3 * kBits,
                                           lane);
                cur = parked[(size_t)c * 32 + lane];
                tot = rc->cur_tot, A = rc->cur_A, nm_cur = rc->cur_n;
                f = rc->cur_f, best_f = rc->best_f, props = (unsigned)rc->proposals, accs = (unsigned)rc->accepted;
                __syncwarp();
            }
            const double scale = p.n_mult > 0 ? p.scale * p.scale_mult[cid % (uint32_t)p.n_mult] : p.scale;
            sinv = scale * inv_t;
            // live units form a prefix (E is nondecreasing along the schedule): the count and the
            // anchor of the first dead unit, for the speculative rejection stage
            int u_live = 0;
            long long e_dead = kPadE;
            auto refresh_live = [&]() {
                int cnt = 0;
#pragma unroll
                for (int kk = 0; kk < UPL; ++kk) cnt += __popc(__ballot_sync(FULL, cur.E[kk] <= dg));
                u_live = cnt;  // unit u = lane * UPL + kk
                long long ed = kPadE;
#pragma unroll
                for (int kk = 0; kk < UPL; ++kk)
                    if (kk == cnt % UPL) ed = cur.E[kk];
                e_dead = cnt < 32 * UPL ? __shfl_sync(FULL, ed, (cnt / UPL) & 31) : kPadE;
            };
            // the live caches hold units [0, rf_nu); accepted moves since the last refresh rebuilt
            // units [rf_lo, rf_hi] (contents or batch structure); units after them only shifted
            int rf_lo = 0, rf_hi = 1 << 20, rf_nu = 0;
            auto refresh_sig = [&]() {
                __syncwarp();
                const int nu = min(u_live, kLiveCap);
                for (int u = min(rf_lo, rf_nu); u < nu; ++u) {  // unit u: register u % UPL of lane u / UPL
                    long long Es = cur.E[0];
                    uint32_t Fs_ = cur.F[0];
#pragma unroll
                    for (int kk = 1; kk < UPL; ++kk)
                        if (u % UPL == kk) Es = cur.E[kk], Fs_ = cur.F[kk];
                    const long long Eu = __shfl_sync(FULL, Es, u / UPL);
                    const uint32_t Fu = __shfl_sync(FULL, Fs_, u / UPL);
                    const int q = (u << 5) + lane;
                    if (u > rf_hi && u < rf_nu) {
                        // same contents and batches, every batch start and the anchor moved by the
                        // same shift: bst stands, each slack moves by it (re-read where it was clamped)
                        const long long dE = Eu - cE[u];
                        if (dE != 0) {
                            const int sg = sig[q];
                            if (sg != INT_MIN) {
                                const long long sl = (sg == INT_MAX || sg == INT_MIN + 1)
                                                         ? __ldg(p.dt + ent[q]) - (Eu + (long long)bst[q])
                                                         : (long long)sg - dE;
                                sig[q] = (int)max(min(sl, (long long)INT_MAX), (long long)INT_MIN + 1);
                            }
                            __syncwarp();
                            if (lane == 0) cE[u] = Eu;
                        }
                        continue;
                    }
                    const uint32_t w = bits[u];
                    uint32_t x = 0;
                    long long D = 0;
                    bool fin = false;
                    if (q < n) {
                        const uint32_t e = ent[q];
                        const uint32_t v = xt_ld<SMEM>(tab, e);
                        x = mkspan<NEG>(v & kTickMask, p.cofs);
                        if (!(v & kAlways)) D = __ldg(p.dt + e), fin = D >= 0;
                    }
                    const uint32_t m = seg_max(x, w, lane, mb);
                    const int f0 = w ? __ffs(w) - 1 : 32;
                    const uint32_t vv = ((w >> lane) & 1u) ? (lane == f0 ? Fu : m) : 0u;
                    uint32_t sc = vv;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t up = __shfl_up_sync(FULL, sc, d);
                        if (lane >= d) sc += up;
                    }
                    const long long sl = D - (Eu + (long long)(sc - vv));
                    sig[q] = fin ? (int)max(min(sl, (long long)INT_MAX), (long long)INT_MIN + 1) : INT_MIN;
                    bst[q] = sc - vv;
                    if (lane == 0) cE[u] = Eu;
                }
                rf_lo = 1 << 20, rf_hi = -1, rf_nu = nu;
                __syncwarp();
            };
            // the live-prefix summary and caches are refreshed at the start of the next speculative
            // pass (one inlined copy: the kernel is instruction-fetch bound); every general-path
            // proposal follows a pass, so it always reads them fresh
            bool need_refresh = true;

            int next_check = 8;
            int pass_it0 = 0, pass_end = 0;  // the speculative pass covering proposals [pass_it0, pass_end)
            unsigned lead_c = 0, span_c = 0;  // rejected proposals of the pass (bit j); lane j's scanned positions
            uint32_t pk_c = kNoMove;          // lane j: the move of the pass's proposal j
            for (int it = 0; it < p.iter; ++it) {
                if (it >= next_check) {
                    // the device budget is checked every 8 proposals (warp-uniform), so a launch
                    // overruns it by at most ~8 proposal latencies; the chain is parked as usual
                    next_check = (it & ~7) + 8;
                    if (p.budget_ns > 0 && __shfl_sync(FULL, gtimer() > deadline ? 1 : 0, 0)) {
                        stop = 1;
                        break;
                    }
                }
                if ((it & (kRows - 1)) == 0) {  // lane j draws the row of proposal prop + j
                    const uint32_t prop0 = (uint32_t)(lev * p.iter + it);
                    __syncwarp();                // every lane is done reading the previous rows
                    {
                        // Philox block b of a row = counter (proposal, chain, b, tag); with 16 rows
                        // per refill the lane pair splits a row's blocks (3 + 2): every lane works
                        constexpr int kSplit = kRows == 32 ? kRndBlocks : (kRndBlocks + 1) / 2;
                        const int row = lane & (kRows - 1);
                        const int b0 = kRows == 32 || lane < kRows ? 0 : kSplit;
                        const int b1 = kRows == 32 || lane >= kRows ? kRndBlocks : kSplit;
                        uint32_t* dst = rnd + rnd_stride<UPL>() * row;
#pragma unroll kPhiloxUnroll
                        for (int b = b0; b < b1; ++b) {
                            uint32_t r[4] = {prop0 + (uint32_t)row, cid, (uint32_t)b, kTagMove};
                            philox_rounds<SLO_PHILOX_ROUNDS>(r, p.key0, p.key1);
                            if constexpr (rnd_stride<UPL>() % 4 == 0) {
                                reinterpret_cast<uint4*>(dst)[b] = make_uint4(r[0], r[1], r[2], r[3]);
                            } else {
#pragma unroll
                                for (int i = 0; i < 4; ++i) dst[4 * b + i] = r[i];
                            }
                        }
                    }
                    __syncwarp();
                }
                {
                    // Speculative rejection (exact), one proposal per lane: lane j scores proposal
                    // it + j (up to the end of the Philox block) against the current state. A
                    // proposal whose move (first valid attempt of 8, else the forced swap) is a swap
                    // that provably cannot raise the score enough to pass its Metropolis test is
                    // rejected without touching the state:
                    //   dead-region swaps -- every unit the swap touches or shifts is dead and stays
                    //     dead: n_met changes only through the +inf-deadline count (exact score);
                    //   live-region swaps whose makespan changes shift no batch earlier -- no other
                    //     request can gain an SLO, so n_met <= nm_cur + the two moved requests'
                    //     change (cached batch starts / slacks of the first kLiveCap units): the test
                    //     is monotone in n_met, so a rejection at this bound is the exact decision
                    //     (x >= 17 with a nonzero uniform keeps __expf's rounding out of it).
                    // While proposals are rejected the state does not change, so each was scored
                    // against exactly the state the sequential chain sees: the leading run of
                    // rejected ones is consumed; the first other proposal goes through the general
                    // path below with the same random words. A general-path rejection leaves the
                    // state bit-identical, so the rest of the pass stays valid; an accept ends it.
                    if (it >= pass_end) {
                        if (need_refresh) {
                            refresh_live();
                            refresh_sig();
                            need_refresh = false;
                        }
                        // kLanesPer lanes per proposal (2 where a refill holds 16 rows: the pair splits
                        // the move attempts and the two batches' gathers); g = the proposal, h = the half
                        constexpr int kLanesPer = 32 / kRows;
                        const int g = lane & (kRows - 1), h = lane / kRows;
                        const unsigned pair = kLanesPer == 1 ? FULL : (1u << g) | (1u << (g + kRows));
                        const int G = min(kRows - (it & (kRows - 1)), p.iter - it);
                        const bool on = g < G;
                        const uint32_t* rl = rnd + rnd_stride<UPL>() * ((it + g) & (kRows - 1));
                        const uint32_t first = __umulhi(ent[0], magic) + 1u;  // size of the first batch
                        uint32_t pk = kNoMove;
                        int jv = kAttempts - 1;  // the first valid attempt this lane found (8: none)
                        if (on && n >= 2) {
                            // the reference's proposal discipline (P:src/priority_mapper.cpp:184-198)
                            uint32_t ops = lemire32(rl[kOpsWord], 6561u);  // 3^8: the 8 ops as base-3 digits
                            if (h) ops /= 3u;
#pragma unroll kDecodeUnroll
                            for (int j = h; j < kAttempts - 1; j += kLanesPer) {
                                const uint32_t r1 = rl[pos_word(j)], r2 = rl[pos_word(j) + 1];
                                const uint32_t op = ops % 3u;
                                ops /= kLanesPer == 1 ? 3u : 9u;
                                const uint32_t a = lemire32(r1, nn);
                                const uint32_t ps = first + lemire32(r1, nn - first);
                                uint32_t b = lemire32(r2, nn - 1);
                                b += b >= a ? 1u : 0u;
                                const uint32_t pos = op == 0 ? ps : a;
                                const uint32_t qf = min(pos, nn - 1);
                                const bool fails = ((op == 0 ? sqb : dlb)[qf >> 5] >> (qf & 31)) & 1u;
                                if (op == 2u || (!fails && (op == 1u || first < nn))) {
                                    pk = op << 30 | pos | (op == 2u ? b << 13 : 0u);
                                    jv = j;
                                    break;
                                }
                            }
                        }
                        if constexpr (kLanesPer == 2) {  // the pair's first valid attempt
                            const int jo = __shfl_xor_sync(FULL, jv, kRows);
                            const uint32_t po = __shfl_xor_sync(FULL, pk, kRows);
                            if (jo < jv) pk = po;
                        }
                        if (on && n >= 2) {
                            if (pk == kNoMove) {  // the forced swap (attempt 8)
                                const uint32_t a8 = lemire32(rl[pos_word(kAttempts - 1)], nn);
                                uint32_t b8 = lemire32(rl[pos_word(kAttempts - 1) + 1], nn - 1);
                                b8 += b8 >= a8 ? 1u : 0u;
                                pk = 2u << 30 | a8 | b8 << 13;
                            }
                        }
                        bool rej = false;
                        unsigned span = 0;
                        if (on && (pk >> 30) == 2u) {
                            const int a0 = (int)(pk & 0x1fffu), b0 = (int)((pk >> 13) & 0x1fffu);
                            const int pa = min(a0, b0), pb = max(a0, b0);
                            const uint32_t ea_ = ent[pa], eb_ = ent[pb];
                            const uint32_t za = __umulhi(ea_, magic), zb = __umulhi(eb_, magic);  // size - 1
                            const uint32_t ba = za * nn, bb = zb * nn;
                            const uint32_t na = ba + (eb_ - bb), nb = bb + (ea_ - ba);
                            const int sa = prev_end16(bits, pa) + 1, sb = prev_end16(bits, pb) + 1;
                            // same batch: nothing changes, the reference accepts (x = 0): general path
                            if (sa != sb) {
                                const int ea = sa + (int)za, eb = sb + (int)zb;
                                // the two batches' makespans, and the maxima without the swapped positions
                                // (4 positions per trip, predicated: the gathers of a trip issue back to back)
                                uint32_t moa = 0, mxa = 0, mob = 0, mxb = 0;
                                // (a lane pair: batch a on the first half, batch b on the second)
                                const int za_ = kLanesPer == 2 && h ? -1 : (int)za, zb_ = kLanesPer == 2 && !h ? -1 : (int)zb;
                                for (int q0 = 0; q0 <= max(za_, zb_); q0 += 4) {
#pragma unroll
                                    for (int j = 0; j < 4; ++j) {
                                        const int qa = sa + q0 + j, qb = sb + q0 + j;
                                        const bool ina = q0 + j <= za_, inb = q0 + j <= zb_;
                                        const uint32_t xa = ina ? xt_ld<SMEM>(tab, ent[qa]) & kTickMask : 0u;
                                        const uint32_t xb = inb ? xt_ld<SMEM>(tab, ent[qb]) & kTickMask : 0u;
                                        moa = max(moa, xa), mob = max(mob, xb);
                                        if (qa != pa) mxa = max(mxa, xa);
                                        if (qb != pb) mxb = max(mxb, xb);
                                    }
                                }
                                if constexpr (kLanesPer == 2) {  // the other half's maxima (0 where not gathered)
                                    moa = max(moa, __shfl_xor_sync(pair, moa, kRows));
                                    mxa = max(mxa, __shfl_xor_sync(pair, mxa, kRows));
                                    mob = max(mob, __shfl_xor_sync(pair, mob, kRows));
                                    mxb = max(mxb, __shfl_xor_sync(pair, mxb, kRows));
                                }
                                const uint32_t voa = xt_ld<SMEM>(tab, ea_), vob = xt_ld<SMEM>(tab, eb_);
                                const uint32_t vna = xt_ld<SMEM>(tab, na), vnb = xt_ld<SMEM>(tab, nb);
                                const int da = (int)mkspan<NEG>(max(mxa, vna & kTickMask), p.cofs) -
                                               (int)mkspan<NEG>(moa, p.cofs);
                                const int db = (int)mkspan<NEG>(max(mxb, vnb & kTickMask), p.cofs) -
                                               (int)mkspan<NEG>(mob, p.cofs);
                                const int dx = (int)(vna & kTickMask) + (int)(vnb & kTickMask) - (int)(voa & kTickMask) -
                                               (int)(vob & kTickMask);
                                const long long dtot = (long long)dx + (long long)da * (n - 1 - ea) + (long long)db * (n - 1 - eb);
                                const int dA = (int)(vna >> 31) + (int)(vnb >> 31) - (int)(voa >> 31) - (int)(vob >> 31);
                                const bool dead = (pa >> 5) >= u_live && e_dead + (long long)min(0, min(da, da + db)) > dg;
                                int n_g = nm_cur + dA;
                                bool bnd = false;
                                const int nc = min(u_live, kLiveCap), ua = pa >> 5, ub = pb >> 5;
                                if (!dead && da >= 0 && da + db >= 0 && ua < nc && (ub < nc || ub >= u_live)) {
                                    // the moved requests' SLO tests before and after, certified on the grid
                                    bool amb = false;
                                    auto met_old = [&](int q, uint32_t v) {
                                        if (v & kAlways) return 1;
                                        const int sg = sig[q];
                                        const uint32_t mq = (uint32_t)cert_margin(q);
                                        amb = amb || (sg != INT_MIN && (uint32_t)sg + mq <= 2u * mq);
                                        return sg != INT_MIN && sg >= 0 ? 1 : 0;
                                    };
                                    auto met_new = [&](int q, uint32_t v, uint32_t e, long long shift) {
                                        if (v & kAlways) return 1;
                                        const long long D = __ldg(p.dt + e);
                                        const long long sl = D - (cE[q >> 5] + (long long)bst[q] + shift);
                                        const uint32_t mq = (uint32_t)cert_margin(q);
                                        amb = amb || (D >= 0 && (unsigned long long)(sl + mq) <= 2ull * mq);
                                        return D >= 0 && sl >= 0 ? 1 : 0;
                                    };
                                    int up = met_new(pa, vna, na, 0) - met_old(pa, voa);
                                    if (ub < nc) up += met_new(pb, vnb, nb, da) - met_old(pb, vob);
                                    else up += (int)(vnb >> 31) - (int)(vob >> 31);  // dead region: only +inf deadlines
                                    bnd = !amb;
                                    n_g = nm_cur + up;
                                }
                                if (dead || bnd) {
                                    const double f_g = objective_fast(n_g, (double)(tot + dtot) * p.tick);
                                    const float x_g = (float)((f - f_g) * sinv);
                                    const uint32_t uw = rl[kAccWord] >> 8;
                                    const bool acc = f_g > f || (float)uw * 0x1.0p-24f < __expf(-x_g);
                                    rej = !acc && (dead || (x_g >= 17.0f && uw != 0u));
                                }
                                span = (unsigned)(ea - sa + eb - sb + 2);
                            }
                        }
                        lead_c = __ballot_sync(FULL, rej && h == 0);
                        span_c = span, pk_c = pk;
                        pass_it0 = it, pass_end = it + G;
                    }
                    // consume the leading rejected run from proposal it
                    const int g0 = it - pass_it0, G = pass_end - pass_it0;
                    const int k = min(__ffsll(~(unsigned long long)(lead_c >> g0)) - 1, G - g0);
#ifndef SLO_DIAG
                    sc1 += __reduce_add_sync(FULL, lane >= g0 && lane < g0 + k ? span_c : 0u);
#endif
                    props += (unsigned)k;
#ifdef SLO_SPEC_COUNT
                    sc2 += (unsigned)k << 16;  // diagnostics: proposals consumed by this stage
#endif
                    it += k;
                    if (it == pass_end) {
                        --it;  // the loop increment moves on to the next unconsumed proposal
                        continue;
                    }
                }
                const uint32_t* rw = rnd + rnd_stride<UPL>() * (it & (kRows - 1));
                const uint32_t pk = __shfl_sync(FULL, pk_c, it - pass_it0);  // the pass decoded it
                const uint32_t op = pk >> 30;
                const int kind = op == 3u ? 0 : (op == 2u ? 2 : 1);
#ifdef SLO_DIAG
                if (kind == 2) {  // diagnostics (tools/spec_diag.py): why a proposal took this path
                    const int a0 = (int)(pk & 0x1fffu), b0 = (int)((pk >> 13) & 0x1fffu);
                    if ((min(a0, b0) >> 5) < u_live) sc2 += 1u << 16;  // live-region swap
                    else sc1 += 1u;                                     // accept / shift into the live region
                } else if (kind == 1) {
                    sc2 += 1u;  // squeeze / delay
                }
#endif

                // ---- apply in place (undo on reject) and score from the rebuilt batches
                LaneState<UPL> nx = cur;
                bool need[UPL] = {}, shf[UPL] = {};
                // live units of the committed state (cached slacks) whose contents and batch
                // structure the move leaves alone and whose anchor only shifts: count by ballot
                auto take_cached = [&]() {
                    if constexpr (UPL == 1) {
                        const bool ch = need[0] && shf[0] && lane < min(u_live, kLiveCap);
                        unsigned cm = __ballot_sync(FULL, ch);
                        const int dE = (int)(nx.E[0] - cur.E[0]);
                        bool walk = false;  // a slack the grid cannot certify: walk the unit
                        while (cm) {
                            const int ln = __ffs(cm) - 1;
                            cm &= cm - 1;
                            const int d = __shfl_sync(FULL, dE, ln);
                            const int sg = sig[(ln << 5) + lane];
                            const int cnt = __popc(__ballot_sync(FULL, sg >= d));
                            // |sg - d| <= cert_margin(q), in wrapping u32 arithmetic (|sg - d| < 2^31 + 2^28)
                            const uint32_t mq = (uint32_t)cert_margin((ln << 5) + lane);
                            const bool amb = __any_sync(FULL, sg != INT_MIN && (uint32_t)sg - (uint32_t)d + mq <= 2u * mq);
                            if (lane == ln) nx.W[0] = cnt, walk = amb;
                        }
                        need[0] = need[0] && (!ch || walk);
                    }
                };
                long long dtot = 0;
                int dA = 0;
                int q = 0;
                uint16_t old_q = 0;
                uint32_t ow0 = 0, ow1 = 0;
                int w0 = 0, w1 = 0;
                uint32_t sw_na = 0, sw_nb = 0;
                int sw_pa = 0, sw_pb = 0;
                bool sw_applied = false;  // swap written to shared memory
                int r_lo = 0, r_hi = -1;   // squeeze / delay: the rebuilt range
                if (kind == 1) {
                    const Move mv = range_move(ent, bits, n, magic, op, (int)(pk & 0x1fffu));
                    r_lo = mv.lo, r_hi = mv.hi;
                    // squeeze / delay: [lo, hi] held old batches [lo, osp], (osp, hi] and holds
                    // new batches [lo, nsp], (nsp, hi] (either part may be empty)
                    q = mv.lo + lane;
                    const bool act = q <= mv.hi;
                    uint16_t nw = 0;
                    if (act) {
                        int s = q;
                        if (mv.dir > 0) s = q == mv.ra ? mv.rb : (q > mv.ra && q <= mv.rb ? q - 1 : q);
                        else s = q == mv.rb ? mv.ra : (q >= mv.ra && q < mv.rb ? q + 1 : q);
                        old_q = ent[q];
                        const uint32_t se = ent[s];
                        const uint32_t idx = se - __umulhi(se, magic) * nn;
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
                    const int lo = mv.lo, hi = mv.hi;
                    const int osp = mv.clr >= 0 ? mv.clr : hi, nsp = mv.split;
                    const uint32_t vo = act ? xt_ld<SMEM>(tab, old_q) : 0u;
                    const uint32_t vn = act ? xt_ld<SMEM>(tab, nw) : 0u;
                    const uint32_t xo = vo & kTickMask, xn = vn & kTickMask;
                    const uint32_t mO0 = mkspan<NEG>(__reduce_max_sync(FULL, q <= osp ? xo : 0u), p.cofs);
                    const uint32_t mO1 = mkspan<NEG>(__reduce_max_sync(FULL, q > osp ? xo : 0u), p.cofs);
                    const uint32_t mN0 = mkspan<NEG>(__reduce_max_sync(FULL, q <= nsp ? xn : 0u), p.cofs);
                    const uint32_t mN1 = mkspan<NEG>(__reduce_max_sync(FULL, q > nsp ? xn : 0u), p.cofs);
                    const long long sN = __reduce_add_sync(FULL, xn), sO = __reduce_add_sync(FULL, xo);
                    dA = __popc(__ballot_sync(FULL, (vn & kAlways) != 0u)) - __popc(__ballot_sync(FULL, (vo & kAlways) != 0u));
                    // makespan * positions-after products: 27 x 12 bits, one widening multiply each
                    const uint32_t after_hi = (uint32_t)(n - 1 - hi);
                    unsigned long long oc, nc;
                    int omk, nmk;
                    if (osp < hi) oc = mulw(mO0, (uint32_t)(n - 1 - osp)) + mulw(mO1, after_hi), omk = (int)(mO0 + mO1);
                    else oc = mulw(mO0, after_hi), omk = (int)mO0;
                    if (nsp < lo) nc = mulw(mN1, after_hi), nmk = (int)mN1;
                    else if (nsp < hi) nc = mulw(mN0, (uint32_t)(n - 1 - nsp)) + mulw(mN1, after_hi), nmk = (int)(mN0 + mN1);
                    else nc = mulw(mN0, after_hi), nmk = (int)mN0;
                    dtot = sN - sO + (long long)(nc - oc);
                    const int delta = nmk - omk;
#pragma unroll
                    for (int kk = 0; kk < UPL; ++kk) {
                        const int pu = (lane * UPL + kk) << 5;
                        if (pu > hi) {
                            nx.E[kk] += delta;
                        } else if (pu >= lo) {
                            const long long Eb = nx.E[kk] - ((osp < hi && pu > osp) ? (long long)mO0 : 0ll);
                            nx.E[kk] = Eb + ((nsp >= lo && pu > nsp) ? (long long)mN0 : 0ll);
                            nx.F[kk] = pu > nsp ? mN1 : mN0;
                        }
                        need[kk] = pu + 31 >= lo && (pu <= hi || delta != 0) && nx.E[kk] <= dg;
                        shf[kk] = pu > hi;
                    }
                    take_cached();
#ifndef SLO_DIAG
                    sc1 += (unsigned)(hi - lo + 1);
#endif
                    __syncwarp();
                } else if (kind == 2) {
                    // swap: batches [sa, ea] and [sb, eb] (sa < sb, or the same batch) keep their
                    // sizes; lanes 0-15 cover the first, 16-31 the second
                    int pa, pb, sa, sb, ea, eb, da, db;
                    uint32_t na, nb, mN0, mN1;
                    {
                        const int sa0 = (int)(pk & 0x1fffu), sb0 = (int)((pk >> 13) & 0x1fffu);
                        pa = min(sa0, sb0), pb = max(sa0, sb0);
                        const uint32_t ea_ = ent[pa], eb_ = ent[pb];
                        ow0 = ea_, ow1 = eb_;
                        const uint32_t za = __umulhi(ea_, magic);  // batch size - 1
                        const uint32_t zb = __umulhi(eb_, magic);
                        const uint32_t ba = za * nn, bb = zb * nn;
                        na = ba + (eb_ - bb), nb = bb + (ea_ - ba);
                        sa = prev_end16(bits, pa) + 1, sb = prev_end16(bits, pb) + 1;
                        ea = sa + (int)za, eb = sb + (int)zb;
                        const bool first = lane < 16;
                        q = first ? sa + lane : sb + lane - 16;
                        const bool act = q <= (first ? ea : eb);
                        uint32_t eo = 0, en = 0;
                        if (act) {
                            eo = ent[q];
                            en = q == pa ? na : (q == pb ? nb : eo);
                        }
                        const uint32_t vo = act ? xt_ld<SMEM>(tab, eo) : 0u;
                        const uint32_t vn = act ? xt_ld<SMEM>(tab, en) : 0u;
                        const uint32_t xo = vo & kTickMask, xn = vn & kTickMask;
                        const uint32_t mO0 = mkspan<NEG>(__reduce_max_sync(FULL, first ? xo : 0u), p.cofs);
                        const uint32_t mO1 = mkspan<NEG>(__reduce_max_sync(FULL, first ? 0u : xo), p.cofs);
                        mN0 = mkspan<NEG>(__reduce_max_sync(FULL, first ? xn : 0u), p.cofs);
                        mN1 = mkspan<NEG>(__reduce_max_sync(FULL, first ? 0u : xn), p.cofs);
                        const long long sN = __reduce_add_sync(FULL, xn), sO = __reduce_add_sync(FULL, xo);
                        dA = __popc(__ballot_sync(FULL, (vn & kAlways) != 0u)) - __popc(__ballot_sync(FULL, (vo & kAlways) != 0u));
                        da = (int)mN0 - (int)mO0, db = (int)mN1 - (int)mO1;
                        dtot = sN - sO + (long long)da * (n - 1 - ea) + (long long)db * (n - 1 - eb);
                        if (sa == sb) dtot = 0, dA = 0;  // one batch: order inside a batch changes nothing
                        r_lo = sa, r_hi = eb;
                    }
                    // the swap is written to shared memory only when an SLO walk or an accept needs
                    // it (the common rejected swap never touches the state)
                    sw_na = na, sw_nb = nb, sw_pa = pa, sw_pb = pb;
#pragma unroll
                    for (int kk = 0; kk < UPL; ++kk) {
                        const int pu = (lane * UPL + kk) << 5;
                        if (pu > eb) nx.E[kk] += da + db;
                        else if (pu >= sb) nx.E[kk] += da, nx.F[kk] = mN1;
                        else if (pu > ea) nx.E[kk] += da;
                        else if (pu >= sa) nx.F[kk] = mN0;
                        // contents (the units of pa, pb) or anchors (F of a rebuilt batch, E after it) changed
                        const int u = lane * UPL + kk;
                        const bool chg = u == (pa >> 5) || u == (pb >> 5) || (pu >= sa && da != 0) || (pu >= sb && db != 0);
                        need[kk] = chg && nx.E[kk] <= dg;
                        shf[kk] = u != (pa >> 5) && u != (pb >> 5) && !(pu >= sa && pu <= ea) && !(pu >= sb && pu <= eb);
                    }
                    take_cached();
#ifndef SLO_DIAG
                    sc1 += (unsigned)(ea - sa + eb - sb + 2);
#endif
                    bool any = false;
#pragma unroll
                    for (int kk = 0; kk < UPL; ++kk) any |= need[kk];
                    if (__any_sync(FULL, any)) {  // the walks read the proposed state
                        __syncwarp();
                        if (lane == 0) ent[pa] = (uint16_t)na, ent[pb] = (uint16_t)nb;
                        __syncwarp();
                        sw_applied = true;
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < UPL; ++kk) need[kk] = false;
                }
                walk_units<UPL, SMEM, NEG>(need, nx, ent, bits, tab, p.dt, n, mb, p.cofs, lane, sc2);
                const long long tot_new = tot + dtot;
                const int A_new = A + dA;
                const int nm = A_new + live_met<UPL>(nx, dg);
                const double t_new = (double)tot_new * p.tick;
                const double f_new = objective_fast(nm, t_new);
                ++props;
                bool accept = f_new > f;  // Metropolis (P:src/priority_mapper.cpp:385-391)
                if (!accept) {
                    // x = (f - f_new) * scale / t; the test u < exp(-x) runs on the SFU in fp32
                    // with a 24-bit uniform (acceptance probabilities within ~1e-7 of exact)
                    const float x = (float)((f - f_new) * sinv);
                    const float u = (float)(rw[kAccWord] >> 8) * 0x1.0p-24f;
                    accept = u < __expf(-x);
                }
                if (accept) {
                    ++accs;
                    if (kind == 2 && !sw_applied) {
                        __syncwarp();
                        if (lane == 0) ent[sw_pa] = (uint16_t)sw_na, ent[sw_pb] = (uint16_t)sw_nb;
                        __syncwarp();
                    }
                    if (kind == 1) {  // rebuilt batches: refresh the move flags around them
                        rebuild_flags(ent, bits, sqb, dlb, n, mb, magic, max(r_lo - mb, 0) >> 5,
                                      min(r_hi + mb, n - 1) >> 5, lane);
                        __syncwarp();
                    }
                    cur = nx, tot = tot_new, A = A_new, nm_cur = nm;
                    f = f_new;
                    need_refresh = true;
                    if (kind != 0) rf_lo = min(rf_lo, r_lo >> 5), rf_hi = max(rf_hi, r_hi >> 5);
                    pass_end = 0;  // the state changed: later speculative scores are stale
                    if (f > best_f) {
                        best_f = f;
                        copy_state<UPL>(p.best_ent + (size_t)c * kEnt, p.best_bits + (size_t)c * kBits, ent, bits,
                                        lane);
                        if (lane == 0) rc->g = objective(nm, t_new), rc->t = t_new, rc->n_met = nm;
                    }
                } else if (kind == 1 || sw_applied) {
                    __syncwarp();  // every lane is done reading the state (SLO walks) before the undo
                    if (kind == 1) {
                        if (q <= r_hi) ent[q] = old_q;
                        if (lane == 0) bits[w1] = ow1, bits[w0] = ow0;
                    } else {
                        if (lane == 0) ent[sw_pa] = (uint16_t)ow0, ent[sw_pb] = (uint16_t)ow1;
                    }
                    __syncwarp();
                }
            }
            if (n_my > 1) {  // park the chain (state + anchors) until the next level
                copy_state<UPL, 3 * kBits>(p.st_ent + (size_t)c * kEnt, p.st_bits + (size_t)c * 3 * kBits, ent, bits,
                                           lane);
                parked[(size_t)c * 32 + lane] = cur;
                __syncwarp();
            }
            if (lane == 0) {
                rc->proposals = props, rc->accepted = accs, rc->levels = lev + 1, rc->cur_f = f, rc->best_f = best_f;
                rc->cur_tot = tot, rc->cur_A = A, rc->cur_n = nm_cur;
                rc->scan1 += sc1, rc->scan2 += sc2;
            }
            if (stop) break;
        }
    }
}
