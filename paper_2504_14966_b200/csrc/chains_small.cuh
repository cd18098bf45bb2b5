// K5: the chain kernel for short queues (n <= 32: an online window's per-instance queue).
// Included by engine.cu after chains.cuh (same anonymous namespace).
//
// Same chains as K3 -- the same Philox rows (proposal, chain, block, tag), the same move decode
// (the reference's 8 + 1 attempt discipline, P:src/priority_mapper.cpp:184-198), the same tick
// objective with the SLO count certified against the reference's fp64 arithmetic and the same
// Metropolis test -- so a K5 chain follows K3's trajectory proposal for proposal and the winner
// is bit-identical (tests/test_short_queue.py: against the sequential model and against K3).
//
// What changes is the shape. At n <= 32 a schedule is one warp row: lane q holds the request at
// position q (a register), the batch ends are one warp-uniform mask. K3's machinery for long
// schedules -- shared-memory entries, unit anchors, the speculative rejection stage, cached
// slacks -- costs ~720 warp instructions per proposal at n = 6 (ncu; K5: 291), because an
// online window's short queue at high temperature accepts a quarter of its proposals and most
// moves are squeezes/delays that skip the speculative stage. K5 instead decodes the nine
// attempts on nine lanes at once, applies the move as one shuffle (rotation or exchange) plus a
// mask edit, and re-scores the whole row from scratch: segmented max, one scan, three REDUX sums.
//
// Rows: lane j < 32 draws proposal prop0 + j's 20 words into the warp's shared row buffer, as K3
// does (stride 20 words).

constexpr int kSmallMaxN = 32;
constexpr int kSmallThreads = 768;  // 24 warps (70 registers; 1024 threads cap them at 64, 512 park chains under an SM share)

struct SmallScore {
    long long tot;  // total latency (ticks)
    int A, nm;      // +inf-deadline count, SLO count (the reference's, certified)
};

// the position's batch bounds in a row whose batch ends are `ends` (bit n-1 set)
__device__ __forceinline__ void small_bounds(uint32_t ends, int lane, int& start, int& end) {
    const uint32_t below = ends & ((1u << lane) - 1u);
    start = below ? 32 - __clz(below) : 0;
    end = lane + __ffs(ends >> lane) - 1;  // lanes past the last end: garbage, never used
}

// move flags (bit q of sqb: a squeeze of q fails; of dlb: a delay of q fails), as rebuild_flags
__device__ __forceinline__ void small_flags(uint32_t ends, int n, int mb, int lane, uint32_t& sqb, uint32_t& dlb) {
    int s, e;
    small_bounds(ends, lane, s, e);
    const int size = e - s + 1;
    const int szp = __shfl_sync(FULL, size, max(s - 1, 0) & 31);
    const int szn = __shfl_sync(FULL, size, min(e + 1, 31) & 31);
    sqb = __ballot_sync(FULL, lane < n && s > 0 && szp >= mb);
    dlb = __ballot_sync(FULL, lane < n && e < n - 1 && szn >= mb);
}

// The chain objective of the row (idx at lane q = dense index of the request at position q).
// Tick total exact; SLO count certified on the grid, else decided by the reference's fp64
// left-to-right elapsed sum (exact_chunk's arithmetic, from registers).
// segmented inclusive max (segments of <= MB positions end at the set bits of w)
template <int MB>
__device__ __forceinline__ uint32_t seg_max_t(uint32_t x, uint32_t w, int lane) {
    uint32_t m = x;
    const uint32_t below = w & ((1u << lane) - 1u);
    const int span = lane - (below ? 32 - __clz(below) : 0);
#pragma unroll
    for (int d = 1; d < MB; d <<= 1) {
        const uint32_t mu = __shfl_up_sync(FULL, m, d);
        if (d <= span) m = max(m, mu);
    }
    return m;
}

template <bool NEG, int MB>
__device__ __forceinline__ SmallScore small_score(const ChainParams& p, const uint32_t* xs, const long long* ds,
                                                  uint32_t idx, uint32_t ends, int lane, uint32_t& e_out) {
    const int n = p.n, mb = p.mb;
    const bool in = lane < n;
    int s, e;
    small_bounds(ends, lane, s, e);
    const uint32_t ent = in ? (uint32_t)(e - s) * (uint32_t)n + idx : 0u;
    e_out = ent;
    const uint32_t v = in ? xs[ent] : 0u;
    const uint32_t x = in ? mkspan<NEG>(v & kTickMask, p.cofs) : 0u;
    const uint32_t m = seg_max_t<MB>(x, ends, lane);
    const uint32_t vv = ((ends >> lane) & 1u) ? m : 0u;
    uint32_t sc = vv;  // makespans of the batches closed at or before q: < 32 * 2^27
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t up = __shfl_up_sync(FULL, sc, d);
        if (lane >= d) sc += up;
    }
    const uint32_t Eq = in ? sc - vv : 0u;  // elapsed at the start of q's batch
    const bool always = in && (v & kAlways);
    const long long D = in && !always ? ds[ent] : -1ll;
    const long long sl = D - (long long)Eq;
    const unsigned marg = (unsigned)cert_margin(lane);
    const bool amb = D >= 0 && (unsigned long long)(sl + marg) <= 2ull * marg;
    unsigned met = __ballot_sync(FULL, D >= 0 && sl >= 0);
    SmallScore r;
    const unsigned long long elo = __reduce_add_sync(FULL, Eq & 0xffffu), ehi = __reduce_add_sync(FULL, Eq >> 16);
    const unsigned long long xsum = __reduce_add_sync(FULL, v & kTickMask);  // < 32 * 2^27
    r.tot = (long long)((ehi << 16) + elo + xsum) - (long long)n * p.cofs;
    r.A = __popc(__ballot_sync(FULL, always));
    if (__any_sync(FULL, amb)) {  // the reference's fp64 arithmetic (exact_chunk with E = 0, mc = 0)
        if (lane == 0 && p.exact_count) atomicAdd(p.exact_count, 1ull);
        double2 tv = make_double2(0.0, -INFINITY);
        if (in) tv = __ldg(&p.tab64[ent]);
        const uint32_t below = ends & ((1u << lane) - 1u);
        const int span = lane - (below ? 32 - __clz(below) : 0);
        double mm = tv.x;
#pragma unroll
        for (int d = 1; d < 16; d <<= 1) {
            const double mu = __shfl_up_sync(FULL, mm, d);
            if (d < mb && d <= span) mm = dmax(mm, mu);
        }
        mm = dmax(0.0, mm);
        double Ec = 0.0, Es = 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double mk = __shfl_sync(FULL, mm, k);
            if ((ends >> k) & 1u) {
                Ec = Ec + mk;
                if (lane > k) Es = Ec;
            }
        }
        met = __ballot_sync(FULL, in && tv.y != INFINITY && Es <= tv.y);
    }
    r.nm = r.A + __popc(met);
    return r;
}

template <bool NEG, int MB>
__global__ void __launch_bounds__(kSmallThreads, 1) k_chains_small(const ChainParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int n = p.n, mb = p.mb, total = n * mb;
    long long* ds = reinterpret_cast<long long*>(smem);                // [mb][n] deadline ticks
    uint32_t* xs = reinterpret_cast<uint32_t*>(smem + (size_t)total * 8);  // [mb][n] exec ticks
    const size_t tab_bytes = ((size_t)total * 12 + 15) & ~(size_t)15;
    uint32_t* rnd = reinterpret_cast<uint32_t*>(smem + tab_bytes) + (size_t)wid * 32 * kRndWords;
    for (int i = threadIdx.x; i < total; i += blockDim.x) ds[i] = p.dt[i], xs[i] = p.xt[i];
    __syncthreads();

    const int gw = blockIdx.x * W + wid, TW = gridDim.x * W;
    if (gw >= p.chain_count) return;
    const int n_my = (p.chain_count - gw + TW - 1) / TW;
    uint64_t deadline = ~0ull;
    if (p.budget_ns > 0) deadline = __shfl_sync(FULL, gtimer(), 0) + (uint64_t)p.budget_ns;

    // attempt j = lane < 8 reads the j-th base-3 digit of the ops word: floor(ops / 3^j) by a
    // 40-bit reciprocal (exact for ops < 3^8)
    unsigned long long p3m;
    {
        unsigned long long d = 1;
        for (int j = 0; j < min(lane, 8); ++j) d *= 3;
        p3m = ((1ull << 40) + d - 1) / d;  // ceil(2^40 / 3^j)
    }
    const uint32_t nn = (uint32_t)n;
    uint32_t idx = 0, ends = 0, sqb = 0, dlb = 0;
    long long tot = 0;
    int A = 0, nm_cur = 0;
    double f = 0.0, best_f = 0.0;
    unsigned props = 0, accs = 0;
    int stop = 0;

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
            uint16_t* best_e = p.best_ent + (size_t)c * 1024;
            if (lev == 0) {
                const uint32_t e0 = lane < n ? p.start_ent[lane] : 0u;
                idx = n >= 2 ? e0 - __umulhi(e0, p.magic) * nn : 0u;
                ends = p.start_bits[0];
                tot = p.start_obj[0], A = (int)p.start_obj[1], nm_cur = (int)p.start_obj[2];
                f = best_f = objective_fast(nm_cur, (double)tot * p.tick), props = 0, accs = 0;
                for (int i = lane; i < 1024 / 8; i += 32)  // the whole best slot once (k_argmax copies it)
                    reinterpret_cast<uint4*>(best_e)[i] = i < 4 ? reinterpret_cast<const uint4*>(p.start_ent)[i]
                                                                : make_uint4(0u, 0u, 0u, 0u);
                p.best_bits[(size_t)c * 32 + lane] = lane == 0 ? ends : 0u;
                if (lane == 0) rc->g = objective(nm_cur, (double)tot * p.tick), rc->t = (double)tot * p.tick, rc->n_met = nm_cur;
            } else if (n_my > 1) {  // resume a parked chain
                idx = p.st_ent[(size_t)c * 1024 + lane];
                ends = p.st_bits[(size_t)c * 96];
                tot = rc->cur_tot, A = rc->cur_A, nm_cur = rc->cur_n;
                f = rc->cur_f, best_f = rc->best_f, props = (unsigned)rc->proposals, accs = (unsigned)rc->accepted;
            }
            small_flags(ends, n, mb, lane, sqb, dlb);
            const double scale = p.n_mult > 0 ? p.scale * p.scale_mult[cid % (uint32_t)p.n_mult] : p.scale;
            const double sinv = scale * inv_t;
            const unsigned props0 = props;
            for (int it = 0; it < p.iter; ++it) {
                if ((it & 7) == 0 && it > 0 && p.budget_ns > 0 && __shfl_sync(FULL, gtimer() > deadline ? 1 : 0, 0)) {
                    stop = 1;
                    break;
                }
                if ((it & 31) == 0) {  // lane j draws the row of proposal prop + j (as K3)
                    const uint32_t prop0 = (uint32_t)(lev * p.iter + it);
                    __syncwarp();
                    uint32_t* dst = rnd + kRndWords * lane;
#pragma unroll 1
                    for (int b = 0; b < kRndBlocks; ++b) {
                        uint32_t r[4] = {prop0 + (uint32_t)lane, cid, (uint32_t)b, kTagMove};
                        philox_rounds<SLO_PHILOX_ROUNDS>(r, p.key0, p.key1);
                        reinterpret_cast<uint4*>(dst)[b] = make_uint4(r[0], r[1], r[2], r[3]);
                    }
                    __syncwarp();
                }
                const uint32_t* rl = rnd + kRndWords * (it & 31);
                // ---- decode: attempt j on lane j (j < 8), the forced swap on lane 8
                uint32_t pk = kNoMove;
                if (n >= 2) {
                    const uint32_t first = (uint32_t)__ffs(ends);  // size of the first batch
                    uint32_t pl = kNoMove;
                    bool valid = false;
                    if (lane < 8) {
                        const uint32_t ops = lemire32(rl[kOpsWord], 6561u);
                        const uint32_t op = (uint32_t)(((unsigned long long)ops * p3m) >> 40) % 3u;
                        const uint32_t r1 = rl[pos_word(lane)], r2 = rl[pos_word(lane) + 1];
                        const uint32_t a = lemire32(r1, nn);
                        const uint32_t ps = first + lemire32(r1, nn - first);
                        uint32_t b = lemire32(r2, nn - 1);
                        b += b >= a ? 1u : 0u;
                        const uint32_t pos = op == 0 ? ps : a;
                        const uint32_t qf = min(pos, nn - 1);
                        const bool fails = ((op == 0 ? sqb : dlb) >> qf) & 1u;
                        valid = op == 2u || (!fails && (op == 1u || first < nn));
                        pl = op << 30 | pos | (op == 2u ? b << 13 : 0u);
                    } else if (lane == 8) {
                        const uint32_t a8 = lemire32(rl[pos_word(kAttempts - 1)], nn);
                        uint32_t b8 = lemire32(rl[pos_word(kAttempts - 1) + 1], nn - 1);
                        b8 += b8 >= a8 ? 1u : 0u;
                        pl = 2u << 30 | a8 | b8 << 13;
                        valid = true;
                    }
                    const unsigned vm = __ballot_sync(FULL, valid);
                    pk = __shfl_sync(FULL, pl, __ffs(vm) - 1);
                }
                // ---- apply: a rotation (squeeze / delay) or an exchange (swap) of the row
                const uint32_t op = pk >> 30;
                int src = lane;
                uint32_t ends2 = ends;
                if (op == 2u) {
                    const int a0 = (int)(pk & 0x1fffu), b0 = (int)((pk >> 13) & 0x1fffu);
                    src = lane == a0 ? b0 : (lane == b0 ? a0 : lane);
                } else if (op == 0u) {  // squeeze: pos joins the previous batch (rotation right on [sk, pos])
                    const int pos = (int)(pk & 0x1fffu);
                    const uint32_t below = ends & ((1u << pos) - 1u);
                    const int sk = below ? 32 - __clz(below) : 0;
                    src = lane == sk ? pos : (lane > sk && lane <= pos ? lane - 1 : lane);
                    ends2 = (ends & ~(1u << (sk - 1))) | (1u << sk);
                } else if (op == 1u) {  // delay: pos goes to the end of the next batch (rotation left)
                    const int pos = (int)(pk & 0x1fffu);
                    const int ek = pos + __ffs(ends >> pos) - 1;
                    int rb;
                    if (ek < n - 1) {
                        rb = ek + __ffs(ends >> (ek + 1));
                        ends2 = (ends & ~(1u << ek)) | (ek >= 1 ? 1u << (ek - 1) : 0u);
                    } else {
                        rb = n - 1;
                        ends2 = ends | (n >= 2 ? 1u << (n - 2) : 0u);
                    }
                    src = lane == rb ? pos : (lane >= pos && lane < rb ? lane + 1 : lane);
                }
                const uint32_t idx2 = __shfl_sync(FULL, idx, src);
                uint32_t e2;
                const SmallScore sc = small_score<NEG, MB>(p, xs, ds, idx2, ends2, lane, e2);
                const double t_new = (double)sc.tot * p.tick;
                const double f_new = objective_fast(sc.nm, t_new);
                ++props;
                bool accept = f_new > f;  // Metropolis (P:src/priority_mapper.cpp:385-391), as K3
                if (!accept) {
                    const float x = (float)((f - f_new) * sinv);
                    const float u = (float)(rl[kAccWord] >> 8) * 0x1.0p-24f;
                    accept = u < __expf(-x);
                }
                if (accept) {
                    ++accs;
                    if (ends2 != ends) small_flags(ends2, n, mb, lane, sqb, dlb);
                    idx = idx2, ends = ends2, tot = sc.tot, A = sc.A, nm_cur = sc.nm, f = f_new;
                    if (f > best_f) {
                        best_f = f;
                        best_e[lane] = (uint16_t)e2;
                        if (lane == 0) {
                            p.best_bits[(size_t)c * 32] = ends;
                            rc->g = objective(sc.nm, t_new), rc->t = t_new, rc->n_met = sc.nm;
                        }
                    }
                }
            }
            if (n_my > 1) {  // park the chain until the next level
                p.st_ent[(size_t)c * 1024 + lane] = (uint16_t)idx;
                if (lane == 0) p.st_bits[(size_t)c * 96] = ends;
            }
            if (lane == 0) {
                rc->proposals = props, rc->accepted = accs, rc->levels = lev + 1, rc->cur_f = f, rc->best_f = best_f;
                rc->cur_tot = tot, rc->cur_A = A, rc->cur_n = nm_cur;
                rc->scan1 += (unsigned long long)(props - props0) * (unsigned)n;  // positions scored
            }
            if (stop) break;
        }
    }
}

__host__ __device__ constexpr size_t small_warp_bytes() { return 32 * kRndWords * 4; }
