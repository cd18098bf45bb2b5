// K2: exact replay of the reference walk, one warp per chain. Included by engine.cu.
//
// Bit-identical to anneal() (P:src/priority_mapper.cpp:340-411) driven by Rng(seed + chain):
// the xoshiro256++ stream is stepped redundantly by every lane (warp-uniform), moves follow
// FlatSchedule's draw discipline (:141-198) on the entry/bitmask representation of K3, and the
// score is the reference's sequential arithmetic (:259-279). The score is incremental yet exact:
// the sequential running state (total, n_met, elapsed) is cached every 16 positions, so a
// proposal restarts the exact left-to-right pass just before the first position it changed.
// The (exec, deadline) pairs and batch makespans of every position stay staged in shared memory;
// a move restages only the (at most 32) positions of the batches it rebuilds, lane-parallel, and
// undoes them on rejection; lane 0 then runs the two dependence chains from shared memory.

struct ReplayParams {
    int n, mb, chains;
    uint64_t magic;      // floor(2^32 / n) + 1
    const double2* tab;  // global [mb][n]
    double t0, t_thres, tau, scale;
    int iter;
    uint64_t seed;
    const uint16_t* start_ent;   // [npad] combined entries of the start schedule
    const uint32_t* start_bits;  // [npad / 32]
    uint16_t* best_ent;          // [chains][npad]
    uint32_t* best_bits;         // [chains][npad / 32]
    ChainRec* rec;
    int npad;                    // n rounded up to 32
};

struct XoshiroW {  // P:include/slosched/rng.hpp:14-57, stepped identically by every lane
    uint64_t s0, s1, s2, s3;
    __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    __device__ explicit XoshiroW(uint64_t seed) {
        uint64_t z = seed;
        uint64_t* s[4] = {&s0, &s1, &s2, &s3};
        for (int i = 0; i < 4; ++i) {
            z += 0x9e3779b97f4a7c15ULL;
            uint64_t v = z;
            v = (v ^ (v >> 30)) * 0xbf58476d1ce4e5b9ULL;
            v = (v ^ (v >> 27)) * 0x94d049bb133111ebULL;
            *s[i] = v ^ (v >> 31);
        }
    }
    __device__ uint64_t next() {
        const uint64_t out = rotl(s0 + s3, 23) + s0;
        const uint64_t t = s1 << 17;
        s2 ^= s0, s3 ^= s1, s1 ^= s2, s0 ^= s3, s2 ^= t;
        s3 = rotl(s3, 45);
        return out;
    }
    __device__ double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
    __device__ uint64_t index(uint64_t n) {
        uint64_t x = next();
        uint64_t lo = x * n, hi = __umul64hi(x, n);
        if (lo < n) {
            const uint64_t thr = (0 - n) % n;
            while (lo < thr) x = next(), lo = x * n, hi = __umul64hi(x, n);
        }
        return hi;
    }
};

// One proposal with FlatSchedule's exact draw order; returns the move (kind 0: none applied).
__device__ __forceinline__ Move replay_propose(const uint16_t* ent, const uint32_t* bits, int n, int mb,
                                               uint64_t magic, XoshiroW& rng) {
    auto size_at = [&](int q) { return (int)(((uint64_t)ent[q] * magic) >> 32) + 1; };
    Move mv{};
    if (n == 0) return mv;
    auto swap_move = [&]() {
        Move m{};
        if (n < 2) return m;  // apply_swap returns false before drawing
        const int a = (int)rng.index((uint64_t)n);
        int b = (int)rng.index((uint64_t)(n - 1));
        if (b >= a) ++b;
        m.kind = 2, m.a = a, m.b = b;
        return m;
    };
    for (int attempt = 0; attempt < 8; ++attempt) {
        const uint64_t op = rng.index(3);
        if (op == 0) {  // apply_squeeze, :141-153
            const int first = size_at(0);
            if (first >= n) continue;  // fewer than two batches: no draw
            const int pos = first + (int)rng.index((uint64_t)(n - first));
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
        } else if (op == 1) {  // apply_delay, :155-170
            const int pos = (int)rng.index((uint64_t)n);
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
        } else {  // apply_swap, :172-180
            mv = swap_move();
            if (mv.kind) return mv;
        }
    }
    return swap_move();  // :197
}

// per-warp slot (~27 B per position): staged {exec, makespan-at-batch-end} pairs, deadlines,
// entries, bits, one trailing partial makespan per 32-position window, and the sequential
// running state {total, elapsed}, n_met before every 16-position block
__host__ __device__ constexpr size_t replay_trail_off(int npad) {
    return ((size_t)npad * (16 + 8 + 2) + (size_t)(npad / 32) * 4 + 15) & ~(size_t)15;
}
__host__ __device__ constexpr size_t replay_cache_off(int npad) {
    return (replay_trail_off(npad) + (size_t)(npad / 32) * 8 + 15) & ~(size_t)15;
}
__host__ __device__ constexpr size_t replay_slot_bytes(int npad) {
    return (replay_cache_off(npad) + (size_t)(npad / 16 + 1) * (16 + 4) + 15) & ~(size_t)15;
}

__global__ void __launch_bounds__(128) k_replay(const ReplayParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * (blockDim.x >> 5) + wid;
    if (c >= p.chains) return;
    const int n = p.n, mb = p.mb, npad = p.npad;
    const uint32_t nn = (uint32_t)n;
    unsigned char* base = smem + (size_t)wid * replay_slot_bytes(npad);
    double2* xa = reinterpret_cast<double2*>(base);  // {exec, elapsed increment after q}
    double* dl = reinterpret_cast<double*>(xa + npad);
    uint16_t* ent = reinterpret_cast<uint16_t*>(dl + npad);
    uint32_t* bits = reinterpret_cast<uint32_t*>(ent + npad);
    const int words = npad / 32;
    double* trail = reinterpret_cast<double*>(base + replay_trail_off(npad));
    double2* c_te = reinterpret_cast<double2*>(base + replay_cache_off(npad));  // {total, elapsed}
    int* c_nmet = reinterpret_cast<int*>(c_te + npad / 16 + 1);
    for (int i = lane; i < npad; i += 32) ent[i] = p.start_ent[i];
    for (int i = lane; i < words; i += 32) bits[i] = p.start_bits[i];
    if (lane == 0) c_te[0] = make_double2(0.0, 0.0), c_nmet[0] = 0;
    __syncwarp();

    // The reference's sequential score (:259-279), restarted at the 16-aligned position r whose
    // running state {total, elapsed, n_met} is cached (every position before r unchanged).
    // Operand gathers and the batch makespans (a max is exact in any order) are lane-parallel
    // from s0, the start of r's batch; the dependence chains run on lane 0 with the
    // reference's arithmetic per position: met += elapsed <= deadline, total += elapsed + exec,
    // and elapsed += makespan at a batch end (elsewhere += 0.0, an exact no-op).
    // {exec, makespan increment} and deadline of every position from s0 (the start of a batch):
    // the whole schedule once; afterwards a move restages only the batches it rebuilds
    auto stage_from = [&](int s0) {
        const int nw = (n - s0 + 31) >> 5;
        // windows of 32 are independent: a segmented max-scan over the lanes; a batch crossing
        // into window w takes window w-1's trailing partial max in the fix-up (batches <= 16)
#pragma unroll 2
        for (int w = 0; w < nw; ++w) {
            const int q = s0 + (w << 5) + lane;
            double x = 0.0;
            bool end = false;
            if (q < n) {
                const double2 v = __ldg(&p.tab[ent[q]]);
                x = v.x, dl[q] = v.y;
                end = (bits[q >> 5] >> (q & 31)) & 1u;
            }
            const unsigned below = __ballot_sync(FULL, end) & ((1u << lane) - 1u);
            const int seg = below ? 32 - __clz(below) : 0;
            double m = x;
#pragma unroll
            for (int d = 1; d < 16; d <<= 1) {
                const double o = __shfl_up_sync(FULL, m, d);
                if (lane - d >= seg) m = dmax(m, o);
            }
            // the reference's makespan starts at 0.0 (:267-273): a batch of negative execs adds 0
            if (q < n) xa[q] = make_double2(x, end ? dmax(0.0, m) : 0.0);
            if (lane == 31) trail[w] = end ? 0.0 : m;
        }
        __syncwarp();
        for (int w = 1 + lane; w < nw; w += 32) {
            const int q0 = s0 + (w << 5);
            if (!((bits[(q0 - 1) >> 5] >> ((q0 - 1) & 31)) & 1u)) {
                const int e = next_end(bits, q0);
                xa[e].y = dmax(xa[e].y, trail[w - 1]);
            }
        }
        __syncwarp();
    };
    auto score_from = [&](int r, double& total_out, int& nmet_out) -> double {
        double total = 0.0;
        int nm = 0;
        if (lane == 0) {
            const double2 st = c_te[r >> 4];
            total = st.x;
            double el = st.y;
            nm = c_nmet[r >> 4];
            // 16-position blocks, one cache entry each; the operands are read from shared memory
            // inside the unrolled block (tools/probes/chain_loop.cu: 13.4 cycles per position,
            // where double-buffering 16 positions in registers measured 15.3 and cost the kernel
            // its registers)
            int q = r;
            for (; q + 16 <= n; q += 16) {
                c_te[q >> 4] = make_double2(total, el), c_nmet[q >> 4] = nm;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const double2 v = xa[q + j];
                    nm += el <= dl[q + j];
                    total += el + v.x;
                    el += v.y;
                }
            }
            if (q < n) {
                c_te[q >> 4] = make_double2(total, el), c_nmet[q >> 4] = nm;
                for (; q < n; ++q) {
                    const double2 v = xa[q];
                    nm += el <= dl[q];
                    total += el + v.x;
                    el += v.y;
                }
            }
        }
        __syncwarp();
        total = __shfl_sync(FULL, total, 0);
        nm = __shfl_sync(FULL, nm, 0);
        total_out = total, nmet_out = nm;
        return total > 0.0 ? (double)nm / total : 0.0;  // :278
    };

    double tot0;
    int nm0;
    stage_from(0);
    double f = score_from(0, tot0, nm0);
    int valid_end = n;  // block caches are valid at every boundary <= valid_end
    double best_f = f, best_t = tot0;
    int best_n = nm0;
    for (int i = lane; i < npad; i += 32) p.best_ent[(size_t)c * npad + i] = ent[i];
    for (int i = lane; i < words; i += 32) p.best_bits[(size_t)c * words + i] = bits[i];
    XoshiroW rng(p.seed + (uint64_t)c);
    unsigned long long props = 0, accs = 0;
    int levels = 0;
#ifdef SLO_K2_TIMING
    long long t_score = 0, t_pre = 0;  // cycles: score_from / propose + apply + restage
#endif
    for (double t = p.t0; t >= p.t_thres; t *= p.tau, ++levels) {
        for (int k = 0; k < p.iter; ++k) {
#ifdef SLO_K2_TIMING
            const long long tk0 = clock64();
#endif
            const Move mv = replay_propose(ent, bits, n, mb, p.magic, rng);
            // apply in place (identical to the chain kernel), remember how to undo
            int q = 0, lo_pos = n;
            uint16_t old_q = 0;
            uint32_t ow0 = 0, ow1 = 0;
            int w0 = 0, w1 = 0;
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
                    const uint32_t idx = se - (uint32_t)(((uint64_t)se * p.magic) >> 32) * nn;
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
                lo_pos = mv.lo;
            } else if (mv.kind == 2) {
                const uint32_t ea = ent[mv.a], eb = ent[mv.b];
                ow0 = ea, ow1 = eb;
                const uint32_t ba = (uint32_t)(((uint64_t)ea * p.magic) >> 32) * nn;
                const uint32_t bb = (uint32_t)(((uint64_t)eb * p.magic) >> 32) * nn;
                __syncwarp();
                if (lane == 0) ent[mv.a] = (uint16_t)(ba + (eb - bb)), ent[mv.b] = (uint16_t)(bb + (ea - ba));
                __syncwarp();
                lo_pos = min(mv.a, mv.b);
            }
            // restage the rebuilt batches (<= 32 positions, one per lane): exec, deadline and the
            // makespan increment at each batch end (the reference's max from 0.0, :267-273)
            int qs = -1, grp = 0;
            if (mv.kind == 1) {
                if (mv.lo + lane <= mv.hi) qs = mv.lo + lane, grp = qs <= mv.split ? 0 : 1;
            } else if (mv.kind == 2) {
                const int pa = min(mv.a, mv.b), pb = max(mv.a, mv.b);
                const int sa = prev_end(bits, pa) + 1, sb = prev_end(bits, pb) + 1;
                const int ea = next_end(bits, pa), eb = next_end(bits, pb);
                if (lane < 16) {
                    if (sa + lane <= ea) qs = sa + lane;
                } else if (sb != sa && sb + lane - 16 <= eb) {
                    qs = sb + lane - 16, grp = 1;
                }
            }
            double2 old_xa = make_double2(0.0, 0.0);
            double old_dl = 0.0;
            if (mv.kind) {
                double x = 0.0, d = 0.0;
                if (qs >= 0) {
                    const double2 v = __ldg(&p.tab[ent[qs]]);
                    x = v.x, d = v.y;
                    old_xa = xa[qs], old_dl = dl[qs];
                }
                double m0 = qs >= 0 && grp == 0 ? x : -INFINITY, m1 = qs >= 0 && grp == 1 ? x : -INFINITY;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    m0 = dmax(m0, __shfl_xor_sync(FULL, m0, o));
                    m1 = dmax(m1, __shfl_xor_sync(FULL, m1, o));
                }
                if (qs >= 0) {
                    const bool end = (bits[qs >> 5] >> (qs & 31)) & 1u;
                    xa[qs] = make_double2(x, end ? dmax(0.0, grp ? m1 : m0) : 0.0);
                    dl[qs] = d;
                }
                __syncwarp();
            }
            // restart at the last cached block boundary before the first changed position (or
            // earlier if a rejected proposal left the later caches stale)
            const int r0 = min(lo_pos, valid_end) & ~15;
            double tot;
            int nm;
#ifdef SLO_K2_TIMING
            const long long tk1 = clock64();
#endif
            const double f_new = mv.kind ? score_from(r0, tot, nm) : (tot = 0.0, nm = 0, f);
#ifdef SLO_K2_TIMING
            const long long tk2 = clock64();
            t_score += tk2 - tk1, t_pre += tk1 - tk0;
#endif
            ++props;
            bool accept = f_new > f;  // :385-391
            if (!accept) {
                const double x = (f - f_new) * p.scale / t;
                const double u = rng.uniform();
                accept = u < exp(-x);
            }
            if (accept) {
                ++accs;
                f = f_new;
                if (mv.kind) valid_end = n;
                if (f > best_f) {
                    best_f = f, best_t = tot, best_n = nm;
                    for (int i = lane; i < npad; i += 32) p.best_ent[(size_t)c * npad + i] = ent[i];
                    for (int i = lane; i < words; i += 32) p.best_bits[(size_t)c * words + i] = bits[i];
                }
            } else if (mv.kind) {
                if (qs >= 0) xa[qs] = old_xa, dl[qs] = old_dl;
                if (mv.kind == 1) {
                    if (q <= mv.hi) ent[q] = old_q;
                    if (lane == 0) bits[w1] = ow1, bits[w0] = ow0;
                } else if (lane == 0) {
                    ent[mv.a] = (uint16_t)ow0, ent[mv.b] = (uint16_t)ow1;
                }
                __syncwarp();
                valid_end = r0;  // caches past r0 describe the rejected state
            }
        }
    }
    if (lane == 0) {
        ChainRec r;
        r.g = best_f, r.t = best_t, r.cur_f = f, r.n_met = best_n, r.levels = levels;
        r.proposals = props, r.accepted = accs, r.scan1 = 0, r.scan2 = 0;
#ifdef SLO_K2_TIMING
        r.scan1 = (unsigned long long)t_score, r.scan2 = (unsigned long long)t_pre;  // diagnostics
#endif
        p.rec[c] = r;
    }
}

