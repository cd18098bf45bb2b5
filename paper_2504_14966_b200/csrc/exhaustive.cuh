// Exhaustive search over every permutation x every batch-size composition (the reference's
// small-n oracle, P:src/priority_mapper.cpp:413-517), one candidate stream per thread.
// Included by engine.cu inside its anonymous namespace.
//
// Work item = (composition, chunk of consecutive permutation ranks). A thread unranks its first
// permutation (Lehmer code, lexicographic order), then steps with next_permutation, scoring each
// candidate with the reference's sequential arithmetic (bit-identical to CostModel::score). The
// reference keeps the minimum of the total order (G desc, t asc, flattened ids lexicographic,
// composition lexicographic); dense indices are id ranks and next_permutation enumerates in
// lexicographic order, so that order is (G desc, t asc, permutation rank asc, composition index
// asc) -- independent of visiting order, hence reducible in parallel.

constexpr int kExMaxN = 16;

struct ExKey {
    double g, t;
    unsigned long long prank;
    unsigned int comp;
    unsigned int valid;
};

__host__ __device__ __forceinline__ bool ex_better(const ExKey& a, const ExKey& b) {
    if (!a.valid) return false;
    if (!b.valid) return true;
    if (a.g != b.g) return a.g > b.g;
    if (a.t != b.t) return a.t < b.t;
    if (a.prank != b.prank) return a.prank < b.prank;
    return a.comp < b.comp;
}

__device__ __forceinline__ void ex_unrank(unsigned long long r, int n, const unsigned long long* fact, uint8_t* perm) {
    uint32_t avail = (1u << n) - 1u;  // bit i set = dense index i unused
    for (int i = 0; i < n; ++i) {
        const unsigned long long f = fact[n - 1 - i];
        int d = (int)(r / f);
        r -= (unsigned long long)d * f;
        uint32_t m = avail;  // d-th smallest unused index
        for (int k = 0; k < d; ++k) m &= m - 1;
        const int v = __ffs(m) - 1;
        perm[i] = (uint8_t)v;
        avail &= ~(1u << v);
    }
}

__device__ __forceinline__ void ex_next(uint8_t* p, int n) {  // std::next_permutation
    int i = n - 2;
    while (i >= 0 && p[i] >= p[i + 1]) --i;
    if (i < 0) return;
    int j = n - 1;
    while (p[j] <= p[i]) --j;
    uint8_t t = p[i];
    p[i] = p[j], p[j] = t;
    for (int a = i + 1, b = n - 1; a < b; ++a, --b) t = p[a], p[a] = p[b], p[b] = t;
}

__global__ void __launch_bounds__(256) k_exhaustive(int n, const double2* __restrict__ tab, int n_comps,
                                                    const uint8_t* __restrict__ comps,
                                                    const uint8_t* __restrict__ comp_len,
                                                    unsigned long long nfact, unsigned long long chunk,
                                                    unsigned long long chunks_per_comp, ExKey* block_best) {
    __shared__ unsigned long long fact[kExMaxN + 1];
    __shared__ ExKey red[256];
    if (threadIdx.x <= kExMaxN) {
        unsigned long long f = 1;
        for (int i = 2; i <= (int)threadIdx.x; ++i) f *= (unsigned long long)i;
        fact[threadIdx.x] = f;
    }
    __syncthreads();
    ExKey best{0.0, 0.0, 0ull, 0u, 0u};
    const unsigned long long w = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (w < (unsigned long long)n_comps * chunks_per_comp) {
        const int comp = (int)(w / chunks_per_comp);
        const unsigned long long r0 = (w % chunks_per_comp) * chunk;
        const unsigned long long r1 = min(nfact, r0 + chunk);
        const uint8_t* sizes = comps + (size_t)comp * kExMaxN;
        const int nb = comp_len[comp];
        uint8_t perm[kExMaxN];
        ex_unrank(r0, n, fact, perm);
        for (unsigned long long r = r0; r < r1; ++r) {
            // CostModel::score, P:src/priority_mapper.cpp:259-279 (exhaustive's inner loop :463-480)
            int met = 0, pos = 0;
            double total = 0.0, elapsed = 0.0;
            for (int k = 0; k < nb; ++k) {
                const int part = sizes[k], bidx = part - 1;
                double makespan = 0.0;
                for (int j = 0; j < part; ++j) {
                    const double2 v = __ldg(&tab[bidx * n + perm[pos + j]]);
                    const double e2e = elapsed + v.x;
                    total += e2e;
                    met += elapsed <= v.y;
                    makespan = dmax(makespan, v.x);
                }
                elapsed += makespan;
                pos += part;
            }
            const ExKey key{total > 0.0 ? (double)met / total : 0.0, total, r, (unsigned)comp, 1u};
            if (ex_better(key, best)) best = key;
            ex_next(perm, n);
        }
    }
    red[threadIdx.x] = best;
    __syncthreads();
    for (int s = blockDim.x >> 1; s; s >>= 1) {
        if (threadIdx.x < s && ex_better(red[threadIdx.x + s], red[threadIdx.x])) red[threadIdx.x] = red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) block_best[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(1024) k_exhaustive_reduce(int blocks, const ExKey* in, ExKey* out) {
    __shared__ ExKey red[1024];
    ExKey best{0.0, 0.0, 0ull, 0u, 0u};
    for (int i = threadIdx.x; i < blocks; i += blockDim.x)
        if (ex_better(in[i], best)) best = in[i];
    red[threadIdx.x] = best;
    __syncthreads();
    for (int s = blockDim.x >> 1; s; s >>= 1) {
        if (threadIdx.x < s && ex_better(red[threadIdx.x + s], red[threadIdx.x])) red[threadIdx.x] = red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}
