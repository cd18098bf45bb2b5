/* Plain-C restatement of the reference SA scheduler hot path -- TEST
 * INFRASTRUCTURE (see slo_oracle.h). Single-threaded, allocation per call,
 * written for clarity over speed. P: = /root/reference/proj/. */
#define _DEFAULT_SOURCE
#include "slo_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng */
/* P:include/slosched/rng.hpp:264-271 (rotl, splitmix64 finaliser) */
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:16-22 */
void or_rng_seed(or_rng* r, uint64_t seed) {
    uint64_t z = seed;
    for (int i = 0; i < 4; ++i) {
        z += 0x9e3779b97f4a7c15ULL;
        r->s[i] = mix64(z);
    }
}

/* rng.hpp:24-34 */
uint64_t or_rng_next(or_rng* r) {
    uint64_t* s = r->s;
    const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

/* rng.hpp:37-39 */
double or_rng_uniform(or_rng* r) { return (double)(or_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:46-57: Lemire multiply-shift with rejection below (2^64 mod n) */
uint64_t or_rng_index(or_rng* r, uint64_t n) {
    unsigned __int128 m = (unsigned __int128)or_rng_next(r) * n;
    uint64_t lo = (uint64_t)m;
    if (lo < n) {
        const uint64_t thr = (0 - n) % n;
        while (lo < thr) {
            m = (unsigned __int128)or_rng_next(r) * n;
            lo = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

/* rng.hpp:66-73 */
double or_rng_normal(or_rng* r) {
    double u1;
    do {
        u1 = or_rng_uniform(r);
    } while (u1 <= 0.0);
    const double u2 = or_rng_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* rng.hpp:85-87 */
uint64_t or_rng_derive(uint64_t seed, uint64_t stream) {
    return mix64(seed + 0x9e3779b97f4a7c15ULL * (stream + 1));
}

/* ------------------------------------------------------ latency model */
/* P:src/latency_model.cpp:86-89 */
double or_predict_prefill(const double* c, int b, int li) {
    const double bd = b, ld = li;
    return c[0] * bd * ld + c[1] * bd + c[2] * ld + c[3];
}

/* latency_model.cpp:96-103 (closed-form arithmetic series) */
double or_predict_decode_total(const double* c, int b, int li, int lo) {
    const double bd = b, l_i = li, l_o = lo;
    const double slope = c[4] * bd + c[6];
    const double len_sum = l_o * l_i + l_o * (l_o + 1.0) / 2.0;
    return slope * len_sum + l_o * (c[5] * bd + c[7]);
}

/* latency_model.cpp:105-107 */
double or_predict_exec(const double* c, int b, int li, int lo) {
    return or_predict_prefill(c, b, li) + or_predict_decode_total(c, b, li, lo);
}

/* latency_model.cpp:109-113 (caller guarantees lo >= 1) */
double or_predict_tpot(const double* c, int b, int li, int lo) {
    return or_predict_decode_total(c, b, li, lo) / (double)lo;
}

/* ---------------------------------------------------------- workload */
static int clamp_len(double v) { /* P:src/workload.cpp:41-43 */
    long long x = llround(v);
    int i = (int)x;
    return i < 1 ? 1 : (i > 2047 ? 2047 : i);
}

static int clamp_round(double v) { /* P:src/output_estimator.cpp:361-363 */
    int i = (int)llround(v);
    return i < 1 ? 1 : i;
}

/* P:src/workload.cpp:158-183 with LengthDists defaults (workload.hpp:23-32) */
void or_generate_mixed(int n, uint64_t seed, int predict_mode, int* id, int* cls, int* in_len,
                       int* true_out, int* pred_out, double* arrival) {
    or_rng r;
    or_rng_seed(&r, seed);
    const int n_code = (n + 1) / 2;
    for (int i = 0; i < n; ++i) {
        const int code = i < n_code;
        cls[i] = code ? 0 : 1;
        const double in_median = code ? 300.0 : 200.0, in_sigma = 0.5;
        const double out_mean = code ? 900.0 : 250.0, out_std = code ? 300.0 : 150.0;
        in_len[i] = clamp_len(in_median * exp(in_sigma * or_rng_normal(&r)));
        true_out[i] = clamp_len(out_mean + out_std * or_rng_normal(&r));
        arrival[i] = 0.0;
    }
    /* Rng::shuffle (rng.hpp:78-82) over whole Request records */
    for (int i = n; i > 1; --i) {
        const int j = (int)or_rng_index(&r, (uint64_t)i);
        int t;
        t = cls[i - 1], cls[i - 1] = cls[j], cls[j] = t;
        t = in_len[i - 1], in_len[i - 1] = in_len[j], in_len[j] = t;
        t = true_out[i - 1], true_out[i - 1] = true_out[j], true_out[j] = t;
    }
    for (int i = 0; i < n; ++i) id[i] = i;
    if (predict_mode == 1) {
        /* estimator cold start: Gaussian prior per class, output_estimator.cpp:367-375 */
        or_rng pr;
        or_rng_seed(&pr, or_rng_derive(seed, 0x9e37));
        for (int i = 0; i < n; ++i) {
            const double mean = cls[i] == 0 ? 900.0 : 250.0, sd = cls[i] == 0 ? 300.0 : 150.0;
            pred_out[i] = clamp_round(mean + sd * or_rng_normal(&pr));
        }
    } else {
        for (int i = 0; i < n; ++i) pred_out[i] = true_out[i];
    }
}

/* ------------------------------------------------------------ lookup */
typedef struct {
    int id, row;
} id_row;

static int cmp_id_row(const void* a, const void* b) {
    const int x = ((const id_row*)a)->id, y = ((const id_row*)b)->id;
    return (x > y) - (x < y);
}

typedef struct {
    id_row* rows;
    int n;
} id_index;

static id_index index_build(const int* ids, int n) {
    id_index ix;
    ix.n = n;
    ix.rows = (id_row*)malloc(sizeof(id_row) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) ix.rows[i].id = ids[i], ix.rows[i].row = i;
    qsort(ix.rows, (size_t)n, sizeof(id_row), cmp_id_row);
    return ix;
}

static int index_find(const id_index* ix, int id) {
    int lo = 0, hi = ix->n - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) / 2;
        if (ix->rows[mid].id == id) return ix->rows[mid].row;
        if (ix->rows[mid].id < id) lo = mid + 1;
        else hi = mid - 1;
    }
    return -1;
}

static int class_row(const or_workload* w, int class_id) {
    for (int c = 0; c < w->n_classes; ++c)
        if (w->class_id[c] == class_id) return c;
    return -1;
}

/* std::max(a, b) as the reference uses it */
static double dmax(double a, double b) { return a < b ? b : a; }

/* ---------------------------------------------------------- evaluate */
/* P:src/objective.cpp:7-82 */
int or_evaluate(const or_workload* w, const double* c, const int* ids, const int* sizes, int nb,
                int* n_met, double* t, double* g, double* wait, double* exec, double* e2e,
                double* ttft, double* tpot, int* met) {
    id_index ix = index_build(w->id, w->n);
    int total_n = 0;
    for (int k = 0; k < nb; ++k) total_n += sizes[k];
    double* ex = (double*)malloc(sizeof(double) * (size_t)(total_n + 1));
    double* pf = (double*)malloc(sizeof(double) * (size_t)(total_n + 1));
    double* tp = (double*)malloc(sizeof(double) * (size_t)(total_n + 1));
    int* rows = (int*)malloc(sizeof(int) * (size_t)(total_n + 1));
    int rc = 0, pos = 0;
    for (int k = 0; k < nb && rc == 0; ++k) { /* batch_exec_profile, objective.cpp:7-30 */
        for (int j = 0; j < sizes[k]; ++j, ++pos) {
            const int row = index_find(&ix, ids[pos]);
            if (row < 0 || w->pred_out[row] < 0) {
                rc = -1;
                break;
            }
            const int li = w->in_len[row], lo = w->pred_out[row];
            ex[pos] = or_predict_exec(c, sizes[k], li, lo);
            pf[pos] = or_predict_prefill(c, sizes[k], li);
            tp[pos] = or_predict_tpot(c, sizes[k], li, lo);
            rows[pos] = row;
        }
    }
    if (rc == 0) {
        int n = 0;
        double tot = 0.0, elapsed = 0.0;
        pos = 0;
        for (int k = 0; k < nb; ++k) { /* waiting_times, objective.cpp:32-47 */
            double makespan = 0.0;
            const int start = pos;
            for (int j = 0; j < sizes[k]; ++j, ++pos) makespan = dmax(makespan, ex[pos]);
            for (int q = start; q < pos; ++q) {
                const double e2e_v = ex[q] + elapsed, ttft_v = pf[q] + elapsed;
                const int cr = class_row(w, w->cls[rows[q]]);
                int ok; /* meets_slo, objective.cpp:49-53 */
                if (w->kind[cr] == 0) ok = e2e_v <= w->e2e[cr];
                else ok = ttft_v <= w->ttft[cr] && tp[q] <= w->tpot[cr];
                n += ok;
                tot += e2e_v;
                if (wait) wait[q] = elapsed;
                if (exec) exec[q] = ex[q];
                if (e2e) e2e[q] = e2e_v;
                if (ttft) ttft[q] = ttft_v;
                if (tpot) tpot[q] = tp[q];
                if (met) met[q] = ok;
            }
            elapsed += makespan;
        }
        *n_met = n;
        *t = tot;
        *g = tot > 0.0 ? (double)n / tot : 0.0;
    }
    free(ex), free(pf), free(tp), free(rows), free(ix.rows);
    return rc;
}

/* --------------------------------------------------------- CostModel */
/* P:src/priority_mapper.cpp:203-288 */
typedef struct {
    int n, mb;
    int* ids; /* sorted */
    double *exec, *prefill, *tpot;
    char* e2e_kind;
    double *e2e_slo, *ttft_slo, *tpot_slo;
} cost_model;

static int cmp_int(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

static int cm_build(cost_model* m, const or_workload* w, const double* c, const int* ids, int n, int mb) {
    memset(m, 0, sizeof *m);
    m->n = n, m->mb = mb;
    const size_t nn = (size_t)(n > 0 ? n : 1), nm = nn * (size_t)mb;
    m->ids = (int*)malloc(sizeof(int) * nn);
    memcpy(m->ids, ids, sizeof(int) * (size_t)n);
    qsort(m->ids, (size_t)n, sizeof(int), cmp_int);
    m->exec = (double*)malloc(sizeof(double) * nm);
    m->prefill = (double*)malloc(sizeof(double) * nm);
    m->tpot = (double*)malloc(sizeof(double) * nm);
    m->e2e_kind = (char*)malloc(nn);
    m->e2e_slo = (double*)malloc(sizeof(double) * nn);
    m->ttft_slo = (double*)malloc(sizeof(double) * nn);
    m->tpot_slo = (double*)malloc(sizeof(double) * nn);
    id_index ix = index_build(w->id, w->n);
    int rc = 0;
    for (int i = 0; i < n; ++i) {
        const int row = index_find(&ix, m->ids[i]);
        if (row < 0 || w->pred_out[row] < 0) {
            rc = -1;
            break;
        }
        const int cr = class_row(w, w->cls[row]);
        const int e2e_kind = w->kind[cr] == 0;
        m->e2e_kind[i] = (char)e2e_kind;
        m->e2e_slo[i] = e2e_kind ? w->e2e[cr] : 0.0;
        m->ttft_slo[i] = e2e_kind ? 0.0 : w->ttft[cr];
        m->tpot_slo[i] = e2e_kind ? 0.0 : w->tpot[cr];
        for (int b = 1; b <= mb; ++b) {
            const int li = w->in_len[row], lo = w->pred_out[row];
            m->exec[(size_t)i * mb + b - 1] = or_predict_exec(c, b, li, lo);
            m->prefill[(size_t)i * mb + b - 1] = or_predict_prefill(c, b, li);
            m->tpot[(size_t)i * mb + b - 1] = or_predict_tpot(c, b, li, lo);
        }
    }
    free(ix.rows);
    return rc;
}

static void cm_free(cost_model* m) {
    free(m->ids), free(m->exec), free(m->prefill), free(m->tpot), free(m->e2e_kind);
    free(m->e2e_slo), free(m->ttft_slo), free(m->tpot_slo);
}

static int cm_dense(const cost_model* m, int id) {
    int lo = 0, hi = m->n - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) / 2;
        if (m->ids[mid] == id) return mid;
        if (m->ids[mid] < id) lo = mid + 1;
        else hi = mid - 1;
    }
    return -1;
}

/* CostModel::met, priority_mapper.cpp:237-241 */
static int cm_met(const cost_model* m, int idx, int bidx, double elapsed, double e2e) {
    if (m->e2e_kind[idx]) return e2e <= m->e2e_slo[idx];
    return elapsed + m->prefill[(size_t)idx * m->mb + bidx] <= m->ttft_slo[idx] &&
           m->tpot[(size_t)idx * m->mb + bidx] <= m->tpot_slo[idx];
}

/* CostModel::score, priority_mapper.cpp:259-279 */
static double cm_score(const cost_model* m, const int* perm, const int* sizes, int nb, int* n_met_out,
                       double* t_out) {
    int n_met = 0;
    double total = 0.0, elapsed = 0.0;
    int pos = 0;
    for (int k = 0; k < nb; ++k) {
        const int part = sizes[k], bidx = part - 1;
        double makespan = 0.0;
        for (int j = 0; j < part; ++j) {
            const int idx = perm[pos + j];
            const double e = m->exec[(size_t)idx * m->mb + bidx];
            const double e2e = elapsed + e;
            total += e2e;
            if (cm_met(m, idx, bidx, elapsed, e2e)) ++n_met;
            makespan = dmax(makespan, e);
        }
        elapsed += makespan;
        pos += part;
    }
    if (n_met_out) *n_met_out = n_met;
    if (t_out) *t_out = total;
    return total > 0.0 ? (double)n_met / total : 0.0;
}

int or_score_batch(const or_workload* w, const double* c, const int* ids, int n, int max_batch,
                   int count, const int* perms, const int* sizes, const int* nb, int* n_met,
                   double* t, double* g) {
    cost_model m;
    int rc = cm_build(&m, w, c, ids, n, max_batch);
    if (rc == 0)
        for (int q = 0; q < count; ++q)
            g[q] = cm_score(&m, perms + (size_t)q * n, sizes + (size_t)q * n, nb[q], n_met + q, t + q);
    cm_free(&m);
    return rc;
}

/* ------------------------------------------------------ FlatSchedule */
/* P:src/priority_mapper.cpp:104-199 */
typedef struct {
    int n, nb;
    int *perm, *sizes;
} flat_sched;

static int fs_batch_of(const flat_sched* f, int pos) { /* :128-133 */
    int k = 0;
    for (int acc = f->sizes[0]; pos >= acc; acc += f->sizes[++k]) {
    }
    return k;
}

static int fs_batch_start(const flat_sched* f, int k) { /* :135-139 */
    int acc = 0;
    for (int i = 0; i < k; ++i) acc += f->sizes[i];
    return acc;
}

static void fs_erase(flat_sched* f, int k) {
    memmove(f->sizes + k, f->sizes + k + 1, sizeof(int) * (size_t)(f->nb - k - 1));
    f->nb--;
}

static int fs_squeeze(flat_sched* f, or_rng* r, int mb) { /* :141-153 */
    if (f->nb < 2) return 0;
    const int first = f->sizes[0];
    const int pos = first + (int)or_rng_index(r, (uint64_t)(f->n - first));
    const int k = fs_batch_of(f, pos);
    if (f->sizes[k - 1] >= mb) return 0;
    const int dst = fs_batch_start(f, k);
    const int v = f->perm[pos]; /* rotate [dst, pos] right by one */
    memmove(f->perm + dst + 1, f->perm + dst, sizeof(int) * (size_t)(pos - dst));
    f->perm[dst] = v;
    f->sizes[k - 1]++;
    if (--f->sizes[k] == 0) fs_erase(f, k);
    return 1;
}

static int fs_delay(flat_sched* f, or_rng* r, int mb) { /* :155-170 */
    if (f->n == 0) return 0;
    const int pos = (int)or_rng_index(r, (uint64_t)f->n);
    const int k = fs_batch_of(f, pos);
    const int has_next = k + 1 < f->nb;
    if (has_next && f->sizes[k + 1] >= mb) return 0;
    const int dst = has_next ? fs_batch_start(f, k + 2) : f->n;
    const int v = f->perm[pos]; /* rotate [pos, dst) left by one */
    memmove(f->perm + pos, f->perm + pos + 1, sizeof(int) * (size_t)(dst - pos - 1));
    f->perm[dst - 1] = v;
    if (has_next) f->sizes[k + 1]++;
    else f->sizes[f->nb++] = 1;
    if (--f->sizes[k] == 0) fs_erase(f, k);
    return 1;
}

static int fs_swap(flat_sched* f, or_rng* r) { /* :172-180 */
    if (f->n < 2) return 0;
    const uint64_t a = or_rng_index(r, (uint64_t)f->n);
    uint64_t b = or_rng_index(r, (uint64_t)(f->n - 1));
    if (b >= a) ++b;
    const int t = f->perm[a];
    f->perm[a] = f->perm[b];
    f->perm[b] = t;
    return 1;
}

static int fs_propose(flat_sched* f, or_rng* r, int mb) { /* :184-198 */
    if (f->n == 0) return 0;
    for (int attempt = 0; attempt < 8; ++attempt) {
        const uint64_t op = or_rng_index(r, 3);
        if (op == 0) {
            if (fs_squeeze(f, r, mb)) return 1;
        } else if (op == 1) {
            if (fs_delay(f, r, mb)) return 1;
        } else {
            if (fs_swap(f, r)) return 1;
        }
    }
    return fs_swap(f, r);
}

static void fs_copy(flat_sched* dst, const flat_sched* src) {
    dst->n = src->n, dst->nb = src->nb;
    memcpy(dst->perm, src->perm, sizeof(int) * (size_t)src->n);
    memcpy(dst->sizes, src->sizes, sizeof(int) * (size_t)src->nb);
}

/* ---------------------------------------------------- candidates */
typedef struct {
    double key;
    int id;
} key_id;

static int cmp_key_id(const void* a, const void* b) {
    const key_id *x = (const key_id*)a, *y = (const key_id*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

static void pack_greedy(const int* ordered, int n, int mb, int* out_ids, int* out_sizes, int* out_nb) {
    /* P:src/priority_mapper.cpp:22-29 */
    *out_nb = 0;
    for (int i = 0; i < n; i += mb) {
        const int end = i + mb < n ? i + mb : n;
        out_sizes[(*out_nb)++] = end - i;
    }
    memcpy(out_ids, ordered, sizeof(int) * (size_t)n);
}

int or_initial_candidates(const or_workload* w, const double* c, const int* ids, int n, int max_batch,
                          int* sorted_ids, int* sorted_sizes, int* sorted_nb, int* input_ids,
                          int* input_sizes, int* input_nb) {
    id_index ix = index_build(w->id, w->n);
    key_id* by_e2e = (key_id*)malloc(sizeof(key_id) * (size_t)(n > 0 ? n : 1));
    key_id* by_arr = (key_id*)malloc(sizeof(key_id) * (size_t)(n > 0 ? n : 1));
    int* tmp = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    int rc = 0;
    for (int i = 0; i < n; ++i) {
        const int row = index_find(&ix, ids[i]);
        if (row < 0 || w->pred_out[row] < 0) { /* standalone_e2e, :92-99 */
            rc = -1;
            break;
        }
        by_e2e[i].key = or_predict_exec(c, max_batch, w->in_len[row], w->pred_out[row]);
        by_e2e[i].id = ids[i];
        by_arr[i].key = w->arrival[row];
        by_arr[i].id = ids[i];
    }
    if (rc == 0) {
        qsort(by_e2e, (size_t)n, sizeof(key_id), cmp_key_id);
        qsort(by_arr, (size_t)n, sizeof(key_id), cmp_key_id);
        for (int i = 0; i < n; ++i) tmp[i] = by_e2e[i].id;
        pack_greedy(tmp, n, max_batch, sorted_ids, sorted_sizes, sorted_nb);
        for (int i = 0; i < n; ++i) tmp[i] = by_arr[i].id;
        pack_greedy(tmp, n, max_batch, input_ids, input_sizes, input_nb);
    }
    free(by_e2e), free(by_arr), free(tmp), free(ix.rows);
    return rc;
}

/* ------------------------------------------------------------ anneal */
/* P:src/priority_mapper.cpp:340-411 */
int or_anneal(const or_workload* w, const double* c, const int* ids, int n, const double* cfg,
              uint64_t seed, int max_batch, int* out_ids, int* out_sizes, int* out_nb, int* n_met,
              double* t_out, double* g_out, double* stats6) {
    const double t0 = cfg[0], t_thres = cfg[1], tau = cfg[3];
    const int iter = (int)cfg[2], has_scale = cfg[4] != 0.0;
    /* AnnealConfig::validate, :9-18 */
    if (!(t0 > t_thres) || !(t_thres > 0.0) || iter < 1 || !(tau > 0.0) || !(tau < 1.0) ||
        (has_scale && !(cfg[5] >= 0.0)))
        return -2;
    for (int i = 0; i < 6; ++i) stats6[i] = 0.0;
    stats6[5] = 1.0;

    const size_t nn = (size_t)(n > 0 ? n : 1);
    int *s_ids = malloc(sizeof(int) * nn), *s_sz = malloc(sizeof(int) * nn);
    int *i_ids = malloc(sizeof(int) * nn), *i_sz = malloc(sizeof(int) * nn);
    int s_nb = 0, i_nb = 0;
    int rc = or_initial_candidates(w, c, ids, n, max_batch, s_ids, s_sz, &s_nb, i_ids, i_sz, &i_nb);
    if (rc != 0) goto done_candidates;

    int ns, ni;
    double ts, gs, ti, gi;
    rc = or_evaluate(w, c, s_ids, s_sz, s_nb, &ns, &ts, &gs, 0, 0, 0, 0, 0, 0);
    if (rc != 0) goto done_candidates;
    stats6[3] = gs;
    if (ns == n) { /* shortcut, :350-354 */
        stats6[2] = 1.0;
        memcpy(out_ids, s_ids, sizeof(int) * (size_t)n);
        memcpy(out_sizes, s_sz, sizeof(int) * (size_t)s_nb);
        *out_nb = s_nb, *n_met = ns, *t_out = ts, *g_out = gs;
        goto done_candidates;
    }
    rc = or_evaluate(w, c, i_ids, i_sz, i_nb, &ni, &ti, &gi, 0, 0, 0, 0, 0, 0);
    if (rc != 0) goto done_candidates;
    stats6[4] = gi;

    cost_model m;
    rc = cm_build(&m, w, c, ids, n, max_batch);
    if (rc != 0) {
        cm_free(&m);
        goto done_candidates;
    }
    flat_sched cur, best, scratch;
    flat_sched* all[3] = {&cur, &best, &scratch};
    for (int q = 0; q < 3; ++q) {
        all[q]->perm = malloc(sizeof(int) * nn);
        all[q]->sizes = malloc(sizeof(int) * (nn + 1));
    }
    { /* FlatSchedule::from(to_index_space(better start)), :360-361 */
        const int use_sorted = gs >= gi;
        const int* src_ids = use_sorted ? s_ids : i_ids;
        const int* src_sz = use_sorted ? s_sz : i_sz;
        cur.n = n;
        cur.nb = use_sorted ? s_nb : i_nb;
        for (int i = 0; i < n; ++i) cur.perm[i] = cm_dense(&m, src_ids[i]);
        memcpy(cur.sizes, src_sz, sizeof(int) * (size_t)cur.nb);
    }
    double f = cm_score(&m, cur.perm, cur.sizes, cur.nb, 0, 0);
    const double scale = has_scale ? cfg[5] : (f > 0.0 ? t0 / f : t0); /* :368-370 */
    stats6[5] = scale;
    fs_copy(&best, &cur);
    double best_f = f;
    or_rng r;
    or_rng_seed(&r, seed);
    uint64_t proposals = 0, accepted = 0;
    for (double t = t0; t >= t_thres; t *= tau) { /* :378-402 */
        for (int k = 0; k < iter; ++k) {
            fs_copy(&scratch, &cur);
            fs_propose(&scratch, &r, max_batch);
            const double f_new = cm_score(&m, scratch.perm, scratch.sizes, scratch.nb, 0, 0);
            proposals++;
            int accept = f_new > f;
            if (!accept) {
                const double x = (f - f_new) * scale / t;
                const double u = or_rng_uniform(&r);
                accept = x < 38.0 ? u < exp(-x) : u == 0.0;
            }
            if (accept) {
                accepted++;
                flat_sched tmp = cur;
                cur = scratch;
                scratch = tmp;
                f = f_new;
                if (f > best_f) {
                    fs_copy(&best, &cur);
                    best_f = f;
                }
            }
        }
    }
    stats6[0] = (double)proposals;
    stats6[1] = (double)accepted;
    { /* final evaluate + floor against both starts, :404-410 */
        int* b_ids = malloc(sizeof(int) * nn);
        for (int i = 0; i < n; ++i) b_ids[i] = m.ids[best.perm[i]];
        int nb_;
        double tb, gb;
        rc = or_evaluate(w, c, b_ids, best.sizes, best.nb, &nb_, &tb, &gb, 0, 0, 0, 0, 0, 0);
        const double floor_g = gs > gi ? gs : gi;
        if (rc == 0 && gb >= floor_g) {
            memcpy(out_ids, b_ids, sizeof(int) * (size_t)n);
            memcpy(out_sizes, best.sizes, sizeof(int) * (size_t)best.nb);
            *out_nb = best.nb, *n_met = nb_, *t_out = tb, *g_out = gb;
        } else if (rc == 0 && gs >= gi) {
            memcpy(out_ids, s_ids, sizeof(int) * (size_t)n);
            memcpy(out_sizes, s_sz, sizeof(int) * (size_t)s_nb);
            *out_nb = s_nb, *n_met = ns, *t_out = ts, *g_out = gs;
        } else if (rc == 0) {
            memcpy(out_ids, i_ids, sizeof(int) * (size_t)n);
            memcpy(out_sizes, i_sz, sizeof(int) * (size_t)i_nb);
            *out_nb = i_nb, *n_met = ni, *t_out = ti, *g_out = gi;
        }
        free(b_ids);
    }
    for (int q = 0; q < 3; ++q) free(all[q]->perm), free(all[q]->sizes);
    cm_free(&m);
done_candidates:
    free(s_ids), free(s_sz), free(i_ids), free(i_sz);
    return rc;
}
