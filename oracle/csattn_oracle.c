/*
 * csattn_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU checker for the CUDA path.
 *
 * A plain-C restatement of the reference algorithm for the hot path. Each
 * function names the reference file:line it follows (paths relative to
 * /root/reference/proj). The arithmetic is restated operation-for-operation
 * where the result depends on it: fp64 sequential dot products, f32 storage of
 * normalized slices, fp64 accumulation with the product w_b*score rounded
 * before the add, (score desc, index asc) orders, strict-win insertion.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
 * Pinned by tests/test_oracle.py against oracle/_ref (the reference itself)
 * and the reference tests' known answers.
 */
#include "csattn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- util.hpp ---------------- */

/* splitmix64 sub-seed, util.hpp:61-66 */
uint64_t ora_mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* ceil(ratio*n - 1e-9), util.hpp:77-81 */
uint64_t ora_ceil_ratio(double ratio, uint64_t n) {
    double c = ceil(ratio * (double)n - 1e-9);
    return c <= 0.0 ? 0 : (uint64_t)c;
}

/* retrieval.cpp:34-38 */
int ora_keep_count(double rho, uint64_t n, uint64_t* out) {
    if (!(rho > 0.0 && rho <= 1.0)) return CSATTN_ERR_PARAMETER;
    uint64_t k = ora_ceil_ratio(rho, n);
    *out = k < 1 ? 1 : k;
    return CSATTN_OK;
}

/* mt19937_64 (the standard's parameters) */
#define MT_N 312
#define MT_M 156
void ora_rng_seed(ora_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
    r->spare = 0.0;
    r->have_spare = 0;
}

uint64_t ora_rng_u64(ora_rng* r) {
    static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t um = 0xFFFFFFFF80000000ULL, lm = 0x7FFFFFFFULL;
    if (r->mti >= MT_N) {
        int i;
        for (i = 0; i < MT_N - MT_M; ++i) {
            uint64_t x = (r->mt[i] & um) | (r->mt[i + 1] & lm);
            r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ mag[x & 1];
        }
        for (; i < MT_N - 1; ++i) {
            uint64_t x = (r->mt[i] & um) | (r->mt[i + 1] & lm);
            r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag[x & 1];
        }
        uint64_t x = (r->mt[MT_N - 1] & um) | (r->mt[0] & lm);
        r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ mag[x & 1];
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* util.hpp:28-36 */
double ora_rng_unit(ora_rng* r) { return (double)(ora_rng_u64(r) >> 11) * 0x1.0p-53; }
uint64_t ora_rng_index(ora_rng* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)ora_rng_u64(r) * n) >> 64);
}
/* Box-Muller with one cached spare, util.hpp:39-52 */
double ora_rng_normal(ora_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = ora_rng_unit(r);
    double u2 = ora_rng_unit(r);
    while (u1 <= 0.0) u1 = ora_rng_unit(r);
    double rad = sqrt(-2.0 * log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(a);
    r->have_spare = 1;
    return rad * cos(a);
}

/* ---------------- core.cpp ---------------- */

/* sequential fp64 inner product, core.cpp:89-94 */
double ora_dot(const float* a, const float* b, size_t n) {
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) acc += (double)a[i] * (double)b[i];
    return acc;
}

/* core.cpp:109-116: returns 1 for a zero vector (left untouched) */
int ora_l2_normalize(float* v, size_t n) {
    double n2 = 0.0;
    for (size_t i = 0; i < n; ++i) n2 += (double)v[i] * (double)v[i];
    if (n2 == 0.0) return 1;
    double inv = 1.0 / sqrt(n2);
    for (size_t i = 0; i < n; ++i) v[i] = (float)(v[i] * inv);
    return 0;
}

/* masked dense attention, core.cpp:118-169 (fp64 logits/exp/accumulate) */
int ora_attention(const float* q, const float* keys, const float* values, size_t n, size_t d,
                  const uint32_t* mask, size_t k, float* out, float* weights) {
    if (n == 0) return CSATTN_ERR_PARAMETER;
    size_t cnt = mask ? k : n;
    if (cnt == 0) return CSATTN_ERR_PARAMETER;
    double* lg = (double*)malloc(cnt * sizeof(double));
    double* acc = (double*)calloc(d, sizeof(double));
    double inv_sqrt_d = 1.0 / sqrt((double)d);
    double mx = -INFINITY;
    for (size_t r = 0; r < cnt; ++r) {
        size_t i = mask ? mask[r] : r;
        if (i >= n) {
            free(lg);
            free(acc);
            return CSATTN_ERR_PARAMETER;
        }
        lg[r] = ora_dot(q, keys + i * d, d) * inv_sqrt_d;
        if (lg[r] > mx) mx = lg[r];
    }
    double den = 0.0;
    for (size_t r = 0; r < cnt; ++r) {
        lg[r] = exp(lg[r] - mx);
        den += lg[r];
    }
    for (size_t r = 0; r < cnt; ++r) {
        size_t i = mask ? mask[r] : r;
        double w = lg[r] / den;
        if (weights) weights[r] = (float)w;
        for (size_t t = 0; t < d; ++t) acc[t] += w * (double)values[i * d + t];
    }
    for (size_t t = 0; t < d; ++t) out[t] = (float)acc[t];
    free(lg);
    free(acc);
    return CSATTN_OK;
}

/* ---------------- index.cpp ---------------- */

/* strict-win insertion with back eviction, index.cpp:22-44 */
int ora_list_try_insert(ora_list* l, uint32_t index, float score) {
    if (l->cap == 0) return 0;
    if (l->len >= l->cap) {
        if (!(score > l->score[l->len - 1])) return 0;
        l->len -= 1;
    }
    /* first slot whose entry does not precede (score, index) */
    size_t lo = 0, hi = l->len;
    while (lo < hi) {
        size_t mid = (lo + hi) / 2;
        int precedes = l->score[mid] != score ? l->score[mid] > score : l->idx[mid] < index;
        if (precedes)
            lo = mid + 1;
        else
            hi = mid;
    }
    memmove(l->score + lo + 1, l->score + lo, (l->len - lo) * sizeof(float));
    memmove(l->idx + lo + 1, l->idx + lo, (l->len - lo) * sizeof(uint32_t));
    l->score[lo] = score;
    l->idx[lo] = index;
    l->len += 1;
    return 1;
}

static const float* g_sort_scores;
static int by_score_desc_idx_asc(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    float sx = g_sort_scores[x], sy = g_sort_scores[y];
    if (sx != sy) return sx > sy ? -1 : 1;
    return x < y ? -1 : (x > y);
}

/* top-L by (score desc, index asc), index.cpp:46-62 (full sort: same set and order) */
void ora_list_from_scores(const float* scores, size_t n, uint32_t cap, ora_list* out) {
    size_t keep = cap < n ? cap : n;
    uint32_t* order = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
    g_sort_scores = scores;
    qsort(order, n, sizeof(uint32_t), by_score_desc_idx_asc);
    out->cap = cap;
    out->len = (uint32_t)keep;
    for (size_t r = 0; r < keep; ++r) {
        out->idx[r] = order[r];
        out->score[r] = scores[order[r]];
    }
    free(order);
}

/* index.cpp:68-91 */
void ora_score_keys(const float* centroid, const float* keys, size_t n_keys, size_t d,
                    size_t off, size_t w, int normalize_keys, float* out) {
    for (size_t i = 0; i < n_keys; ++i) {
        const float* sl = keys + i * d + off;
        double s = ora_dot(centroid, sl, w);
        if (normalize_keys) {
            double n2 = 0.0;
            for (size_t t = 0; t < w; ++t) n2 += (double)sl[t] * (double)sl[t];
            s = n2 == 0.0 ? 0.0 : s / sqrt(n2);
        }
        out[i] = (float)s;
    }
}

/* ---------------- retrieval.cpp ---------------- */

/* retrieval.cpp:40-87 */
int ora_select_centroids(const float* q, size_t d, const uint64_t* widths, size_t m,
                         size_t c, const float* cent, size_t tau, double threshold,
                         uint32_t* ids, uint32_t* nids, double* best, uint64_t* dot_ops) {
    (void)d;
    if (tau == 0) return CSATTN_ERR_PARAMETER;
    float sl[1024];
    double* sc = (double*)malloc(c * sizeof(double));
    size_t off = 0, coff = 0;
    *dot_ops = 0;
    for (size_t b = 0; b < m; ++b) {
        size_t w = widths[b];
        memcpy(sl, q + off, w * sizeof(float));
        const float* cb = cent + coff;
        off += w;
        coff += c * w;
        if (ora_l2_normalize(sl, w)) {
            ids[b * tau] = 0;
            nids[b] = 1;
            best[b] = 1.0;
            continue;
        }
        for (size_t j = 0; j < c; ++j) sc[j] = ora_dot(sl, cb + j * w, w);
        *dot_ops += c * w;
        size_t bj = 0;
        for (size_t j = 1; j < c; ++j)
            if (sc[j] > sc[bj]) bj = j;
        best[b] = sc[bj];
        if (sc[bj] >= threshold) {
            ids[b * tau] = (uint32_t)bj;
            nids[b] = 1;
            continue;
        }
        /* backoff: top-tau by (score desc, j asc) via repeated selection */
        size_t take = tau < c ? tau : c;
        unsigned char* used = (unsigned char*)calloc(c, 1);
        for (size_t r = 0; r < take; ++r) {
            size_t pick = c;
            for (size_t j = 0; j < c; ++j) {
                if (used[j]) continue;
                if (pick == c || sc[j] > sc[pick]) pick = j;
            }
            used[pick] = 1;
            ids[b * tau + r] = (uint32_t)pick;
        }
        nids[b] = (uint32_t)take;
        free(used);
    }
    free(sc);
    return CSATTN_OK;
}

typedef struct {
    uint32_t idx;
    uint32_t order; /* position in the flattened (list, rank) sequence */
    double score;
} ora_entry;

static int by_idx_then_order(const void* a, const void* b) {
    const ora_entry* x = (const ora_entry*)a;
    const ora_entry* y = (const ora_entry*)b;
    if (x->idx != y->idx) return x->idx < y->idx ? -1 : 1;
    return x->order < y->order ? -1 : (x->order > y->order);
}

/* retrieval.cpp:111-148. The reference sorts by index with an unstable sort and
 * sums each key's entries in fp64; each entry is w_b*double(score) rounded
 * before the add. The restatement fixes the order (gathered-list order), which
 * is the order the CUDA kernel uses; sums of <= m*tau such terms are exact in
 * practice and tests/test_oracle.py pins equality. */
size_t ora_reduce_by_key(const ora_list* const* lists, const uint32_t* subspace, size_t nl,
                         const double* weights, uint32_t* cidx, double* cscore,
                         uint32_t* ccount) {
    size_t total = 0;
    for (size_t l = 0; l < nl; ++l) total += lists[l]->len;
    ora_entry* e = (ora_entry*)malloc((total ? total : 1) * sizeof(ora_entry));
    size_t p = 0;
    for (size_t l = 0; l < nl; ++l) {
        double w = weights[subspace[l]];
        for (uint32_t r = 0; r < lists[l]->len; ++r, ++p) {
            e[p].idx = lists[l]->idx[r];
            e[p].order = (uint32_t)p;
            e[p].score = w * (double)lists[l]->score[r];
        }
    }
    qsort(e, total, sizeof(ora_entry), by_idx_then_order);
    size_t nc = 0, r = 0;
    while (r < total) {
        uint32_t key = e[r].idx;
        double sum = 0.0;
        uint32_t src = 0;
        while (r < total && e[r].idx == key) {
            sum += e[r].score;
            src += 1;
            ++r;
        }
        cidx[nc] = key;
        cscore[nc] = sum;
        ccount[nc] = src;
        ++nc;
    }
    free(e);
    return nc;
}

typedef struct {
    uint32_t idx;
    double score;
} ora_scored;

static int by_rank(const void* a, const void* b) {
    const ora_scored* x = (const ora_scored*)a;
    const ora_scored* y = (const ora_scored*)b;
    if (x->score != y->score) return x->score > y->score ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int u32_asc(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}

/* retrieval.cpp:150-228 */
size_t ora_select_topk(const uint32_t* cidx, const double* cscore, size_t ncand, size_t n,
                       double rho, size_t window, int passthrough, size_t k_override,
                       uint32_t* out) {
    if (n == 0) return 0;
    size_t k;
    if (k_override)
        k = k_override < n ? k_override : n;
    else {
        uint64_t kk;
        if (ora_keep_count(rho, n, &kk)) return 0;
        k = (size_t)kk;
    }
    size_t r_eff = window < n ? window : n;
    size_t wlo = n - r_eff;
    size_t ns = 0;
    ora_scored* pool = (ora_scored*)malloc((ncand + r_eff + 1) * sizeof(ora_scored));
    size_t np = 0;
    if (passthrough) {
        if (k <= r_eff) {
            for (size_t i = n - k; i < n; ++i) out[ns++] = (uint32_t)i;
            free(pool);
            return ns;
        }
        for (size_t i = wlo; i < n; ++i) out[ns++] = (uint32_t)i;
        for (size_t c = 0; c < ncand; ++c)
            if (cidx[c] < wlo) {
                pool[np].idx = cidx[c];
                pool[np].score = cscore[c];
                ++np;
            }
        size_t need = k - r_eff;
        size_t take = need < np ? need : np;
        qsort(pool, np, sizeof(ora_scored), by_rank);
        for (size_t c = 0; c < take; ++c) out[ns++] = pool[c].idx;
    } else {
        size_t c = 0;
        for (; c < ncand && cidx[c] < wlo; ++c) {
            pool[np].idx = cidx[c];
            pool[np].score = cscore[c];
            ++np;
        }
        for (size_t i = wlo; i < n; ++i) {
            pool[np].idx = (uint32_t)i;
            if (c < ncand && cidx[c] == i) {
                pool[np].score = cscore[c];
                ++c;
            } else {
                pool[np].score = 0.0;
            }
            ++np;
        }
        size_t take = k < np ? k : np;
        qsort(pool, np, sizeof(ora_scored), by_rank);
        for (size_t p = 0; p < take; ++p) out[ns++] = pool[p].idx;
    }
    free(pool);
    if (ns < k) {
        unsigned char* taken = (unsigned char*)calloc(n, 1);
        for (size_t s = 0; s < ns; ++s) taken[out[s]] = 1;
        for (size_t i = n; i-- > 0 && ns < k;)
            if (!taken[i]) out[ns++] = (uint32_t)i;
        free(taken);
    }
    qsort(out, ns, sizeof(uint32_t), u32_asc);
    return ns;
}

/* ---------------- clustering.cpp ---------------- */

/* k-means++ seeding, clustering.cpp:13-71 */
static void ora_kmeanspp(const float* pts, size_t n, size_t dim, size_t k, ora_rng* rng,
                         float* seeds) {
    size_t dup = 0;
    size_t first = (size_t)ora_rng_index(rng, n);
    memcpy(seeds, pts + first * dim, dim * sizeof(float));
    double* best = (double*)malloc(n * sizeof(double));
    double* wt = (double*)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) best[i] = ora_dot(pts + i * dim, seeds, dim);
    best[first] = 2.0;
    for (size_t j = 1; j < k; ++j) {
        double total = 0.0;
        for (size_t i = 0; i < n; ++i) {
            double dd = 1.0 - best[i];
            if (dd < 0.0) dd = 0.0;
            wt[i] = dd * dd;
            total += wt[i];
        }
        if (total > 0.0) {
            double target = ora_rng_unit(rng) * total;
            size_t pick = n - 1;
            double run = 0.0;
            for (size_t i = 0; i < n; ++i) {
                run += wt[i];
                if (target < run) {
                    pick = i;
                    break;
                }
            }
            memcpy(seeds + j * dim, pts + pick * dim, dim * sizeof(float));
            for (size_t i = 0; i < n; ++i) {
                double c = ora_dot(pts + i * dim, seeds + j * dim, dim);
                if (c > best[i]) best[i] = c;
            }
            best[pick] = 2.0;
        } else {
            memcpy(seeds + j * dim, seeds + (dup % j) * dim, dim * sizeof(float));
            dup += 1;
        }
    }
    free(best);
    free(wt);
}

static size_t ora_argmax_centroid(const float* x, const float* cent, size_t k, size_t dim,
                                  double* bc_out) {
    double bc = -INFINITY;
    size_t bj = 0;
    for (size_t j = 0; j < k; ++j) {
        double c = ora_dot(x, cent + j * dim, dim);
        if (c > bc) {
            bc = c;
            bj = j;
        }
    }
    *bc_out = bc;
    return bj;
}

static void ora_renormalize(const double* sums, size_t k, size_t dim, float* cent,
                            const size_t* counts, int skip_empty) {
    for (size_t j = 0; j < k; ++j) {
        if (skip_empty && counts[j] == 0) continue;
        const double* s = sums + j * dim;
        double n2 = 0.0;
        for (size_t t = 0; t < dim; ++t) n2 += s[t] * s[t];
        if (n2 == 0.0) continue;
        double inv = 1.0 / sqrt(n2);
        for (size_t t = 0; t < dim; ++t) cent[j * dim + t] = (float)(s[t] * inv);
    }
}

/* clustering.cpp:73-240 */
int ora_cosine_kmeans(const float* points, size_t n_total, size_t dim, size_t k,
                      size_t iterations, size_t batch_size, uint64_t seed, double tolerance,
                      float* cent) {
    if (dim == 0 || n_total == 0 || k == 0) return CSATTN_ERR_PARAMETER;
    float* train = (float*)malloc(n_total * dim * sizeof(float));
    size_t n = 0;
    for (size_t i = 0; i < n_total; ++i) {
        float* row = train + n * dim;
        memcpy(row, points + i * dim, dim * sizeof(float));
        if (!ora_l2_normalize(row, dim)) ++n;
    }
    if (n == 0) {
        free(train);
        return CSATTN_ERR_DATA;
    }
    ora_rng rng;
    ora_rng_seed(&rng, seed);
    if (k > n) {
        for (size_t j = 0; j < k; ++j)
            memcpy(cent + j * dim, train + (j % n) * dim, dim * sizeof(float));
        free(train);
        return CSATTN_OK;
    }
    ora_kmeanspp(train, n, dim, k, &rng, cent);
    size_t batch = batch_size == 0 ? (n < 4096 ? n : 4096) : (batch_size < n ? batch_size : n);
    int status = CSATTN_OK;
    double* sums = (double*)malloc(k * dim * sizeof(double));
    size_t* counts = (size_t*)malloc(k * sizeof(size_t));
    if (batch >= n) {
        /* full-batch Lloyd, clustering.cpp:125-192 */
        size_t* assign = (size_t*)malloc(n * sizeof(size_t));
        double* best = (double*)malloc(n * sizeof(double));
        int have_prev = 0;
        double prev = 0.0;
        for (size_t it = 0; it < iterations; ++it) {
            double obj = 0.0;
            for (size_t i = 0; i < n; ++i) {
                assign[i] = ora_argmax_centroid(train + i * dim, cent, k, dim, &best[i]);
                obj += 2.0 - 2.0 * best[i];
            }
            obj /= (double)n;
            if (have_prev && obj > prev + tolerance) {
                status = CSATTN_ERR_PROPERTY;
                break;
            }
            int converged = have_prev && prev - obj < tolerance;
            prev = obj;
            have_prev = 1;
            if (converged) break;
            memset(sums, 0, k * dim * sizeof(double));
            memset(counts, 0, k * sizeof(size_t));
            for (size_t i = 0; i < n; ++i) {
                double* s = sums + assign[i] * dim;
                for (size_t t = 0; t < dim; ++t) s[t] += train[i * dim + t];
                counts[assign[i]] += 1;
            }
            for (size_t j = 0; j < k; ++j) {
                if (counts[j] != 0) continue;
                /* empty cluster: re-seed at the worst-covered row, in j order */
                size_t far = 0;
                for (size_t i = 1; i < n; ++i)
                    if (best[i] < best[far]) far = i;
                memcpy(cent + j * dim, train + far * dim, dim * sizeof(float));
                best[far] = 2.0;
            }
            ora_renormalize(sums, k, dim, cent, counts, 1);
        }
        free(assign);
        free(best);
    } else {
        /* mini-batch streaming means, clustering.cpp:193-238 */
        for (size_t t = 0; t < k * dim; ++t) sums[t] = (double)cent[t];
        for (size_t j = 0; j < k; ++j) counts[j] = 1;
        double first = 0.0, last = 0.0;
        for (size_t it = 0; it < iterations; ++it) {
            double obj = 0.0;
            for (size_t s = 0; s < batch; ++s) {
                const float* x = train + ora_rng_index(&rng, n) * dim;
                double bc;
                size_t bj = ora_argmax_centroid(x, cent, k, dim, &bc);
                obj += 2.0 - 2.0 * bc;
                for (size_t t = 0; t < dim; ++t) sums[bj * dim + t] += x[t];
                counts[bj] += 1;
            }
            last = obj / (double)batch;
            if (it == 0) first = last;
            ora_renormalize(sums, k, dim, cent, counts, 0);
        }
        if (iterations >= 2 && last > first + 1e-3) status = CSATTN_ERR_PROPERTY;
    }
    free(sums);
    free(counts);
    free(train);
    return status;
}

/* ---------------- session.cpp composition ---------------- */

typedef struct {
    int has_cache;
    size_t ncand;
    uint32_t* cidx;
    double* cscore;
    uint32_t* ccount;
    double worst;
} ora_state;

struct ora_session {
    uint64_t d, m, c, p, n, cap_rows, group, step;
    uint64_t widths[64], offs[64];
    float* keys;
    float* values;
    float* cent; /* C*d packed per subspace */
    ora_list* tables;
    uint32_t L;
    int normalize_keys;
    csattn_retrieval_config rc;
    double weights[64];
    ora_state* st;
};

static int ora_layout(ora_session* s, const uint64_t* widths, uint64_t m, uint64_t d) {
    if (m == 0 || m > 64) return CSATTN_ERR_PARAMETER;
    uint64_t off = 0;
    for (uint64_t b = 0; b < m; ++b) {
        if (widths[b] == 0) return CSATTN_ERR_PARAMETER;
        s->widths[b] = widths[b];
        s->offs[b] = off;
        off += widths[b];
    }
    if (off != d) return CSATTN_ERR_DIMENSION;
    s->m = m;
    s->d = d;
    return CSATTN_OK;
}

static int ora_common(ora_session* s, const float* k, const float* v, uint64_t p,
                      const csattn_index_config* icfg, const csattn_retrieval_config* rcfg,
                      uint64_t group) {
    s->p = p;
    s->n = p;
    s->cap_rows = p + 64;
    s->keys = (float*)malloc(s->cap_rows * s->d * sizeof(float));
    s->values = (float*)malloc(s->cap_rows * s->d * sizeof(float));
    memcpy(s->keys, k, p * s->d * sizeof(float));
    memcpy(s->values, v, p * s->d * sizeof(float));
    s->rc = *rcfg;
    for (uint64_t b = 0; b < s->m; ++b)
        s->weights[b] = (rcfg->weights && rcfg->n_weights) ? rcfg->weights[b] : 1.0;
    s->rc.weights = NULL;
    s->group = group ? group : 1;
    s->st = (ora_state*)calloc(s->group, sizeof(ora_state));
    /* list sizing, index.cpp:115-124 */
    s->L = icfg->list_capacity ? (uint32_t)icfg->list_capacity
                               : (uint32_t)ora_ceil_ratio(icfg->alpha, p);
    if (s->L == 0) return CSATTN_ERR_PARAMETER;
    s->normalize_keys = icfg->normalize_keys;
    /* assemble_index: m*C lists, subspace-major, index.cpp:127-139 */
    s->tables = (ora_list*)calloc(s->m * s->c, sizeof(ora_list));
    float* sc = (float*)malloc(p * sizeof(float));
    const float* cb = s->cent;
    for (uint64_t b = 0; b < s->m; ++b) {
        uint64_t w = s->widths[b];
        for (uint64_t j = 0; j < s->c; ++j) {
            ora_list* l = &s->tables[b * s->c + j];
            l->idx = (uint32_t*)malloc((s->L + 1) * sizeof(uint32_t));
            l->score = (float*)malloc((s->L + 1) * sizeof(float));
            ora_score_keys(cb + j * w, s->keys, p, s->d, s->offs[b], w, s->normalize_keys, sc);
            ora_list_from_scores(sc, p, s->L, l);
        }
        cb += s->c * w;
    }
    free(sc);
    return CSATTN_OK;
}

int ora_prefill(const float* q, uint64_t nq, const float* k, const float* v, uint64_t p,
                uint64_t d, const uint64_t* widths, uint64_t m, const csattn_index_config* icfg,
                const csattn_retrieval_config* rcfg, uint64_t group, ora_session** out) {
    ora_session* s = (ora_session*)calloc(1, sizeof(ora_session));
    int st = ora_layout(s, widths, m, d);
    if (st) {
        free(s);
        return st;
    }
    s->c = icfg->centroids;
    s->cent = (float*)malloc(s->c * d * sizeof(float));
    /* build_index: per-subspace k-means with seed mix_seed(seed, b), index.cpp:157-175 */
    float* sub = (float*)malloc(nq * 64 * sizeof(float));
    float* cb = s->cent;
    for (uint64_t b = 0; b < m; ++b) {
        uint64_t w = widths[b];
        for (uint64_t i = 0; i < nq; ++i)
            memcpy(sub + i * w, q + i * d + s->offs[b], w * sizeof(float));
        st = ora_cosine_kmeans(sub, nq, w, s->c, icfg->iterations, icfg->batch_size,
                               ora_mix_seed(icfg->seed, b), icfg->tolerance, cb);
        if (st) {
            free(sub);
            free(s->cent);
            free(s);
            return st;
        }
        cb += s->c * w;
    }
    free(sub);
    st = ora_common(s, k, v, p, icfg, rcfg, group);
    if (st) {
        ora_free(s);
        return st;
    }
    *out = s;
    return CSATTN_OK;
}

int ora_prefill_from_centroids(const float* cent, uint64_t c, const float* k, const float* v,
                               uint64_t p, uint64_t d, const uint64_t* widths, uint64_t m,
                               const csattn_index_config* icfg,
                               const csattn_retrieval_config* rcfg, uint64_t group,
                               ora_session** out) {
    ora_session* s = (ora_session*)calloc(1, sizeof(ora_session));
    int st = ora_layout(s, widths, m, d);
    if (st) {
        free(s);
        return st;
    }
    s->c = c;
    s->cent = (float*)malloc(c * d * sizeof(float));
    memcpy(s->cent, cent, c * d * sizeof(float));
    st = ora_common(s, k, v, p, icfg, rcfg, group);
    if (st) {
        ora_free(s);
        return st;
    }
    *out = s;
    return CSATTN_OK;
}

void ora_free(ora_session* s) {
    if (!s) return;
    if (s->tables)
        for (uint64_t t = 0; t < s->m * s->c; ++t) {
            free(s->tables[t].idx);
            free(s->tables[t].score);
        }
    free(s->tables);
    if (s->st)
        for (uint64_t h = 0; h < s->group; ++h) {
            free(s->st[h].cidx);
            free(s->st[h].cscore);
            free(s->st[h].ccount);
        }
    free(s->st);
    free(s->keys);
    free(s->values);
    free(s->cent);
    free(s);
}

uint64_t ora_context(const ora_session* s) { return s->n; }

/* streaming_insert, retrieval.cpp:272-301 */
static uint64_t ora_insert(ora_session* s, const float* key, uint32_t key_index) {
    uint64_t applied = 0;
    float sl[1024];
    const float* cb = s->cent;
    for (uint64_t b = 0; b < s->m; ++b) {
        uint64_t w = s->widths[b];
        memcpy(sl, key + s->offs[b], w * sizeof(float));
        int zero = 0;
        if (s->normalize_keys) zero = ora_l2_normalize(sl, w);
        for (uint64_t j = 0; j < s->c; ++j) {
            double sc = zero ? 0.0 : ora_dot(cb + j * w, sl, w);
            applied += (uint64_t)ora_list_try_insert(&s->tables[b * s->c + j], key_index,
                                                     (float)sc);
        }
        cb += s->c * w;
    }
    return applied;
}

/* decode_step for each query head of the group, then one append + insert
 * (session.cpp:46-99; GQA composition as in oracle/ref_adapter.cpp). */
int ora_step(ora_session* s, const float* q, const float* key, const float* value,
             uint32_t* selected, uint64_t sel_stride, float* out, float* weights,
             csattn_step_report* reps) {
    const uint64_t d = s->d, m = s->m, c = s->c, n = s->n;
    const uint64_t tau = s->rc.backoff_tau;
    if (tau == 0) return CSATTN_ERR_PARAMETER;
    uint32_t* ids = (uint32_t*)malloc(m * tau * sizeof(uint32_t));
    uint32_t nids[64];
    double best[64];
    uint64_t kk;
    if (ora_keep_count(s->rc.keep_ratio, n, &kk)) return CSATTN_ERR_PARAMETER;
    uint32_t* sel = (uint32_t*)malloc((kk + 1) * sizeof(uint32_t));
    for (uint64_t h = 0; h < s->group; ++h) {
        ora_state* st = &s->st[h];
        const float* qh = q + h * d;
        csattn_step_report rep;
        memset(&rep, 0, sizeof(rep));
        int searched = !st->has_cache || (s->step % s->rc.search_period) == 0;
        if (searched) {
            uint64_t dot_ops;
            ora_select_centroids(qh, d, s->widths, m, c, s->cent, tau,
                                 s->rc.backoff_threshold, ids, nids, best, &dot_ops);
            const ora_list* lists[64 * 64];
            uint32_t subs[64 * 64];
            size_t nl = 0, total = 0;
            for (uint64_t b = 0; b < m; ++b)
                for (uint32_t r = 0; r < nids[b]; ++r) {
                    lists[nl] = &s->tables[b * c + ids[b * tau + r]];
                    subs[nl] = (uint32_t)b;
                    total += lists[nl]->len;
                    ++nl;
                }
            free(st->cidx);
            free(st->cscore);
            free(st->ccount);
            st->cidx = (uint32_t*)malloc((total + 1) * sizeof(uint32_t));
            st->cscore = (double*)malloc((total + 1) * sizeof(double));
            st->ccount = (uint32_t*)malloc((total + 1) * sizeof(uint32_t));
            st->ncand = ora_reduce_by_key(lists, subs, nl, s->weights, st->cidx, st->cscore,
                                          st->ccount);
            st->has_cache = 1;
            st->worst = 1.0;
            for (uint64_t b = 0; b < m; ++b)
                if (best[b] < st->worst) st->worst = best[b];
            rep.centroid_dot_ops = dot_ops;
            rep.gathered_entries = total;
            rep.reduce_ops = total;
            rep.searches = 1;
        }
        size_t k = ora_select_topk(st->cidx, st->cscore, st->ncand, n, s->rc.keep_ratio,
                                   s->rc.recent_window, s->rc.recent_passthrough, 0, sel);
        rep.k = k;
        rep.searched = searched;
        rep.attention_key_ops = k * d;
        rep.h2d_bytes_model = 2.0 * s->rc.keep_ratio * (double)n * (double)d * 2.0 /
                              (double)s->rc.search_period;
        rep.worst_best_cosine = st->worst;
        float o[1024];
        ora_attention(qh, s->keys, s->values, n, d, sel, k, o,
                      weights ? weights + h * sel_stride : NULL);
        if (out) memcpy(out + h * d, o, d * sizeof(float));
        if (selected) memcpy(selected + h * sel_stride, sel, k * sizeof(uint32_t));
        if (reps) reps[h] = rep;
    }
    free(ids);
    free(sel);
    /* append (core.cpp:71-79), then insert with key_index = pre-append n */
    if (s->n == s->cap_rows) {
        s->cap_rows *= 2;
        s->keys = (float*)realloc(s->keys, s->cap_rows * d * sizeof(float));
        s->values = (float*)realloc(s->values, s->cap_rows * d * sizeof(float));
    }
    memcpy(s->keys + s->n * d, key, d * sizeof(float));
    memcpy(s->values + s->n * d, value, d * sizeof(float));
    s->n += 1;
    uint64_t applied = ora_insert(s, key, (uint32_t)n);
    s->step += 1;
    if (reps)
        for (uint64_t h = 0; h < s->group; ++h) {
            reps[h].inserts_attempted = m * c;
            reps[h].inserts_applied = applied;
            reps[h].insert_dot_ops = c * d;
        }
    return CSATTN_OK;
}

int ora_export(const ora_session* s, uint32_t* lens, uint32_t* idx, float* scores,
               uint64_t stride, float* centroids) {
    for (uint64_t t = 0; t < s->m * s->c; ++t) {
        const ora_list* l = &s->tables[t];
        if (l->len > stride) return CSATTN_ERR_PARAMETER;
        lens[t] = l->len;
        memcpy(idx + t * stride, l->idx, l->len * sizeof(uint32_t));
        memcpy(scores + t * stride, l->score, l->len * sizeof(float));
    }
    if (centroids) memcpy(centroids, s->cent, s->c * s->d * sizeof(float));
    return CSATTN_OK;
}
