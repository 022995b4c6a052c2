/*
 * csattn_oracle.h — TEST INFRASTRUCTURE ONLY. A plain-C restatement of the
 * reference CSAttention hot path (proj/src/{core,clustering,index,retrieval,
 * session}.cpp), used as the checker for the CUDA path. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Parity: pinned against the reference itself (oracle/_ref, built from the
 * unmodified sources) and against the reference tests' known answers
 * (tests/test_oracle.py, tests/golden/).
 */
#ifndef CSATTN_ORACLE_H_
#define CSATTN_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/csattn_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* util.hpp:61-81 */
uint64_t ora_mix_seed(uint64_t seed, uint64_t salt);
uint64_t ora_ceil_ratio(double ratio, uint64_t n);
int ora_keep_count(double rho, uint64_t n, uint64_t* out);

/* core.cpp:89-116 */
double ora_dot(const float* a, const float* b, size_t n);
int ora_l2_normalize(float* v, size_t n);

/* mt19937_64 + draws (util.hpp:21-58) */
typedef struct ora_rng {
    uint64_t mt[312];
    int mti;
    double spare;
    int have_spare;
} ora_rng;
void ora_rng_seed(ora_rng* r, uint64_t seed);
uint64_t ora_rng_u64(ora_rng* r);
double ora_rng_unit(ora_rng* r);
uint64_t ora_rng_index(ora_rng* r, uint64_t n);
double ora_rng_normal(ora_rng* r);

/* TopList (index.hpp:19-34) */
typedef struct ora_list {
    uint32_t cap;
    uint32_t len;
    uint32_t* idx;
    float* score;
} ora_list;
int ora_list_try_insert(ora_list* l, uint32_t index, float score);
void ora_list_from_scores(const float* scores, size_t n, uint32_t cap, ora_list* out);
void ora_score_keys(const float* centroid, const float* keys, size_t n_keys, size_t d,
                    size_t off, size_t w, int normalize_keys, float* out);

/* select_centroids (retrieval.cpp:40-87). ids: m*tau, nids: m, best: m */
int ora_select_centroids(const float* q, size_t d, const uint64_t* widths, size_t m,
                         size_t c, const float* cent, size_t tau, double threshold,
                         uint32_t* ids, uint32_t* nids, double* best, uint64_t* dot_ops);

/* reduce_by_key (retrieval.cpp:111-148) over nl lists; returns candidate count.
 * cidx/cscore/ccount must hold sum(len) entries. */
size_t ora_reduce_by_key(const ora_list* const* lists, const uint32_t* subspace, size_t nl,
                         const double* weights, uint32_t* cidx, double* cscore,
                         uint32_t* ccount);

/* select_topk (retrieval.cpp:150-228); out holds K entries; returns K or 0 on error */
size_t ora_select_topk(const uint32_t* cidx, const double* cscore, size_t ncand, size_t n,
                       double rho, size_t window, int passthrough, size_t k_override,
                       uint32_t* out);

/* masked dense_attention (core.cpp:118-169); mask NULL = all n keys */
int ora_attention(const float* q, const float* keys, const float* values, size_t n, size_t d,
                  const uint32_t* mask, size_t k, float* out, float* weights);

/* cosine_kmeans (clustering.cpp:73-240); centroids out: k*dim.
 * returns CSATTN_OK / CSATTN_ERR_PROPERTY / CSATTN_ERR_DATA / CSATTN_ERR_PARAMETER */
int ora_cosine_kmeans(const float* points, size_t n_total, size_t dim, size_t k,
                      size_t iterations, size_t batch_size, uint64_t seed, double tolerance,
                      float* centroids);

/* Session composition (session.cpp:25-99), GQA-aware (group query heads). */
typedef struct ora_session ora_session;
int ora_prefill(const float* q, uint64_t nq, const float* k, const float* v, uint64_t p,
                uint64_t d, const uint64_t* widths, uint64_t m, const csattn_index_config* icfg,
                const csattn_retrieval_config* rcfg, uint64_t group, ora_session** out);
int ora_prefill_from_centroids(const float* cent, uint64_t c, const float* k, const float* v,
                               uint64_t p, uint64_t d, const uint64_t* widths, uint64_t m,
                               const csattn_index_config* icfg,
                               const csattn_retrieval_config* rcfg, uint64_t group,
                               ora_session** out);
void ora_free(ora_session* s);
int ora_step(ora_session* s, const float* q, const float* key, const float* value,
             uint32_t* selected, uint64_t sel_stride, float* out, float* weights,
             csattn_step_report* reps);
int ora_export(const ora_session* s, uint32_t* lens, uint32_t* idx, float* scores,
               uint64_t stride, float* centroids);
uint64_t ora_context(const ora_session* s);

#ifdef __cplusplus
}
#endif
#endif
