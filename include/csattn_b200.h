/*
 * csattn_b200.h — C ABI of the B200-native CSAttention decode hot path.
 *
 * This is the drop-in boundary for the path BASELINE.json names: the offline
 * table build from prefill Q/K and the online decode step (centroid routing,
 * gather/accumulate, top-K, sparse attention, append + streaming insert).
 * Every entry point replaces one function (or one composition) of the
 * reference C++ API in proj/include/csattn/ (file:line cited per entry).
 *
 * Conventions (reference: errors.hpp:8-52):
 *   - Every function returns a csattn_status. Nothing throws across the ABI.
 *     The message of the last failure on the calling thread is returned by
 *     csattn_last_error(). One status per reference exception class.
 *   - Pointers are plain host or device pointers; CSATTN_HOST_BUFFERS in a
 *     `flags` argument says the data pointers of that call are host memory
 *     (copied in/out inside the call), otherwise they are device pointers
 *     on the context's device.
 *   - All float data is row-major fp32; indices are uint32.
 *   - Validation happens on the host before any launch, in the reference's
 *     order, so the same bad input yields the same error class + message.
 */
#ifndef CSATTN_B200_H_
#define CSATTN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception class (errors.hpp:8-52) ---- */
typedef enum csattn_status {
    CSATTN_OK = 0,
    CSATTN_ERR_GENERIC = 1,          /* csattn::Error */
    CSATTN_ERR_DIMENSION = 2,        /* csattn::DimensionError */
    CSATTN_ERR_PARAMETER = 3,        /* csattn::ParameterError */
    CSATTN_ERR_DATA = 4,             /* csattn::DataError */
    CSATTN_ERR_BAD_MAGIC = 5,        /* csattn::BadMagicError */
    CSATTN_ERR_VERSION = 6,          /* csattn::VersionError */
    CSATTN_ERR_TRUNCATED = 7,        /* csattn::TruncatedError */
    CSATTN_ERR_CORRUPT = 8,          /* csattn::CorruptError */
    CSATTN_ERR_PROPERTY = 9,         /* csattn::PropertyError */
    CSATTN_ERR_STREAM_EXHAUSTED = 10,/* csattn::StreamExhaustedError */
    CSATTN_ERR_CUDA = 20,            /* CUDA runtime / launch failure */
    CSATTN_ERR_CAPACITY = 21         /* session sized too small (max_decode_steps) */
} csattn_status;

/* flags */
#define CSATTN_HOST_BUFFERS 0x1u   /* data pointers of this call are host memory */
#define CSATTN_NO_SYNC      0x2u   /* do not synchronize the stream before returning
                                      (device buffers only) */

/* ---- configuration PODs (mirror the reference structs) ---- */

/* IndexConfig + ClusterConfig (index.hpp:36-42, clustering.hpp:17-28) */
typedef struct csattn_index_config {
    double alpha;              /* L = ceil_ratio(alpha, P); default 0.2 */
    uint64_t list_capacity;    /* absolute L override; 0 = derive */
    int32_t normalize_keys;    /* score against normalized key slices */
    int32_t score_bits;        /* 16 or 32 (serialization width) */
    uint64_t centroids;        /* C per subspace; default 64 */
    uint64_t iterations;       /* k-means rounds; default 10 */
    uint64_t batch_size;       /* 0 = min(4096, n) */
    uint64_t seed;             /* cluster seed */
    double tolerance;          /* full-batch early stop / monotonicity slack */
} csattn_index_config;

/* RetrievalConfig (retrieval.hpp:17-32). k_bump is a host callback in the
 * reference; across the ABI it is replaced by a per-call k_override. */
typedef struct csattn_retrieval_config {
    double keep_ratio;          /* rho; default 0.05 */
    uint64_t search_period;     /* default 1 */
    uint64_t recent_window;     /* R; default 32 */
    const double* weights;      /* w_b per subspace, host memory; NULL = all ones */
    uint64_t n_weights;         /* 0 or m */
    uint64_t backoff_tau;       /* default 1 */
    double backoff_threshold;   /* default -inf */
    int32_t recent_passthrough; /* default 1 */
    int32_t reserved;
} csattn_retrieval_config;

/* SyntheticSpec (synthetic.hpp:16-28) */
typedef struct csattn_synthetic_spec {
    uint64_t rows;
    uint64_t dim;
    uint64_t clusters;
    uint64_t seed;
    double plant_fraction;
    double plant_scale;
    double query_noise;
    uint64_t dwell;
} csattn_synthetic_spec;

/* DecodeStepReport.counters (metrics.hpp:15-37) + selection facts */
typedef struct csattn_step_report {
    uint64_t k;                  /* |selected| */
    int32_t searched;
    int32_t reserved;
    uint64_t centroid_dot_ops;
    uint64_t gathered_entries;
    uint64_t reduce_ops;
    uint64_t attention_key_ops;  /* k * d */
    double h2d_bytes_model;      /* h2d_bytes(rho, N, d, B, period) */
    uint64_t searches;
    uint64_t inserts_attempted;
    uint64_t inserts_applied;
    uint64_t insert_dot_ops;
    double worst_best_cosine;    /* min_b best_cosine of the last search */
} csattn_step_report;

typedef struct csattn_session_info {
    uint64_t dim;            /* d */
    uint64_t subspaces;      /* m */
    uint64_t centroids;      /* C */
    uint64_t list_capacity;  /* L */
    uint64_t prefill_len;    /* P */
    uint64_t context_len;    /* N = P + steps */
    uint64_t steps;          /* decode steps taken */
    uint64_t max_context;    /* P + max_decode_steps */
    uint64_t group;          /* query heads sharing this KV head's tables */
    double alpha;
    int32_t normalize_keys;
    int32_t score_bits;
    uint64_t device_bytes;   /* HBM owned by the session */
} csattn_session_info;

typedef struct csattn_ctx_s* csattn_ctx;
typedef struct csattn_session_s* csattn_session;

/* ---- defaults / small pure helpers ---- */
void csattn_index_config_default(csattn_index_config* cfg);
void csattn_retrieval_config_default(csattn_retrieval_config* cfg);
void csattn_synthetic_spec_default(csattn_synthetic_spec* spec);

/* keep_count (retrieval.cpp:34-38): max(1, ceil_ratio(rho, n)) */
csattn_status csattn_keep_count(double rho, uint64_t n, uint64_t* out);
/* parse_schedule (retrieval.cpp:10-32): "<rho>-step-<P>" */
csattn_status csattn_parse_schedule(const char* name, double* rho, uint64_t* period);
/* h2d_bytes (metrics.cpp:32-38) */
csattn_status csattn_h2d_bytes(double rho, uint64_t n, uint64_t d, uint64_t bytes_per_elem,
                               uint64_t period, double* out);

/* make_synthetic (synthetic.cpp:18-74): host-side input generator, bit-identical
 * to the reference (mt19937_64 + hand-rolled draws). Outputs rows*dim floats each. */
csattn_status csattn_make_synthetic(const csattn_synthetic_spec* spec, float* queries,
                                    float* keys, float* values);

const char* csattn_last_error(void);
const char* csattn_status_name(csattn_status s);

/* ---- context: device + stream ---- */
csattn_status csattn_ctx_create(int device, void* cuda_stream, csattn_ctx* out);
csattn_status csattn_ctx_destroy(csattn_ctx ctx);
csattn_status csattn_ctx_synchronize(csattn_ctx ctx);
/* KV placement of sessions created on this context from now on (the paper's
 * CPU<->GPU offload mode; the reference has only its byte
 * model, metrics.cpp:32-38). CSATTN_KV_HOST keeps every KV row (prefill and
 * appended) in mapped pinned host memory: the tables stay in HBM, and a
 * decode step moves only the selected K/V rows (and the appended row) across
 * the host link. */
#define CSATTN_KV_DEVICE 0
#define CSATTN_KV_HOST 1
csattn_status csattn_ctx_set_kv_placement(csattn_ctx ctx, int32_t placement);
/* The CUDA stream (cudaStream_t) the context enqueues on. */
void* csattn_ctx_stream(csattn_ctx ctx);
/* Number of CUDA kernels this context has launched (driver-side evidence). */
uint64_t csattn_ctx_launch_count(csattn_ctx ctx);
/* Table builds on this context that ran the tcgen05 screen (build_tc.cu),
 * and how many of those were rebuilt by the plain fp64 kernels because a
 * table's screen was inconclusive (results are identical either way). */
csattn_status csattn_ctx_build_stats(csattn_ctx ctx, uint64_t* tc_builds, uint64_t* fallbacks);
/* Kernel timing: when enabled, the three kernels of every decode step
 * (select, attend, insert) are bracketed by CUDA events on the context's
 * stream. read returns the summed milliseconds per kernel (ms[3]) and the
 * number of profiled steps since the last reset (synchronizes the stream). */
csattn_status csattn_ctx_profile(csattn_ctx ctx, int32_t enable);
csattn_status csattn_ctx_profile_read(csattn_ctx ctx, double* ms, uint64_t* steps, int32_t reset);

/* ---- offline build ----
 * prefill (session.cpp:25-44) = KvStore + build_index (index.cpp:145-177)
 * on the GPU: per-subspace exact spherical k-means (clustering.cpp:73-240),
 * exact fp64 centroid x key scores (index.cpp:68-91) and top-L lists
 * (index.cpp:46-62, 107-141).
 * queries: n_queries x d (n_queries may exceed p: a GQA group pools its heads'
 * prefill queries, index.cpp:150-151); keys/values: p x d.
 * group: query heads that will decode against this KV head (>= 1).
 * max_decode_steps: capacity for appended rows. */
csattn_status csattn_prefill(csattn_ctx ctx, const float* queries, uint64_t n_queries,
                             const float* keys, const float* values, uint64_t p, uint64_t d,
                             const uint64_t* widths, uint64_t m,
                             const csattn_index_config* icfg,
                             const csattn_retrieval_config* rcfg, uint64_t group,
                             uint64_t max_decode_steps, uint32_t flags, csattn_session* out);
/* A layer's prefill: n sessions (one per KV head) with the same layout and
 * retrieval config, index configs icfgs[0..n) (e.g. per-head seeds), built with
 * ONE k-means launch of n x m CTAs (one launch per session leaves most SMs
 * idle). Session i equals csattn_prefill of rows[i] with icfgs[i]. */
typedef struct {
    const float* queries; /* n_queries x d */
    uint64_t n_queries;
    const float* keys;    /* n_rows x d */
    const float* values;  /* n_rows x d */
    uint64_t n_rows;
} csattn_prefill_rows;
csattn_status csattn_prefill_batch(csattn_ctx ctx, uint64_t n, const csattn_prefill_rows* rows,
                                   uint64_t d, const uint64_t* widths, uint64_t m,
                                   const csattn_index_config* icfgs,
                                   const csattn_retrieval_config* rcfg, uint64_t group,
                                   uint64_t max_decode_steps, uint32_t flags, csattn_session* out);

/* build_index_from_centroids (index.cpp:179-202): caller-supplied unit centroid
 * rows, packed per subspace: subspace b holds C x widths[b] floats, subspaces
 * concatenated (C*d floats total). Always host memory. */
csattn_status csattn_prefill_from_centroids(csattn_ctx ctx, const float* centroids,
                                            uint64_t c, const float* keys,
                                            const float* values, uint64_t p, uint64_t d,
                                            const uint64_t* widths, uint64_t m,
                                            const csattn_index_config* icfg,
                                            const csattn_retrieval_config* rcfg,
                                            uint64_t group, uint64_t max_decode_steps,
                                            uint32_t flags, csattn_session* out);

/* Adopt a host CsIndex image (the offline -> online handoff; reference layout:
 * per table t = b*C + j, lens[t] entries in TopList order (score desc, index
 * asc), stored at indices/scores + t*stride). Host memory only. */
csattn_status csattn_session_import(csattn_ctx ctx, const float* centroids, uint64_t c,
                                    const uint32_t* lens, const uint32_t* indices,
                                    const float* scores, uint64_t stride,
                                    uint64_t list_capacity, double alpha,
                                    int32_t normalize_keys, int32_t score_bits,
                                    const float* keys, const float* values, uint64_t p,
                                    uint64_t d, const uint64_t* widths, uint64_t m,
                                    const csattn_retrieval_config* rcfg, uint64_t group,
                                    uint64_t max_decode_steps, csattn_session* out);

/* Export the current tables in reference TopList order (score desc, index asc).
 * lens: m*C; indices/scores: m*C*stride (stride >= L); centroids: C*d (nullable).
 * Host memory. */
csattn_status csattn_session_export(csattn_session s, uint32_t* lens, uint32_t* indices,
                                    float* scores, uint64_t stride, float* centroids);

/* The per-subspace unit centroids (CsIndex::centroid_sets, index.hpp:46-68),
 * packed per subspace as for csattn_prefill_from_centroids: C*d floats, host. */
csattn_status csattn_session_centroids(csattn_session s, float* centroids);

/* Independent copy (Session is a value type, session.hpp:19-31): tables are
 * copied, the immutable prefill KV rows are shared. */
csattn_status csattn_session_fork(csattn_session src, uint64_t max_decode_steps,
                                  csattn_session* out);
csattn_status csattn_session_destroy(csattn_session s);
csattn_status csattn_session_info_get(csattn_session s, csattn_session_info* out);
csattn_status csattn_session_set_retrieval(csattn_session s, const csattn_retrieval_config* rcfg);
/* SearchState::cached (retrieval.hpp:88-94): the CandidateSet of the last
 * search of query head `head` — ascending key indices with their fp64
 * accumulated scores (reduce_by_key, retrieval.cpp:111-148). Candidates are
 * kept on the device only when the search period is > 1 or after
 * keep_candidates(s, 1). Host memory; *n receives the candidate count. */
csattn_status csattn_session_keep_candidates(csattn_session s, int32_t enable);
csattn_status csattn_session_candidates(csattn_session s, uint64_t head, uint32_t* indices,
                                        double* scores, uint64_t cap, uint64_t* n);
/* Gather accounting of the last search of every query head (bench/roofline):
 * total = sum over heads of the gathered lists' live entries
 * (CostCounters::gathered_entries), unique = live entries of the union of the
 * heads' gathered tables (what one pass over HBM must read). */
csattn_status csattn_session_gather_stats(csattn_session s, uint64_t* unique_entries,
                                          uint64_t* total_entries);

/* KvStore rows back to the host (core.cpp:84-90): rows [first, first+count). */
csattn_status csattn_session_read_kv(csattn_session s, uint64_t first, uint64_t count,
                                     float* keys, float* values);

/* ---- online decode ----
 * decode_step (session.cpp:46-99) for every query head of the group:
 * decode_search (retrieval.cpp:230-270) -> masked dense_attention
 * (core.cpp:118-169) -> KvStore::append (core.cpp:71-79) -> streaming_insert
 * (retrieval.cpp:272-301).
 *   q:        group x d        new_key, new_value: d
 *   out:      group x d        (nullable)
 *   selected: group x sel_stride uint32, ascending (nullable)
 *   weights:  group x sel_stride f32 softmax weights in selected order (nullable)
 *   reports:  group reports, host memory (nullable)
 *   k_override: group entries, host memory (nullable; 0 = keep_count) — the
 *               ABI form of RetrievalConfig::k_bump.
 * compare_dense is not part of the hot path (see csattn_dense_attention). */
csattn_status csattn_decode_step(csattn_session s, const float* q, const float* new_key,
                                 const float* new_value, float* out, uint32_t* selected,
                                 float* weights, uint64_t sel_stride,
                                 csattn_step_report* reports, const uint64_t* k_override,
                                 uint32_t flags);

/* One decode step for many sessions at once (a layer: KV heads x sequences),
 * one kernel launch per stage. sessions[i] has group g_i; q holds
 * sum_i g_i rows in session order, new_keys/new_values one row per session.
 * out: sum_i g_i rows (nullable). selected: sum_i g_i rows of sel_stride. */
csattn_status csattn_decode_batch(csattn_ctx ctx, uint64_t n_sessions,
                                  const csattn_session* sessions, const float* q,
                                  const float* new_keys, const float* new_values, float* out,
                                  uint32_t* selected, uint64_t sel_stride, uint32_t flags);

/* run_decode over n_steps steps of a session set as ONE CUDA graph (SURVEY
 * §8(f) row 2; session.cpp:101-126 without the per-step reports): step t reads
 * q + t*nq*d, new_keys/new_values + t*n*d and writes out + t*nq*d and selected +
 * t*nq*sel_stride (either may be NULL); k_override, when given, is n_steps x nq
 * (0 = keep_count). The steps and their results equal n_steps calls of
 * csattn_decode_batch. Every session needs n_steps free decode steps (else
 * CSATTN_ERR_CAPACITY with no state changed). Synchronous. */
csattn_status csattn_decode_run(csattn_ctx ctx, uint64_t n_sessions, const csattn_session* sessions,
                                uint64_t n_steps, const float* q, const float* new_keys,
                                const float* new_values, float* out, uint32_t* selected,
                                uint64_t sel_stride, const uint64_t* k_override, uint32_t flags);

/* The dense oracle on the GPU, over the session's current
 * KV rows: masked (mask = n_mask row indices) or full (mask == NULL)
 * dense_attention (core.cpp:118-169): fp64 logits from the reference's
 * sequential dot, fp64 softmax, f32 weights in mask order, f32 output. Used for
 * compare_dense and recall at scale. Not on the decode hot path. */
csattn_status csattn_dense_attention(csattn_session s, const float* q, const uint32_t* mask,
                                     uint64_t n_mask, float* out, float* weights,
                                     uint32_t flags);
/* dense_topk (core.cpp:171-192): the k rows with the largest sequential-fp64
 * dot q.k (lower index first on equal scores), returned ascending. */
csattn_status csattn_dense_topk(csattn_session s, const float* q, uint64_t k, uint32_t* out,
                                uint32_t flags);

/* ---- Function-level API: the reference's free functions on host values ----
 * (index.hpp:79-96, retrieval.hpp:40-118, core.hpp:96-102). All buffers are
 * host memory; the work runs on ctx's device with the decode path's exact
 * arithmetic. The C++ facade wraps them with the reference's signatures. */

/* score_keys (index.cpp:68-91) generalised: for centroid j (widths[j] floats,
 * packed one after another in `centroids`, scoring key dims
 * [offsets[j], offsets[j] + widths[j])) and key i < n (keys: n x d):
 * out[j*n + i] = float(sum_t double(c[t]) * double(k_i[off + t])).
 * normalize: 0 raw keys; 1 score_keys' normalize_keys (divide by the slice
 * norm, zero slice -> 0); 2 streaming_insert's (retrieval.cpp:283-291: score
 * the l2_normalize'd f32 slice, zero slice -> 0). out64 (instead of out):
 * the unrounded fp64 sums (centroid_scores, clustering.cpp:242-250). */
csattn_status csattn_score_keys(csattn_ctx ctx, const float* centroids, uint64_t n_centroids,
                                const uint64_t* offsets, const uint64_t* widths, const float* keys,
                                uint64_t n, uint64_t d, int32_t normalize, float* out, double* out64);
/* TopList::from_scores (index.cpp:46-62): the min(capacity, n) best of n
 * scores by (score desc, index asc), in that order. */
csattn_status csattn_toplist_from_scores(csattn_ctx ctx, const float* scores, uint64_t n,
                                         uint64_t capacity, uint32_t* out_indices, float* out_scores,
                                         uint64_t* out_len);
/* select_centroids (retrieval.cpp:40-87) over unit centroids packed per
 * subspace (C x widths[b] floats each, subspaces concatenated): ids[b*tau ..]
 * the counts[b] selected centroid ids of subspace b (1, or up to tau on
 * backoff), best_cosine[b], dot_ops. */
csattn_status csattn_select_centroids(csattn_ctx ctx, const float* centroids, uint64_t c,
                                      const uint64_t* widths, uint64_t m, const float* q,
                                      uint64_t tau, double threshold, uint32_t* ids, uint32_t* counts,
                                      double* best_cosine, uint64_t* dot_ops);
/* reduce_by_key (retrieval.cpp:111-148): lists in gathered order with their
 * weights (w_b of each list's subspace) -> ascending unique keys, fp64 sums
 * of w * double(score) in list order, source counts. capacity bounds out_*. */
csattn_status csattn_reduce_by_key(csattn_ctx ctx, uint64_t n_lists, const uint64_t* lens,
                                   const uint32_t* const* indices, const float* const* scores,
                                   const double* weights, uint32_t* out_indices, double* out_scores,
                                   uint32_t* out_counts, uint64_t capacity, uint64_t* out_n);
/* select_topk (retrieval.cpp:150-228) of a candidate set (ascending keys,
 * fp64 scores) for a context of n keys: out gets K ascending indices (K =
 * k_override ? min(k_override, n) : keep_count(rho, n)), *out_k = K. Runs the
 * decode select kernel on the candidates as its cached scores. */
csattn_status csattn_select_topk(csattn_ctx ctx, const uint32_t* cand_indices, const double* cand_scores,
                                 uint64_t n_cand, uint64_t n, const csattn_retrieval_config* rcfg,
                                 uint64_t k_override, uint32_t* out, uint64_t* out_k);
/* dense_attention / dense_topk (core.cpp:118-192) over host rows (n x d). */
csattn_status csattn_dense_attention_rows(csattn_ctx ctx, const float* q, const float* keys,
                                          const float* values, uint64_t n, uint64_t d,
                                          const uint32_t* mask, uint64_t n_mask, float* out,
                                          float* weights);
csattn_status csattn_dense_topk_rows(csattn_ctx ctx, const float* q, const float* keys, uint64_t n,
                                     uint64_t d, uint64_t k, uint32_t* out);

/* ---- CSAT v1 index image (index.hpp:98-121) ----
 * Little-endian image written by serialize_index (index.cpp:289-318) and
 * validated by deserialize_index (:320-396): "CSAT" | version u16 | flags u16 |
 * m u32 | C u32 | L u32 | d u32 | prefill u64 | widths u32 x m | centroid rows |
 * per table: len u32, indices u32 x len, scores x len. Flag bit 0 stores
 * scores AND centroid elements as IEEE half (RNE), bit 1 marks normalized keys.
 * The codec below is host-only (no GPU needed); the session calls run the
 * table ordering and byte writing on the device. */
#define CSATTN_CSAT_MAX_SUBSPACES 32
typedef struct csattn_csat_header {
    uint64_t m, centroids, list_capacity, dim, prefill_len;
    int32_t score_bits;     /* 16 or 32 */
    int32_t normalize_keys; /* 0 / 1 */
    uint64_t widths[CSATTN_CSAT_MAX_SUBSPACES];
} csattn_csat_header;

/* f32_to_f16 / f16_to_f32 (util.cpp:8-74) */
uint16_t csattn_f32_to_f16(float value);
float csattn_f16_to_f32(uint16_t bits);
/* The header of an image (errors as deserialize_index through the widths). */
csattn_status csattn_csat_read_header(const uint8_t* bytes, uint64_t n, csattn_csat_header* header);
/* index_footprint (index.cpp:419-431): header (incl. widths and length
 * prefixes), centroid and entry bytes for the given list lengths. */
csattn_status csattn_csat_footprint(const csattn_csat_header* header, const uint32_t* lens,
                                    uint64_t* header_bytes, uint64_t* centroid_bytes,
                                    uint64_t* entry_bytes);
/* serialize_index over host tables in TopList order (lists of `stride`).
 * out == NULL: *size = bytes needed. */
csattn_status csattn_csat_encode(const csattn_csat_header* header, const float* centroids,
                                 const uint32_t* lens, const uint32_t* indices, const float* scores,
                                 uint64_t stride, uint8_t* out, uint64_t capacity, uint64_t* size);
/* deserialize_index: same check order, error classes and messages. Tables
 * land at `stride` >= list_capacity; centroids hold C x d floats. */
csattn_status csattn_csat_decode(const uint8_t* bytes, uint64_t n, csattn_csat_header* header,
                                 float* centroids, uint32_t* lens, uint32_t* indices,
                                 float* scores, uint64_t stride);
/* The session's current index (tables after any streaming inserts) as a CSAT
 * image: tables sorted into TopList order and encoded on the device, header
 * and centroids prepended on the host. out == NULL: *size = bytes needed. */
csattn_status csattn_session_serialize(csattn_session s, uint8_t* out, uint64_t capacity,
                                       uint64_t* size);
/* A session from a CSAT image plus the prefill KV rows it indexes
 * (load_index + KvStore + Session, session.hpp:19-31); n_rows must equal the
 * image's prefill length. */
csattn_status csattn_session_deserialize(csattn_ctx ctx, const uint8_t* bytes, uint64_t n,
                                         const float* keys, const float* values, uint64_t n_rows,
                                         const csattn_retrieval_config* rcfg, uint64_t group,
                                         uint64_t max_decode_steps, csattn_session* out);

/* ---- sequence sharding ----
 * A logical session (one KV head, P prefill keys) is split by key range over
 * shards. Shard s holds keys [key_lo, key_hi) of every global TopList (global
 * indices kept), their KV rows, and (owner shard only) the appended keys.
 * Boundaries are multiples of 4096 keys (the select tile). The global list
 * sizes and score bounds are replicated on every shard.
 *
 * A decode step runs as phases on every shard, in order, with the caller's
 * collectives between them (NCCL across GPUs, or plain device ops when the
 * shards share a GPU); the union of the shards' selections is exactly the
 * unsharded selection and the merged output agrees within 1e-3:
 *   SCAN    route + per-shard gather/accumulate/histogram -> io.ghist
 *           caller: all-reduce(sum, uint32) io.ghist over shards
 *   BUCKET  threshold bin; this shard's members of it -> io.bucket. If
 *           *io.spec_fail became non-zero the speculative cut missed: RESCAN,
 *           all-reduce, BUCKET again (every shard sees the same flag)
 *           caller: all-gather io.bucket -> io.bucket_all (shard order)
 *   MARK    global rank of the bucket; local selection -> io.counts (2/problem)
 *           caller: all-gather io.counts -> io.counts_all
 *   EMIT    newest-first padding across shards, local selection (ascending
 *           global indices -> io.selected / io.n_selected), sparse attention
 *           partials (max, sum, acc[d]) -> io.partial
 *           caller: all-gather io.partial -> io.partial_all
 *   MERGE   log-sum-exp merge -> io.out (every shard may run it)
 *   VICTIM  per table, this shard's next eviction key -> io.victim
 *           caller: all-reduce(min, uint64) io.victim
 *   INSERT  KvStore::append on the owner + global strict-win streaming insert
 * All io pointers are device pointers on the context's device. */
typedef enum csattn_shard_phase {
    CSATTN_SHARD_SCAN = 0,
    CSATTN_SHARD_BUCKET = 1,
    CSATTN_SHARD_MARK = 2,
    CSATTN_SHARD_EMIT = 3,
    CSATTN_SHARD_MERGE = 4,
    CSATTN_SHARD_VICTIM = 5,
    CSATTN_SHARD_INSERT = 6,
    CSATTN_SHARD_RESCAN = 7   /* SCAN without the speculative cut (after *io.spec_fail) */
} csattn_shard_phase;

typedef struct csattn_shard_io {
    const float* q;                  /* sum of groups x d */
    const float* new_keys;           /* n x d */
    const float* new_values;         /* n x d */
    uint32_t* ghist;                 /* nq x hist_words */
    uint32_t* bucket;                /* nq x bucket_words */
    const uint32_t* bucket_all;      /* n_shards x nq x bucket_words */
    uint32_t* counts;                /* nq x 2 */
    const uint32_t* counts_all;      /* n_shards x nq x 2 */
    float* partial;                  /* nq x (d + 2) */
    const float* partial_all;        /* n_shards x nq x (d + 2) */
    float* out;                      /* nq x d */
    uint32_t* selected;              /* nq x sel_stride (nullable) */
    uint32_t* n_selected;            /* nq (nullable) */
    uint64_t sel_stride;
    unsigned long long* victim;      /* n x m*C */
    uint32_t* spec_fail;             /* 1 word, set by BUCKET when the scan's speculative
                                        cut (the previous step's threshold) was too high:
                                        zero it, RESCAN, all-reduce, BUCKET again */
    uint32_t shard_index;
    uint32_t n_shards;
} csattn_shard_io;

/* Shard [key_lo, key_hi) of a freshly prefilled session (no decode steps
 * yet), created on context `ctx` (one context per shard: a context runs one
 * sharded step at a time). owner != 0: this shard also receives the appended
 * keys. */
csattn_status csattn_shard_create(csattn_ctx ctx, csattn_session full, uint64_t key_lo,
                                  uint64_t key_hi, int32_t owner, uint64_t max_decode_steps,
                                  csattn_session* out);
/* Buffer sizes per problem (hist, bucket: uint32 words; partial: floats) and
 * per session (victim: uint64 words). */
csattn_status csattn_shard_buffer_words(csattn_session shard, uint64_t* hist_words,
                                        uint64_t* bucket_words, uint64_t* partial_floats,
                                        uint64_t* victim_words);
/* One phase of a sharded decode step for n shard sessions of this shard
 * (one per KV head, groups as in csattn_decode_batch). Phases are enqueued on
 * the context's stream and never synchronize it: the collectives between
 * phases must run on (or be ordered with) that stream. */
csattn_status csattn_shard_step(csattn_ctx ctx, uint64_t n, const csattn_session* shards,
                                int32_t phase, const csattn_shard_io* io);
/* Local combine steps of the collectives between phases (device pointers,
 * enqueued on ctx's stream): dst[i] += src[i] over uint32 (histograms, flags),
 * dst[i] = min(dst[i], src[i]) over uint64 (victim keys). The C++ orchestrator
 * include/csattn_b200_shard.hpp uses them with its local / NCCL transports. */
csattn_status csattn_buffer_add_u32(csattn_ctx ctx, uint32_t* dst, const uint32_t* src, uint64_t count);
csattn_status csattn_buffer_min_u64(csattn_ctx ctx, uint64_t* dst, const uint64_t* src, uint64_t count);

#ifdef __cplusplus
}
#endif

#endif /* CSATTN_B200_H_ */
