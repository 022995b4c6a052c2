// csattn_b200.hpp — C++ drop-in facade of the B200 decode hot path.
//
// Mirrors the reference API in proj/include/csattn/ (same type names, field
// names, function names and exception classes) on top of the C ABI in
// csattn_b200.h, so reference call sites compile against it with
//
//     namespace csattn = csattn_b200;
//
// Covered (the hot path):
//   errors.hpp:8-52        Error, DimensionError, ParameterError, DataError (+4),
//                          PropertyError, StreamExhaustedError
//   core.hpp:23-39         SubspaceLayout (uniform, dim, count, slice)
//   core.hpp:74-79         AttentionOutput
//   clustering.hpp:17-28   ClusterConfig
//   index.hpp:19-42        TopList (host image), IndexConfig
//   index.hpp:46-68        CsIndex (host image: export of the device tables)
//   retrieval.hpp:17-38    RetrievalConfig (incl. k_bump), parse_schedule, keep_count
//   metrics.hpp:15-37      CostCounters
//   metrics.cpp:32-38      h2d_bytes
//   session.hpp:19-66      Session, DecodeStepReport, prefill, decode_step, run_decode
// Differences a caller can observe (documented in INTEGRATION.md):
//   * Session owns device state; `index` is materialised on demand by
//     Session::export_index() instead of being a public value member, and
//     KvStore rows live in HBM (Session::read_kv()).
//   * decode_step's compare_dense runs the dense oracle on the GPU
//     (csattn_dense_attention, csattn_dense_topk); recall/l2 follow on the host.
//   * k_bump is honoured: the callback's input (worst best-cosine of the
//     step's own routing) is evaluated on the host from the exported
//     centroids before the step is launched, exactly as decode_search
//     (retrieval.cpp:259-265) feeds it.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <fstream>
#include <string>
#include <utility>
#include <vector>

#include "csattn_b200.h"

namespace csattn_b200 {

// ---- errors.hpp:8-52 ----
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DimensionError : Error {
    using Error::Error;
};
struct ParameterError : Error {
    using Error::Error;
};
struct DataError : Error {
    using Error::Error;
};
struct BadMagicError : DataError {
    using DataError::DataError;
};
struct VersionError : DataError {
    using DataError::DataError;
};
struct TruncatedError : DataError {
    using DataError::DataError;
};
struct CorruptError : DataError {
    using DataError::DataError;
};
struct PropertyError : Error {
    using Error::Error;
};
struct StreamExhaustedError : Error {
    using Error::Error;
};
// B200-only failure classes (no reference counterpart)
struct CudaError : Error {
    using Error::Error;
};
struct CapacityError : ParameterError {
    using ParameterError::ParameterError;
};

// status -> the same exception class and message the reference throws
inline void check(csattn_status s) {
    if (s == CSATTN_OK) return;
    const std::string m = csattn_last_error();
    switch (s) {
        case CSATTN_ERR_DIMENSION: throw DimensionError(m);
        case CSATTN_ERR_PARAMETER: throw ParameterError(m);
        case CSATTN_ERR_DATA: throw DataError(m);
        case CSATTN_ERR_BAD_MAGIC: throw BadMagicError(m);
        case CSATTN_ERR_VERSION: throw VersionError(m);
        case CSATTN_ERR_TRUNCATED: throw TruncatedError(m);
        case CSATTN_ERR_CORRUPT: throw CorruptError(m);
        case CSATTN_ERR_PROPERTY: throw PropertyError(m);
        case CSATTN_ERR_STREAM_EXHAUSTED: throw StreamExhaustedError(m);
        case CSATTN_ERR_CUDA: throw CudaError(m);
        case CSATTN_ERR_CAPACITY: throw CapacityError(m);
        default: throw Error(m);
    }
}

using HeadVector = std::vector<float>;

// ---- core.hpp:23-39 / core.cpp:35-50 ----
struct SubspaceLayout {
    std::vector<std::size_t> sizes;
    std::vector<std::size_t> offsets;

    SubspaceLayout() = default;
    explicit SubspaceLayout(std::vector<std::size_t> subspace_sizes) : sizes(std::move(subspace_sizes)) {
        if (sizes.empty()) throw ParameterError("subspace layout needs m >= 1");
        std::size_t off = 0;
        for (std::size_t b = 0; b < sizes.size(); ++b) {
            if (sizes[b] == 0)
                throw ParameterError("subspace width must be >= 1 (subspace " + std::to_string(b) + ")");
            offsets.push_back(off);
            off += sizes[b];
        }
    }
    static SubspaceLayout uniform(std::size_t dim, std::size_t subspaces) {
        if (subspaces == 0 || subspaces > dim)
            throw ParameterError("uniform layout requires 1 <= m <= d");
        std::vector<std::size_t> s(subspaces, dim / subspaces);
        for (std::size_t b = 0; b < dim % subspaces; ++b) s[b] += 1;
        return SubspaceLayout(std::move(s));
    }
    std::size_t dim() const {
        std::size_t d = 0;
        for (std::size_t x : sizes) d += x;
        return d;
    }
    std::size_t count() const { return sizes.size(); }
    std::span<const float> slice(std::span<const float> v, std::size_t b) const {
        return v.subspan(offsets[b], sizes[b]);
    }
};

// ---- core.hpp:74-79 ----
struct AttentionOutput {
    std::vector<float> weights;
    HeadVector output;
};

// ---- clustering.hpp:17-28, index.hpp:19-68 ----
struct ClusterConfig {
    std::size_t centroids = 64;
    std::size_t iterations = 10;
    std::size_t batch_size = 0;
    std::uint64_t seed = 0;
    double tolerance = 1e-7;
};

struct IndexConfig {
    double alpha = 0.2;
    std::size_t list_capacity = 0;
    bool normalize_keys = false;
    int score_bits = 16;
    ClusterConfig cluster;

    csattn_index_config c() const {
        csattn_index_config x{};
        x.alpha = alpha;
        x.list_capacity = list_capacity;
        x.normalize_keys = normalize_keys ? 1 : 0;
        x.score_bits = score_bits;
        x.centroids = cluster.centroids;
        x.iterations = cluster.iterations;
        x.batch_size = cluster.batch_size;
        x.seed = cluster.seed;
        x.tolerance = cluster.tolerance;
        return x;
    }
};

struct TopList {
    std::uint32_t capacity = 0;
    std::vector<std::uint32_t> indices;  // score desc, index asc
    std::vector<float> scores;
    bool full() const { return indices.size() >= capacity; }
    float min_score() const {
        return scores.empty() ? -std::numeric_limits<float>::infinity() : scores.back();
    }
    // index.cpp:22-44: a full list admits (index, score) only when the score
    // strictly beats its minimum (evicting it); sorted position by (score
    // desc, index asc). A host value-type operation: the device tables of a
    // Session take the same decision in insert.cu.
    bool try_insert(std::uint32_t index, float score) {
        if (capacity == 0) return false;
        if (full()) {
            if (!(score > scores.back())) return false;
            scores.pop_back();
            indices.pop_back();
        }
        std::size_t lo = 0, hi = scores.size();
        while (lo < hi) {
            const std::size_t mid = (lo + hi) / 2;
            const bool precedes = scores[mid] != score ? scores[mid] > score : indices[mid] < index;
            if (precedes) lo = mid + 1;
            else hi = mid;
        }
        scores.insert(scores.begin() + static_cast<std::ptrdiff_t>(lo), score);
        indices.insert(indices.begin() + static_cast<std::ptrdiff_t>(lo), index);
        return true;
    }
    // index.cpp:46-62, on the device (defined below)
    static TopList from_scores(std::span<const float> scores, std::uint32_t capacity);
};

// clustering.hpp:31-41
struct FitStats {
    std::vector<double> objective;
    std::size_t reseeded = 0;
    std::size_t degenerate_points = 0;
    std::size_t duplicated_seeds = 0;
    std::size_t dot_ops = 0;
};

struct CentroidSet {
    std::size_t subspace_id = 0;
    std::vector<float> centroids;  // count x dim, unit rows
    std::size_t count = 0;
    std::size_t dim = 0;
    FitStats stats;
    std::span<const float> centroid(std::size_t j) const { return {centroids.data() + j * dim, dim}; }
};

// Host image of the device tables (Session::export_index).
struct CsIndex {
    SubspaceLayout layout;
    std::vector<CentroidSet> centroid_sets;
    std::vector<TopList> tables;  // m x C, subspace-major
    double alpha = 0.0;
    std::uint32_t list_capacity = 0;
    std::uint64_t prefill_len = 0;
    bool normalize_keys = false;
    int score_bits = 16;

    explicit CsIndex(SubspaceLayout l) : layout(std::move(l)) {}
    std::size_t subspaces() const { return layout.count(); }
    std::size_t centroids_per_subspace() const {
        return centroid_sets.empty() ? 0 : centroid_sets[0].count;
    }
    TopList& table(std::size_t b, std::size_t j) { return tables[b * centroids_per_subspace() + j]; }
    const TopList& table(std::size_t b, std::size_t j) const {
        return tables[b * centroids_per_subspace() + j];
    }
};

// ---- retrieval.hpp:17-38 ----
struct RetrievalConfig {
    double keep_ratio = 0.05;
    std::size_t search_period = 1;
    std::size_t recent_window = 32;
    std::vector<double> weights;
    std::size_t backoff_tau = 1;
    double backoff_threshold = -std::numeric_limits<double>::infinity();
    bool recent_passthrough = true;
    std::function<std::size_t(std::size_t, double)> k_bump;

    csattn_retrieval_config c() const {
        csattn_retrieval_config x{};
        x.keep_ratio = keep_ratio;
        x.search_period = search_period;
        x.recent_window = recent_window;
        x.weights = weights.empty() ? nullptr : weights.data();
        x.n_weights = weights.size();
        x.backoff_tau = backoff_tau;
        x.backoff_threshold = backoff_threshold;
        x.recent_passthrough = recent_passthrough ? 1 : 0;
        return x;
    }
};

inline std::size_t keep_count(double rho, std::size_t n) {
    uint64_t k = 0;
    check(csattn_keep_count(rho, n, &k));
    return static_cast<std::size_t>(k);
}

inline std::pair<double, std::size_t> parse_schedule(const std::string& name) {
    double rho = 0.0;
    uint64_t period = 0;
    check(csattn_parse_schedule(name.c_str(), &rho, &period));
    return {rho, static_cast<std::size_t>(period)};
}

// ---- metrics.hpp:15-37, metrics.cpp:32-38 ----
struct CostCounters {
    std::size_t centroid_dot_ops = 0;
    std::size_t gathered_entries = 0;
    std::size_t reduce_ops = 0;
    std::size_t attention_key_ops = 0;
    double h2d_bytes_model = 0.0;
    std::size_t searches = 0;
    std::size_t inserts_attempted = 0;
    std::size_t inserts_applied = 0;
    std::size_t insert_dot_ops = 0;

    void add(const CostCounters& o) {
        centroid_dot_ops += o.centroid_dot_ops;
        gathered_entries += o.gathered_entries;
        reduce_ops += o.reduce_ops;
        attention_key_ops += o.attention_key_ops;
        h2d_bytes_model += o.h2d_bytes_model;
        searches += o.searches;
        inserts_attempted += o.inserts_attempted;
        inserts_applied += o.inserts_applied;
        insert_dot_ops += o.insert_dot_ops;
    }
};

inline double h2d_bytes(double rho, std::size_t n, std::size_t d, std::size_t b, std::size_t period) {
    double out = 0.0;
    check(csattn_h2d_bytes(rho, n, d, b, period, &out));
    return out;
}

// ---- one device + stream (no reference counterpart: the CPU path has none) ----
class Context {
   public:
    explicit Context(int device = 0, void* cuda_stream = nullptr) {
        check(csattn_ctx_create(device, cuda_stream, &h_));
    }
    ~Context() {
        if (h_) csattn_ctx_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    csattn_ctx handle() const { return h_; }
    uint64_t launches() const { return csattn_ctx_launch_count(h_); }
    static Context& default_context() {
        static Context c(0);
        return c;
    }

   private:
    csattn_ctx h_ = nullptr;
};

// ===========================================================================
// Function-level API (core.hpp:47-102, index.hpp:79-96, retrieval.hpp:40-118):
// the reference's free functions on host values. Compute runs on the device
// through the C ABI (score_keys / TopList::from_scores / select_centroids /
// reduce_by_key / select_topk / dense_attention / dense_topk / the insert
// scoring); container bookkeeping (KvStore rows, gather_lists views,
// TopList::try_insert on a host list) stays with the host value, as in the
// reference. A Session is the device-resident form of the same path.
// ===========================================================================

// ---- core.hpp:47-68 / core.cpp:52-88 ----
class KvStore {
   public:
    explicit KvStore(std::size_t dim) : dim_(dim) {
        if (dim == 0) throw ParameterError("head dimension must be >= 1");
    }
    KvStore(std::size_t dim, std::span<const float> prefill_keys, std::span<const float> prefill_values)
        : KvStore(dim) {
        if (prefill_keys.size() % dim != 0 || prefill_values.size() % dim != 0)
            throw DimensionError("prefill rows are not a multiple of d");
        if (prefill_keys.size() != prefill_values.size())
            throw DimensionError("prefill key/value counts differ");
        require_finite(prefill_keys, "prefill keys");
        require_finite(prefill_values, "prefill values");
        keys_.assign(prefill_keys.begin(), prefill_keys.end());
        values_.assign(prefill_values.begin(), prefill_values.end());
        prefill_len_ = prefill_keys.size() / dim;
        total_len_ = prefill_len_;
    }
    void append(std::span<const float> key, std::span<const float> value) {
        if (key.size() != dim_ || value.size() != dim_)
            throw DimensionError("appended key/value width does not match d");
        require_finite(key, "appended key");
        require_finite(value, "appended value");
        keys_.insert(keys_.end(), key.begin(), key.end());
        values_.insert(values_.end(), value.begin(), value.end());
        total_len_ += 1;
    }
    std::span<const float> key(std::size_t i) const { return {keys_.data() + i * dim_, dim_}; }
    std::span<const float> value(std::size_t i) const { return {values_.data() + i * dim_, dim_}; }
    std::size_t dim() const { return dim_; }
    std::size_t size() const { return total_len_; }
    std::size_t prefill_len() const { return prefill_len_; }
    const float* key_data() const { return keys_.data(); }
    const float* value_data() const { return values_.data(); }

   private:
    static void require_finite(std::span<const float> v, const char* what) {
        for (float x : v)
            if (!std::isfinite(x)) throw DataError(std::string(what) + " contains a non-finite value");
    }
    std::size_t dim_;
    std::size_t prefill_len_ = 0;
    std::size_t total_len_ = 0;
    std::vector<float> keys_, values_;
};

// core.cpp:89-116: value helpers the callers use to prepare inputs
inline double dot(std::span<const float> a, std::span<const float> b) {
    double acc = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) acc += static_cast<double>(a[i]) * static_cast<double>(b[i]);
    return acc;
}
inline std::vector<std::span<const float>> split_subspaces(std::span<const float> v, const SubspaceLayout& layout) {
    if (v.size() != layout.dim())
        throw DimensionError("vector length " + std::to_string(v.size()) + " does not match layout dimension " +
                             std::to_string(layout.dim()));
    std::vector<std::span<const float>> out;
    for (std::size_t b = 0; b < layout.count(); ++b) out.push_back(layout.slice(v, b));
    return out;
}
inline bool l2_normalize(std::span<float> v) {
    double norm2 = 0.0;
    for (float x : v) norm2 += static_cast<double>(x) * static_cast<double>(x);
    if (norm2 == 0.0) return true;
    const double inv = 1.0 / std::sqrt(norm2);
    for (float& x : v) x = static_cast<float>(x * inv);
    return false;
}

// core.cpp:118-169 (masked or full), on the device
inline AttentionOutput dense_attention(std::span<const float> q, const KvStore& kv,
                                       std::optional<std::span<const std::uint32_t>> mask = std::nullopt,
                                       Context& ctx = Context::default_context()) {
    if (kv.size() == 0) throw ParameterError("attention over an empty KV store");
    if (q.size() != kv.dim()) throw DimensionError("query width does not match KV dimension");
    if (mask && mask->empty()) throw ParameterError("attention over an empty index set");
    const std::size_t rows = mask ? mask->size() : kv.size();
    AttentionOutput out;
    out.output.resize(kv.dim());
    out.weights.resize(rows);
    check(csattn_dense_attention_rows(ctx.handle(), q.data(), kv.key_data(), kv.value_data(), kv.size(),
                                      kv.dim(), mask ? mask->data() : nullptr, mask ? mask->size() : 0,
                                      out.output.data(), out.weights.data()));
    return out;
}

// core.cpp:171-192, on the device
inline std::vector<std::uint32_t> dense_topk(std::span<const float> q, const KvStore& kv, std::size_t k,
                                             Context& ctx = Context::default_context()) {
    if (k < 1 || k > kv.size()) throw ParameterError("top-k count out of range: " + std::to_string(k));
    if (q.size() != kv.dim()) throw DimensionError("query width does not match KV dimension");
    std::vector<std::uint32_t> out(k);
    check(csattn_dense_topk_rows(ctx.handle(), q.data(), kv.key_data(), kv.size(), kv.dim(), k, out.data()));
    return out;
}

// clustering.cpp:242-250: every centroid's fp64 dot with v (v as given), on the device
inline std::vector<double> centroid_scores(std::span<const float> v, const CentroidSet& cs,
                                           Context& ctx = Context::default_context()) {
    if (v.size() != cs.dim) throw DimensionError("vector width does not match centroid width");
    std::vector<double> out(cs.count);
    if (cs.count == 0) return out;
    std::vector<uint64_t> off(cs.count, 0), wid(cs.count, cs.dim);
    check(csattn_score_keys(ctx.handle(), cs.centroids.data(), cs.count, off.data(), wid.data(), v.data(), 1,
                            cs.dim, 0, nullptr, out.data()));
    return out;
}

inline TopList TopList::from_scores(std::span<const float> scores, std::uint32_t capacity) {
    TopList l;
    l.capacity = capacity;
    const std::size_t keep = std::min<std::size_t>(capacity, scores.size());
    l.indices.resize(keep);
    l.scores.resize(keep);
    if (keep == 0) return l;
    uint64_t n = 0;
    check(csattn_toplist_from_scores(Context::default_context().handle(), scores.data(), scores.size(), capacity,
                                     l.indices.data(), l.scores.data(), &n));
    return l;
}

// ---- index.hpp:79-96 ----
struct BuildStats {
    std::size_t cluster_dot_ops = 0;  // not reported by the device k-means (stays 0)
    std::size_t score_dot_ops = 0;
};

// index.cpp:68-91, on the device
inline std::vector<float> score_keys(std::span<const float> centroid, const KvStore& kv,
                                     const SubspaceLayout& layout, std::size_t b, bool normalize_keys,
                                     std::size_t n_keys, Context& ctx = Context::default_context()) {
    if (b >= layout.count()) throw ParameterError("subspace id out of range");
    if (centroid.size() != layout.sizes[b]) throw DimensionError("centroid width does not match subspace width");
    if (n_keys > kv.size()) throw ParameterError("asked to score more keys than the store holds");
    std::vector<float> out(n_keys);
    if (n_keys == 0) return out;
    const uint64_t off = layout.offsets[b], wid = layout.sizes[b];
    check(csattn_score_keys(ctx.handle(), centroid.data(), 1, &off, &wid, kv.key_data(), n_keys, kv.dim(),
                            normalize_keys ? 1 : 0, out.data(), nullptr));
    return out;
}

namespace detail {
inline void validate_index_config(const IndexConfig& c) {
    if (c.list_capacity == 0 && !(c.alpha > 0.0 && c.alpha <= 1.0))
        throw ParameterError("alpha must lie in (0, 1]");
    if (c.score_bits != 16 && c.score_bits != 32) throw ParameterError("score width must be 16 or 32 bits");
    if (c.cluster.centroids == 0) throw ParameterError("centroid count must be >= 1");
}
// the tables of a device session, as the host CsIndex (TopList order)
inline CsIndex index_of(csattn_session h, const SubspaceLayout& layout) {
    csattn_session_info in{};
    check(csattn_session_info_get(h, &in));
    const std::size_t T = in.subspaces * in.centroids;
    const std::size_t stride = std::max<std::size_t>(in.list_capacity, 1);
    std::vector<uint32_t> lens(T), idx(T * stride);
    std::vector<float> sc(T * stride), cent(in.centroids * in.dim);
    check(csattn_session_export(h, lens.data(), idx.data(), sc.data(), stride, cent.data()));
    CsIndex ix(layout);
    ix.alpha = in.alpha;
    ix.list_capacity = static_cast<uint32_t>(in.list_capacity);
    ix.prefill_len = in.prefill_len;
    ix.normalize_keys = in.normalize_keys != 0;
    ix.score_bits = in.score_bits;
    for (std::size_t b = 0; b < layout.count(); ++b) {
        CentroidSet cs;
        cs.subspace_id = b;
        cs.count = in.centroids;
        cs.dim = layout.sizes[b];
        const float* src = cent.data() + in.centroids * layout.offsets[b];
        cs.centroids.assign(src, src + cs.count * cs.dim);
        ix.centroid_sets.push_back(std::move(cs));
    }
    for (std::size_t t = 0; t < T; ++t) {
        TopList l;
        l.capacity = static_cast<uint32_t>(in.list_capacity);
        l.indices.assign(idx.begin() + t * stride, idx.begin() + t * stride + lens[t]);
        l.scores.assign(sc.begin() + t * stride, sc.begin() + t * stride + lens[t]);
        ix.tables.push_back(std::move(l));
    }
    return ix;
}
struct SessionHandle {  // a transient device session
    csattn_session h = nullptr;
    ~SessionHandle() {
        if (h) csattn_session_destroy(h);
    }
};
}  // namespace detail

// index.cpp:145-177: device k-means per subspace + device tables, exported
inline CsIndex build_index(std::span<const float> queries, std::size_t query_count, const KvStore& kv,
                           const SubspaceLayout& layout, const IndexConfig& config, BuildStats* stats = nullptr,
                           Context& ctx = Context::default_context()) {
    detail::validate_index_config(config);
    if (query_count == 0) throw ParameterError("need at least one query row");
    if (queries.size() != query_count * layout.dim()) throw DimensionError("query buffer does not match count x d");
    if (layout.dim() != kv.dim()) throw DimensionError("layout dimension does not match KV dimension");
    if (kv.prefill_len() == 0) throw ParameterError("cannot build over an empty prefill");
    const std::size_t d = kv.dim(), p = kv.prefill_len();
    std::vector<uint64_t> widths(layout.sizes.begin(), layout.sizes.end());
    const csattn_index_config ic = config.c();
    const csattn_retrieval_config rc = RetrievalConfig{}.c();
    detail::SessionHandle s;
    check(csattn_prefill(ctx.handle(), queries.data(), query_count, kv.key_data(), kv.value_data(), p, d,
                         widths.data(), widths.size(), &ic, &rc, 1, 1, CSATTN_HOST_BUFFERS, &s.h));
    CsIndex ix = detail::index_of(s.h, layout);
    if (stats) stats->score_dot_ops += p * d * ix.centroids_per_subspace();
    return ix;
}

// index.cpp:179-202: the same tables from given centroids, on the device
inline CsIndex build_index_from_centroids(std::vector<CentroidSet> centroid_sets, const KvStore& kv,
                                          const SubspaceLayout& layout, const IndexConfig& config,
                                          BuildStats* stats = nullptr,
                                          Context& ctx = Context::default_context()) {
    detail::validate_index_config(config);
    if (layout.dim() != kv.dim()) throw DimensionError("layout dimension does not match KV dimension");
    if (kv.prefill_len() == 0) throw ParameterError("cannot build over an empty prefill");
    if (centroid_sets.size() != layout.count()) throw DimensionError("need one centroid set per subspace");
    const std::size_t c = centroid_sets[0].count;
    if (c == 0) throw ParameterError("centroid sets are empty");
    std::vector<float> packed;
    for (std::size_t b = 0; b < centroid_sets.size(); ++b) {
        if (centroid_sets[b].count != c) throw DimensionError("centroid counts differ across subspaces");
        if (centroid_sets[b].dim != layout.sizes[b])
            throw DimensionError("centroid width does not match subspace " + std::to_string(b));
        packed.insert(packed.end(), centroid_sets[b].centroids.begin(),
                      centroid_sets[b].centroids.begin() + static_cast<std::ptrdiff_t>(c * layout.sizes[b]));
    }
    const std::size_t d = kv.dim(), p = kv.prefill_len();
    std::vector<uint64_t> widths(layout.sizes.begin(), layout.sizes.end());
    IndexConfig cfg = config;
    cfg.cluster.centroids = c;
    const csattn_index_config ic = cfg.c();
    const csattn_retrieval_config rc = RetrievalConfig{}.c();
    detail::SessionHandle s;
    check(csattn_prefill_from_centroids(ctx.handle(), packed.data(), c, kv.key_data(), kv.value_data(), p, d,
                                        widths.data(), widths.size(), &ic, &rc, 1, 1, CSATTN_HOST_BUFFERS, &s.h));
    CsIndex ix = detail::index_of(s.h, layout);
    for (std::size_t b = 0; b < ix.centroid_sets.size(); ++b) ix.centroid_sets[b].stats = centroid_sets[b].stats;
    if (stats) stats->score_dot_ops += p * d * c;
    return ix;
}

// ---- retrieval.hpp:41-118 ----
struct CandidateSet {
    std::vector<std::uint32_t> indices;        // ascending
    std::vector<double> scores;                // aligned weighted sums
    std::vector<std::uint32_t> source_counts;  // contributing subspaces
    std::size_t size() const { return indices.size(); }
};

struct CentroidSelection {
    std::vector<std::vector<std::uint32_t>> per_subspace;
    std::vector<double> best_cosine;
    std::size_t dot_ops = 0;
};

// retrieval.cpp:40-87, on the device (route.cu)
inline CentroidSelection select_centroids(std::span<const float> q, const CsIndex& index, std::size_t tau,
                                          double threshold, Context& ctx = Context::default_context()) {
    if (q.size() != index.layout.dim()) throw DimensionError("query width does not match index dimension");
    if (tau == 0) throw ParameterError("backoff tau must be >= 1");
    const std::size_t m = index.subspaces(), c = index.centroids_per_subspace();
    std::vector<float> packed;
    for (const CentroidSet& cs : index.centroid_sets)
        packed.insert(packed.end(), cs.centroids.begin(), cs.centroids.end());
    std::vector<uint64_t> widths(index.layout.sizes.begin(), index.layout.sizes.end());
    std::vector<uint32_t> ids(m * tau), counts(m);
    CentroidSelection sel;
    sel.best_cosine.resize(m);
    uint64_t dots = 0;
    check(csattn_select_centroids(ctx.handle(), packed.data(), c, widths.data(), m, q.data(), tau, threshold,
                                  ids.data(), counts.data(), sel.best_cosine.data(), &dots));
    sel.dot_ops = dots;
    for (std::size_t b = 0; b < m; ++b)
        sel.per_subspace.emplace_back(ids.begin() + static_cast<std::ptrdiff_t>(b * tau),
                                      ids.begin() + static_cast<std::ptrdiff_t>(b * tau + counts[b]));
    return sel;
}

struct GatheredLists {
    std::vector<const TopList*> lists;
    std::vector<std::size_t> subspace;
    std::size_t total_entries() const {
        std::size_t n = 0;
        for (const TopList* l : lists) n += l->indices.size();
        return n;
    }
};

// retrieval.cpp:95-109: views of the selected tables, (b, selection) order
inline GatheredLists gather_lists(const CsIndex& index, const CentroidSelection& selection) {
    if (selection.per_subspace.size() != index.subspaces())
        throw DimensionError("selection does not cover every subspace");
    GatheredLists out;
    for (std::size_t b = 0; b < selection.per_subspace.size(); ++b)
        for (std::uint32_t j : selection.per_subspace[b]) {
            if (j >= index.centroids_per_subspace()) throw ParameterError("centroid id out of range");
            out.lists.push_back(&index.table(b, j));
            out.subspace.push_back(b);
        }
    return out;
}

// retrieval.cpp:111-148, on the device (fnapi.cu reduce_lists_kernel)
inline CandidateSet reduce_by_key(const GatheredLists& gathered, std::span<const double> weights,
                                  Context& ctx = Context::default_context()) {
    const std::size_t nl = gathered.lists.size();
    std::vector<uint64_t> lens(nl);
    std::vector<const uint32_t*> idx(nl);
    std::vector<const float*> sc(nl);
    std::vector<double> w(nl);
    for (std::size_t l = 0; l < nl; ++l) {
        const std::size_t b = gathered.subspace[l];
        if (b >= weights.size()) throw DimensionError("need one weight per subspace");
        w[l] = weights[b];
        lens[l] = gathered.lists[l]->indices.size();
        idx[l] = gathered.lists[l]->indices.data();
        sc[l] = gathered.lists[l]->scores.data();
    }
    const std::size_t cap = gathered.total_entries();
    CandidateSet out;
    out.indices.resize(cap);
    out.scores.resize(cap);
    out.source_counts.resize(cap);
    uint64_t n = 0;
    if (cap)
        check(csattn_reduce_by_key(ctx.handle(), nl, lens.data(), idx.data(), sc.data(), w.data(),
                                   out.indices.data(), out.scores.data(), out.source_counts.data(), cap, &n));
    out.indices.resize(n);
    out.scores.resize(n);
    out.source_counts.resize(n);
    return out;
}

// retrieval.cpp:150-228, on the device (the decode select kernel over the
// candidates as its cached scores)
inline std::vector<std::uint32_t> select_topk(const CandidateSet& candidates, const KvStore& kv,
                                              const RetrievalConfig& cfg, std::size_t k_override = 0,
                                              Context& ctx = Context::default_context()) {
    const std::size_t n = kv.size();
    if (n == 0) throw ParameterError("cannot select from an empty context");
    const std::size_t k = k_override ? std::min(k_override, n) : keep_count(cfg.keep_ratio, n);
    std::vector<std::uint32_t> out(k);
    uint64_t got = 0;
    const csattn_retrieval_config rc = cfg.c();
    check(csattn_select_topk(ctx.handle(), candidates.indices.data(), candidates.scores.data(), candidates.size(),
                             n, &rc, k_override, out.data(), &got));
    out.resize(got);
    return out;
}

struct SearchState {
    std::size_t step = 0;
    CandidateSet cached;
    bool has_cache = false;
    CentroidSelection last_selection;
};

struct SearchResult {
    std::vector<std::uint32_t> selected;
    std::size_t k = 0;
    bool searched = false;
    std::size_t centroid_dot_ops = 0;
    std::size_t gathered_entries = 0;
    std::size_t reduce_ops = 0;
};

// retrieval.cpp:230-270: the same composition, each stage on the device
inline SearchResult decode_search(std::span<const float> q, const CsIndex& index, const KvStore& kv,
                                  const RetrievalConfig& cfg, SearchState& state,
                                  Context& ctx = Context::default_context()) {
    if (cfg.search_period == 0) throw ParameterError("search period must be >= 1");
    SearchResult result;
    result.searched = !state.has_cache || state.step % cfg.search_period == 0;
    if (result.searched) {
        CentroidSelection sel = select_centroids(q, index, cfg.backoff_tau, cfg.backoff_threshold, ctx);
        const GatheredLists gathered = gather_lists(index, sel);
        std::vector<double> ones;
        std::span<const double> w = cfg.weights;
        if (w.empty()) {
            ones.assign(index.subspaces(), 1.0);
            w = ones;
        } else if (w.size() != index.subspaces()) {
            throw DimensionError("need one weight per subspace");
        }
        result.centroid_dot_ops = sel.dot_ops;
        result.gathered_entries = gathered.total_entries();
        result.reduce_ops = result.gathered_entries;
        state.cached = reduce_by_key(gathered, w, ctx);
        state.last_selection = std::move(sel);
        state.has_cache = true;
    }
    std::size_t k_override = 0;
    if (cfg.k_bump) {
        double worst = 1.0;
        for (double c : state.last_selection.best_cosine) worst = std::min(worst, c);
        k_override = cfg.k_bump(keep_count(cfg.keep_ratio, kv.size()), worst);
    }
    result.selected = select_topk(state.cached, kv, cfg, k_override, ctx);
    result.k = result.selected.size();
    state.step += 1;
    return result;
}

struct InsertReport {
    std::size_t attempted = 0;
    std::size_t applied = 0;
    std::size_t dot_ops = 0;
    std::vector<std::uint8_t> applied_mask;
};

// retrieval.cpp:272-301: the key's m x C scores on the device (the
// l2_normalize'd slices when the index normalizes keys), then each host
// table's strict-win admission
inline InsertReport streaming_insert(std::span<const float> new_key, std::uint32_t key_index, CsIndex& index,
                                     Context& ctx = Context::default_context()) {
    if (new_key.size() != index.layout.dim()) throw DimensionError("key width does not match index dimension");
    const std::size_t m = index.subspaces(), c = index.centroids_per_subspace();
    InsertReport report;
    report.applied_mask.assign(m * c, 0);
    if (m * c == 0) return report;
    std::vector<float> packed;
    std::vector<uint64_t> off, wid;
    for (std::size_t b = 0; b < m; ++b) {
        const CentroidSet& cs = index.centroid_sets[b];
        packed.insert(packed.end(), cs.centroids.begin(), cs.centroids.end());
        for (std::size_t j = 0; j < c; ++j) {
            off.push_back(index.layout.offsets[b]);
            wid.push_back(index.layout.sizes[b]);
        }
    }
    std::vector<float> s(m * c);
    check(csattn_score_keys(ctx.handle(), packed.data(), m * c, off.data(), wid.data(), new_key.data(), 1,
                            index.layout.dim(), index.normalize_keys ? 2 : 0, s.data(), nullptr));
    for (std::size_t b = 0; b < m; ++b)
        for (std::size_t j = 0; j < c; ++j) {
            report.dot_ops += index.centroid_sets[b].dim;
            report.attempted += 1;
            if (index.table(b, j).try_insert(key_index, s[b * c + j])) {
                report.applied += 1;
                report.applied_mask[b * c + j] = 1;
            }
        }
    return report;
}

// ---- session.hpp:19-42 ----
struct DecodeStepReport {
    std::vector<std::uint32_t> selected;  // ascending, size K
    std::size_t k = 0;
    bool searched = false;
    AttentionOutput attention;
    std::optional<AttentionOutput> dense_reference;
    std::optional<double> recall;
    std::optional<double> l2_error;
    CostCounters counters;
};

class Session {
   public:
    Session(csattn_session h, SubspaceLayout layout, RetrievalConfig cfg)
        : cfg(std::move(cfg)), h_(h), layout_(std::move(layout)) {
        csattn_session_info info{};
        check(csattn_session_info_get(h_, &info));
        dim_ = info.dim;
        pushed_ = this->cfg;
        pushed_.k_bump = nullptr;
    }
    ~Session() {
        if (h_) csattn_session_destroy(h_);
    }
    Session(Session&& o) noexcept
        : cfg(std::move(o.cfg)), step(o.step), h2d_elem_bytes(o.h2d_elem_bytes), totals(o.totals),
          last_worst_(o.last_worst_), pushed_(std::move(o.pushed_)),
          h_(std::exchange(o.h_, nullptr)), layout_(std::move(o.layout_)),
          centroids_(std::move(o.centroids_)), dim_(o.dim_) {}
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    // Session is a value type in the reference: copy = fork the device tables.
    Session fork(std::size_t max_decode_steps) const {
        csattn_session out = nullptr;
        check(csattn_session_fork(h_, max_decode_steps, &out));
        Session s(out, layout_, cfg);
        s.step = step;
        s.totals = totals;
        s.last_worst_ = last_worst_;
        s.pushed_ = pushed_;
        return s;
    }

    // `cfg` is a public member (session.hpp:19-31): hand any change to the
    // device session before the next step
    void sync_config() {
        const RetrievalConfig& a = cfg;
        const RetrievalConfig& b = pushed_;
        if (a.keep_ratio == b.keep_ratio && a.search_period == b.search_period &&
            a.recent_window == b.recent_window && a.weights == b.weights &&
            a.backoff_tau == b.backoff_tau && a.backoff_threshold == b.backoff_threshold &&
            a.recent_passthrough == b.recent_passthrough)
            return;
        const csattn_retrieval_config rc = cfg.c();
        check(csattn_session_set_retrieval(h_, &rc));
        pushed_ = cfg;
        pushed_.k_bump = nullptr;
    }

    // decode_search's k_bump input (retrieval.cpp:257-263): the worst best
    // cosine of state.last_selection, i.e. of THIS query on a searching step
    // (!has_cache || step % period == 0, :237-238) and of the last search's
    // query otherwise
    double k_bump_cosine(std::span<const float> q) {
        const csattn_session_info in = info();
        const bool searching = in.steps == 0 || in.steps % std::max<std::size_t>(cfg.search_period, 1) == 0;
        if (searching) last_worst_ = worst_best_cosine(q);
        return last_worst_;
    }

    csattn_session handle() const { return h_; }
    const SubspaceLayout& layout() const { return layout_; }
    std::size_t dim() const { return dim_; }
    csattn_session_info info() const {
        csattn_session_info i{};
        check(csattn_session_info_get(h_, &i));
        return i;
    }
    std::size_t size() const { return info().context_len; }  // kv.size()

    // CsIndex image of the current device tables (index.hpp:46-68)
    CsIndex export_index() const {
        const csattn_session_info in = info();
        const std::size_t T = in.subspaces * in.centroids;
        const std::size_t stride = std::max<std::size_t>(in.list_capacity, 1);
        std::vector<uint32_t> lens(T), idx(T * stride);
        std::vector<float> sc(T * stride), cent(in.centroids * in.dim);
        check(csattn_session_export(h_, lens.data(), idx.data(), sc.data(), stride, cent.data()));
        CsIndex ix(layout_);
        ix.alpha = in.alpha;
        ix.list_capacity = static_cast<uint32_t>(in.list_capacity);
        ix.prefill_len = in.prefill_len;
        ix.normalize_keys = in.normalize_keys != 0;
        ix.score_bits = in.score_bits;
        for (std::size_t b = 0; b < layout_.count(); ++b) {
            CentroidSet cs;
            cs.subspace_id = b;
            cs.count = in.centroids;
            cs.dim = layout_.sizes[b];
            const float* src = cent.data() + in.centroids * layout_.offsets[b];
            cs.centroids.assign(src, src + cs.count * cs.dim);
            ix.centroid_sets.push_back(std::move(cs));
        }
        for (std::size_t t = 0; t < T; ++t) {
            TopList l;
            l.capacity = static_cast<uint32_t>(in.list_capacity);
            l.indices.assign(idx.begin() + t * stride, idx.begin() + t * stride + lens[t]);
            l.scores.assign(sc.begin() + t * stride, sc.begin() + t * stride + lens[t]);
            ix.tables.push_back(std::move(l));
        }
        return ix;
    }

    // CSAT v1 image of the current tables (serialize_index, index.cpp:289-318),
    // ordered and encoded on the device
    std::vector<std::uint8_t> serialize() const {
        uint64_t n = 0;
        check(csattn_session_serialize(h_, nullptr, 0, &n));
        std::vector<std::uint8_t> out(n);
        check(csattn_session_serialize(h_, out.data(), out.size(), &n));
        return out;
    }

    // KvStore rows [first, first + count) (core.hpp:47-68)
    void read_kv(std::size_t first, std::size_t count, std::vector<float>& keys,
                 std::vector<float>& values) const {
        keys.resize(count * dim_);
        values.resize(count * dim_);
        check(csattn_session_read_kv(h_, first, count, keys.data(), values.data()));
    }

    // select_centroids' worst best-cosine (retrieval.cpp:40-87) for k_bump:
    // fp64 dots of the normalised query slice with the unit centroids.
    double worst_best_cosine(std::span<const float> q) const {
        const std::vector<float>& cent = centroids();
        const std::size_t C = cent.size() / std::max<std::size_t>(dim_, 1);
        double worst = 1.0;
        for (std::size_t b = 0; b < layout_.count(); ++b) {
            const std::size_t off = layout_.offsets[b], w = layout_.sizes[b];
            double n2 = 0.0;
            for (std::size_t t = 0; t < w; ++t) n2 += static_cast<double>(q[off + t]) * q[off + t];
            if (n2 == 0.0) continue;  // zero slice: best cosine 1.0
            const double inv = 1.0 / std::sqrt(n2);
            std::vector<float> qn(w);
            for (std::size_t t = 0; t < w; ++t) qn[t] = static_cast<float>(q[off + t] * inv);
            double best = -std::numeric_limits<double>::infinity();
            for (std::size_t j = 0; j < C; ++j) {
                const float* c = cent.data() + C * off + j * w;
                double s = 0.0;
                for (std::size_t t = 0; t < w; ++t) s += static_cast<double>(qn[t]) * c[t];
                best = std::max(best, s);
            }
            worst = std::min(worst, best);
        }
        return worst;
    }

    RetrievalConfig cfg;
    std::size_t step = 0;
    std::size_t h2d_elem_bytes = 2;
    CostCounters totals;

   private:
    double last_worst_ = 1.0;  // worst best-cosine of the last search (k_bump)
    RetrievalConfig pushed_;   // the configuration the device session holds

    const std::vector<float>& centroids() const {  // immutable after the build
        if (centroids_.empty()) {
            const csattn_session_info in = info();
            centroids_.resize(in.centroids * in.dim);
            check(csattn_session_centroids(h_, centroids_.data()));
        }
        return centroids_;
    }

    csattn_session h_ = nullptr;
    SubspaceLayout layout_;
    mutable std::vector<float> centroids_;
    std::size_t dim_ = 0;
};

// metrics.cpp:9-30 / :40-46 (host cost models and the recall metric)
inline double recall_at_k(std::span<const std::uint32_t> selected, std::span<const std::uint32_t> truth) {
    if (truth.empty()) throw ParameterError("recall is undefined against an empty truth set");
    std::vector<std::uint32_t> a(selected.begin(), selected.end()), b(truth.begin(), truth.end());
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    std::size_t hits = 0, i = 0, j = 0;
    while (i < a.size() && j < b.size()) {
        if (a[i] < b[j]) ++i;
        else if (b[j] < a[i]) ++j;
        else {
            ++hits;
            ++i;
            ++j;
        }
    }
    return static_cast<double>(hits) / static_cast<double>(b.size());
}
inline std::size_t table_bytes(std::size_t m, std::size_t c, std::size_t l, std::size_t d,
                               std::size_t bytes_per_score) {
    if (m == 0 || c == 0 || d == 0 || bytes_per_score == 0) throw ParameterError("size model needs positive parameters");
    return m * c * l * (4 + bytes_per_score) + bytes_per_score * c * d;
}

// Session(KvStore, CsIndex, cfg) (session.hpp:19-31): a device session over a
// host index value and its prefill rows (csattn_session_import)
inline Session make_session(const KvStore& kv, const CsIndex& index, const RetrievalConfig& cfg,
                            std::size_t max_decode_steps = 4096, Context& ctx = Context::default_context()) {
    const std::size_t d = kv.dim(), m = index.subspaces(), c = index.centroids_per_subspace();
    if (index.layout.dim() != d) throw DimensionError("layout dimension does not match KV dimension");
    std::vector<float> cent;
    for (const CentroidSet& cs : index.centroid_sets) cent.insert(cent.end(), cs.centroids.begin(), cs.centroids.end());
    std::size_t stride = 1;
    for (const TopList& l : index.tables) stride = std::max(stride, l.indices.size());
    std::vector<uint32_t> lens(index.tables.size()), idx(index.tables.size() * stride, 0);
    std::vector<float> sc(index.tables.size() * stride, 0.0f);
    for (std::size_t t = 0; t < index.tables.size(); ++t) {
        const TopList& l = index.tables[t];
        lens[t] = static_cast<uint32_t>(l.indices.size());
        std::copy(l.indices.begin(), l.indices.end(), idx.begin() + static_cast<std::ptrdiff_t>(t * stride));
        std::copy(l.scores.begin(), l.scores.end(), sc.begin() + static_cast<std::ptrdiff_t>(t * stride));
    }
    std::vector<uint64_t> widths(index.layout.sizes.begin(), index.layout.sizes.end());
    const csattn_retrieval_config rc = cfg.c();
    csattn_session s = nullptr;
    check(csattn_session_import(ctx.handle(), cent.data(), c, lens.data(), idx.data(), sc.data(), stride,
                                index.list_capacity, index.alpha, index.normalize_keys ? 1 : 0, index.score_bits,
                                kv.key_data(), kv.value_data(), kv.size(), d, widths.data(), m, &rc, 1,
                                max_decode_steps, &s));
    return Session(s, index.layout, cfg);
}

// ---- index.hpp:98-121: the CSAT v1 image of a host CsIndex ----
struct IndexFootprint {
    std::size_t header_bytes = 0;
    std::size_t centroid_bytes = 0;
    std::size_t entry_bytes = 0;
    std::size_t payload() const { return centroid_bytes + entry_bytes; }
    std::size_t total() const { return header_bytes + payload(); }
};

namespace detail {
inline csattn_csat_header csat_header_of(const CsIndex& ix) {
    csattn_csat_header h{};
    h.m = ix.subspaces();
    h.centroids = ix.centroids_per_subspace();
    h.list_capacity = ix.list_capacity;
    h.dim = ix.layout.dim();
    h.prefill_len = ix.prefill_len;
    h.score_bits = ix.score_bits == 16 ? 16 : 32;
    h.normalize_keys = ix.normalize_keys ? 1 : 0;
    if (h.m > CSATTN_CSAT_MAX_SUBSPACES) throw ParameterError("too many subspaces for a CSAT image");
    for (std::size_t b = 0; b < h.m; ++b) h.widths[b] = ix.layout.sizes[b];
    return h;
}
struct FlatTables {
    std::vector<float> cent, sc;
    std::vector<std::uint32_t> lens, idx;
    std::size_t stride = 1;
};
inline FlatTables flatten(const CsIndex& ix) {
    FlatTables f;
    for (const TopList& l : ix.tables) f.stride = std::max(f.stride, l.indices.size());
    for (const CentroidSet& cs : ix.centroid_sets) f.cent.insert(f.cent.end(), cs.centroids.begin(), cs.centroids.end());
    f.lens.resize(ix.tables.size());
    f.idx.assign(ix.tables.size() * f.stride, 0);
    f.sc.assign(ix.tables.size() * f.stride, 0.0f);
    for (std::size_t t = 0; t < ix.tables.size(); ++t) {
        const TopList& l = ix.tables[t];
        f.lens[t] = static_cast<std::uint32_t>(l.indices.size());
        std::copy(l.indices.begin(), l.indices.end(), f.idx.begin() + t * f.stride);
        std::copy(l.scores.begin(), l.scores.end(), f.sc.begin() + t * f.stride);
    }
    return f;
}
}  // namespace detail

inline std::vector<std::uint8_t> serialize_index(const CsIndex& index) {
    const csattn_csat_header h = detail::csat_header_of(index);
    const detail::FlatTables f = detail::flatten(index);
    uint64_t n = 0;
    check(csattn_csat_encode(&h, f.cent.data(), f.lens.data(), f.idx.data(), f.sc.data(), f.stride, nullptr, 0, &n));
    std::vector<std::uint8_t> out(n);
    check(csattn_csat_encode(&h, f.cent.data(), f.lens.data(), f.idx.data(), f.sc.data(), f.stride, out.data(),
                             out.size(), &n));
    return out;
}

inline CsIndex deserialize_index(std::span<const std::uint8_t> bytes) {
    csattn_csat_header h{};
    check(csattn_csat_read_header(bytes.data(), bytes.size(), &h));
    const std::size_t T = h.m * h.centroids, L = h.list_capacity;
    std::vector<float> cent(h.centroids * h.dim), sc(T * L);
    std::vector<std::uint32_t> lens(T), idx(T * L);
    check(csattn_csat_decode(bytes.data(), bytes.size(), &h, cent.data(), lens.data(), idx.data(), sc.data(), L));
    CsIndex ix(SubspaceLayout(std::vector<std::size_t>(h.widths, h.widths + h.m)));
    ix.alpha = static_cast<double>(L) / static_cast<double>(h.prefill_len);
    ix.list_capacity = static_cast<std::uint32_t>(L);
    ix.prefill_len = h.prefill_len;
    ix.normalize_keys = h.normalize_keys != 0;
    ix.score_bits = h.score_bits;
    const float* src = cent.data();
    for (std::size_t b = 0; b < h.m; ++b) {
        CentroidSet cs;
        cs.subspace_id = b;
        cs.count = h.centroids;
        cs.dim = h.widths[b];
        cs.centroids.assign(src, src + cs.count * cs.dim);
        src += cs.count * cs.dim;
        ix.centroid_sets.push_back(std::move(cs));
    }
    for (std::size_t t = 0; t < T; ++t) {
        TopList l;
        l.capacity = static_cast<std::uint32_t>(L);
        l.indices.assign(idx.begin() + t * L, idx.begin() + t * L + lens[t]);
        l.scores.assign(sc.begin() + t * L, sc.begin() + t * L + lens[t]);
        ix.tables.push_back(std::move(l));
    }
    return ix;
}

inline void save_index(const CsIndex& index, const std::string& path) {
    const auto bytes = serialize_index(index);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw DataError("cannot open for writing: " + path);
    out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw DataError("short write to " + path);
}

inline CsIndex load_index(const std::string& path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw DataError("cannot open: " + path);
    const std::streamsize size = in.tellg();
    in.seekg(0);
    std::vector<std::uint8_t> bytes(static_cast<std::size_t>(size));
    in.read(reinterpret_cast<char*>(bytes.data()), size);
    if (!in) throw DataError("short read from " + path);
    return deserialize_index(bytes);
}

inline IndexFootprint index_footprint(const CsIndex& index) {
    const csattn_csat_header h = detail::csat_header_of(index);
    std::vector<std::uint32_t> lens(index.tables.size());
    for (std::size_t t = 0; t < lens.size(); ++t) lens[t] = static_cast<std::uint32_t>(index.tables[t].indices.size());
    uint64_t a = 0, b = 0, c = 0;
    check(csattn_csat_footprint(&h, lens.data(), &a, &b, &c));
    return IndexFootprint{a, b, c};
}

// A device session from a CSAT image and the prefill rows it indexes
// (load_index + KvStore + Session, session.hpp:19-31).
inline Session load_session(std::span<const std::uint8_t> bytes, std::span<const float> keys,
                            std::span<const float> values, const RetrievalConfig& cfg,
                            std::size_t max_decode_steps = 4096, std::size_t group = 1,
                            Context& ctx = Context::default_context()) {
    csattn_csat_header h{};
    check(csattn_csat_read_header(bytes.data(), bytes.size(), &h));
    SubspaceLayout layout(std::vector<std::size_t>(h.widths, h.widths + h.m));
    const csattn_retrieval_config rc = cfg.c();
    csattn_session s = nullptr;
    check(csattn_session_deserialize(ctx.handle(), bytes.data(), bytes.size(), keys.data(), values.data(),
                                     keys.size() / std::max<std::size_t>(h.dim, 1), &rc, group,
                                     max_decode_steps, &s));
    return Session(s, layout, cfg);
}

// ---- session.hpp:44-66 ----
// prefill (session.cpp:25-44): KvStore + build_index on the GPU. `group`
// query heads may share the index (GQA): queries then hold their pooled rows.
inline Session prefill(std::span<const float> queries, std::span<const float> keys,
                       std::span<const float> values, const SubspaceLayout& layout,
                       const IndexConfig& index_cfg, const RetrievalConfig& cfg,
                       std::size_t max_decode_steps = 4096, std::size_t group = 1,
                       Context& ctx = Context::default_context()) {
    const std::size_t d = layout.dim();
    if (queries.size() % d != 0 || keys.size() % d != 0 || values.size() % d != 0)
        throw DimensionError("prefill rows are not a multiple of d");
    if (queries.size() / d == 0) throw ParameterError("prefill must be non-empty");
    if (keys.size() * group != queries.size() || values.size() != keys.size())
        throw ParameterError("prefill query/key/value counts must be equal");
    const std::size_t p = keys.size() / d;
    std::vector<uint64_t> widths(layout.sizes.begin(), layout.sizes.end());
    const csattn_index_config ic = index_cfg.c();
    const csattn_retrieval_config rc = cfg.c();
    csattn_session s = nullptr;
    check(csattn_prefill(ctx.handle(), queries.data(), queries.size() / d, keys.data(), values.data(),
                         p, d, widths.data(), widths.size(), &ic, &rc, group, max_decode_steps,
                         CSATTN_HOST_BUFFERS, &s));
    return Session(s, layout, cfg);
}

// decode_step (session.cpp:46-99) for a single-head session.
inline DecodeStepReport decode_step(Session& session, std::span<const float> q,
                                    std::span<const float> new_key,
                                    std::span<const float> new_value, bool compare_dense) {
    const std::size_t d = session.dim();
    if (q.size() != d || new_key.size() != d || new_value.size() != d)
        throw DimensionError("decode step inputs must have width d");
    if (session.info().group != 1)
        throw ParameterError("decode_step takes one query: this session serves a GQA group of " +
                             std::to_string(session.info().group) + " heads (use csattn_decode_step)");
    session.sync_config();
    const std::size_t n = session.size();
    uint64_t k_override = 0;
    if (session.cfg.k_bump)
        k_override = session.cfg.k_bump(keep_count(session.cfg.keep_ratio, n), session.k_bump_cosine(q));
    DecodeStepReport r;
    std::vector<uint32_t> sel(n);
    std::vector<float> out(d), w(n);
    csattn_step_report rep{};
    std::optional<AttentionOutput> dense;
    std::vector<uint32_t> truth;
    if (compare_dense) {  // the dense oracle sees the same pre-append context
        AttentionOutput full;
        full.output.resize(d);
        full.weights.resize(n);
        check(csattn_dense_attention(session.handle(), q.data(), nullptr, 0, full.output.data(),
                                     full.weights.data(), CSATTN_HOST_BUFFERS));
        dense = std::move(full);
        // dense_topk (core.cpp:171-192) at this step's K, on the device
        const std::size_t kk = k_override ? std::min<std::size_t>(k_override, n)
                                          : keep_count(session.cfg.keep_ratio, n);
        truth.resize(kk);
        check(csattn_dense_topk(session.handle(), q.data(), kk, truth.data(), CSATTN_HOST_BUFFERS));
    }
    check(csattn_decode_step(session.handle(), q.data(), new_key.data(), new_value.data(),
                             out.data(), sel.data(), w.data(), n, &rep,
                             k_override ? &k_override : nullptr, CSATTN_HOST_BUFFERS));
    r.k = rep.k;
    r.searched = rep.searched != 0;
    r.selected.assign(sel.begin(), sel.begin() + rep.k);
    r.attention.output = std::move(out);
    r.attention.weights.assign(w.begin(), w.begin() + rep.k);
    r.counters.centroid_dot_ops = rep.centroid_dot_ops;
    r.counters.gathered_entries = rep.gathered_entries;
    r.counters.reduce_ops = rep.reduce_ops;
    r.counters.attention_key_ops = rep.attention_key_ops;
    r.counters.h2d_bytes_model =
        h2d_bytes(session.cfg.keep_ratio, n, d, session.h2d_elem_bytes, session.cfg.search_period);
    r.counters.searches = rep.searches;
    r.counters.inserts_attempted = rep.inserts_attempted;
    r.counters.inserts_applied = rep.inserts_applied;
    r.counters.insert_dot_ops = rep.insert_dot_ops;
    if (dense) {
        // recall_at_k (metrics.cpp:9-30) against the dense top-K
        std::size_t hit = 0;
        for (uint32_t x : r.selected) hit += std::binary_search(truth.begin(), truth.end(), x) ? 1 : 0;
        r.recall = truth.empty() ? 1.0 : static_cast<double>(hit) / static_cast<double>(truth.size());
        double e2 = 0.0;
        for (std::size_t t = 0; t < d; ++t) {
            const double x = static_cast<double>(r.attention.output[t]) - dense->output[t];
            e2 += x * x;
        }
        r.l2_error = std::sqrt(e2);
        r.dense_reference = std::move(dense);
    }
    session.step += 1;
    session.totals.add(r.counters);
    return r;
}

// run_decode (session.cpp:101-126): validates stream lengths up front.
inline std::vector<DecodeStepReport> run_decode(Session& session, std::span<const float> queries,
                                                std::span<const float> keys,
                                                std::span<const float> values, std::size_t steps,
                                                bool compare_dense) {
    const std::size_t d = session.dim();
    if (queries.size() % d != 0 || keys.size() % d != 0 || values.size() % d != 0)
        throw DimensionError("decode rows are not a multiple of d");
    const std::size_t available = std::min({queries.size() / d, keys.size() / d, values.size() / d});
    if (available < steps)
        throw StreamExhaustedError("decode streams run out at step " + std::to_string(available) +
                                   " of " + std::to_string(steps));
    std::vector<DecodeStepReport> out;
    out.reserve(steps);
    for (std::size_t t = 0; t < steps; ++t)
        out.push_back(decode_step(session, queries.subspan(t * d, d), keys.subspan(t * d, d),
                                  values.subspan(t * d, d), compare_dense));
    return out;
}

// run_decode as ONE CUDA graph (csattn_decode_run): the same
// steps, the same selected sets and outputs, without per-step reports. The
// session's step count advances; its totals are not accumulated (no counters
// are read back).
struct GraphRun {
    std::vector<std::vector<std::uint32_t>> selected;  // per step, ascending
    std::vector<float> outputs;                         // steps x d
};

inline GraphRun run_decode_graph(Session& session, std::span<const float> queries,
                                 std::span<const float> keys, std::span<const float> values,
                                 std::size_t steps,
                                 Context& ctx = Context::default_context()) {
    const std::size_t d = session.dim();
    if (queries.size() % d != 0 || keys.size() % d != 0 || values.size() % d != 0)
        throw DimensionError("decode rows are not a multiple of d");
    const std::size_t available = std::min({queries.size() / d, keys.size() / d, values.size() / d});
    if (available < steps)
        throw StreamExhaustedError("decode streams run out at step " + std::to_string(available) +
                                   " of " + std::to_string(steps));
    if (session.info().group != 1)
        throw ParameterError("run_decode_graph takes one query per step: this session serves a GQA group");
    if (session.cfg.k_bump)
        throw ParameterError("run_decode_graph has no per-step k_bump hook: use run_decode");
    session.sync_config();
    GraphRun r;
    if (steps == 0) return r;
    const std::size_t n0 = session.size();
    const std::size_t stride = n0 + steps;
    r.outputs.assign(steps * d, 0.0f);
    std::vector<std::uint32_t> sel(steps * stride);
    csattn_session h = session.handle();
    check(csattn_decode_run(ctx.handle(), 1, &h, steps, queries.data(), keys.data(),
                            values.data(), r.outputs.data(), sel.data(), stride, nullptr,
                            CSATTN_HOST_BUFFERS));
    for (std::size_t t = 0; t < steps; ++t) {
        const std::size_t k = keep_count(session.cfg.keep_ratio, n0 + t);
        r.selected.emplace_back(sel.begin() + t * stride, sel.begin() + t * stride + k);
    }
    session.step += steps;
    return r;
}

}  // namespace csattn_b200
