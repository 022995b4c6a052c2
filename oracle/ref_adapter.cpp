// oracle/ref_adapter.cpp — TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled from
// /root/reference/proj/src/*.cpp with -Dcsattn=csattn_ref (oracle/Makefile) into
// oracle/_ref/libcsattn_ref.so. It lets the pytest suite and bench.py's
// cpu_baseline / --impl reference legs drive the reference's own public API
// (session.hpp:46-66, index.hpp:86-96, synthetic.hpp:38-41) on identical inputs.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load it.
//
// GQA composition: one KV head = one reference Session whose
// index is built over the pooled queries of its `group` query heads; each query
// head keeps its own SearchState and runs decode_search + masked
// dense_attention; the KV head then appends once and streaming_inserts once —
// exactly decode_step (session.cpp:46-99) with the search/attention part
// repeated per query head. For group == 1 the real decode_step is called.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "csattn/core.hpp"
#include "csattn/index.hpp"
#include "csattn/metrics.hpp"
#include "csattn/retrieval.hpp"
#include "csattn/session.hpp"
#include "csattn/synthetic.hpp"
#include "csattn/util.hpp"
#include "csattn_b200.h"

namespace R = csattn_ref;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
    if (dynamic_cast<const R::StreamExhaustedError*>(&e)) return CSATTN_ERR_STREAM_EXHAUSTED;
    if (dynamic_cast<const R::PropertyError*>(&e)) return CSATTN_ERR_PROPERTY;
    if (dynamic_cast<const R::CorruptError*>(&e)) return CSATTN_ERR_CORRUPT;
    if (dynamic_cast<const R::TruncatedError*>(&e)) return CSATTN_ERR_TRUNCATED;
    if (dynamic_cast<const R::VersionError*>(&e)) return CSATTN_ERR_VERSION;
    if (dynamic_cast<const R::BadMagicError*>(&e)) return CSATTN_ERR_BAD_MAGIC;
    if (dynamic_cast<const R::DataError*>(&e)) return CSATTN_ERR_DATA;
    if (dynamic_cast<const R::ParameterError*>(&e)) return CSATTN_ERR_PARAMETER;
    if (dynamic_cast<const R::DimensionError*>(&e)) return CSATTN_ERR_DIMENSION;
    if (dynamic_cast<const R::Error*>(&e)) return CSATTN_ERR_GENERIC;
    return CSATTN_ERR_GENERIC;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return CSATTN_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return status_of(e);
    }
}

R::SubspaceLayout layout_of(const uint64_t* widths, uint64_t m) {
    std::vector<std::size_t> w(widths, widths + m);
    return R::SubspaceLayout(std::move(w));
}

R::IndexConfig icfg_of(const csattn_index_config* c) {
    R::IndexConfig k;
    k.alpha = c->alpha;
    k.list_capacity = c->list_capacity;
    k.normalize_keys = c->normalize_keys != 0;
    k.score_bits = c->score_bits;
    k.cluster.centroids = c->centroids;
    k.cluster.iterations = c->iterations;
    k.cluster.batch_size = c->batch_size;
    k.cluster.seed = c->seed;
    k.cluster.tolerance = c->tolerance;
    return k;
}

R::RetrievalConfig rcfg_of(const csattn_retrieval_config* c) {
    R::RetrievalConfig r;
    r.keep_ratio = c->keep_ratio;
    r.search_period = c->search_period;
    r.recent_window = c->recent_window;
    if (c->weights && c->n_weights) r.weights.assign(c->weights, c->weights + c->n_weights);
    r.backoff_tau = c->backoff_tau;
    r.backoff_threshold = c->backoff_threshold;
    r.recent_passthrough = c->recent_passthrough != 0;
    return r;
}

struct Group {
    R::Session session;
    std::vector<R::SearchState> states;  // one per query head (group > 1)
    uint64_t group;
    Group(R::Session s, uint64_t g) : session(std::move(s)), group(g) {
        if (g > 1) states.resize(g);
    }
};

void fill_report(csattn_step_report* rep, const R::DecodeStepReport& r, double worst) {
    std::memset(rep, 0, sizeof(*rep));
    rep->k = r.k;
    rep->searched = r.searched ? 1 : 0;
    rep->centroid_dot_ops = r.counters.centroid_dot_ops;
    rep->gathered_entries = r.counters.gathered_entries;
    rep->reduce_ops = r.counters.reduce_ops;
    rep->attention_key_ops = r.counters.attention_key_ops;
    rep->h2d_bytes_model = r.counters.h2d_bytes_model;
    rep->searches = r.counters.searches;
    rep->inserts_attempted = r.counters.inserts_attempted;
    rep->inserts_applied = r.counters.inserts_applied;
    rep->insert_dot_ops = r.counters.insert_dot_ops;
    rep->worst_best_cosine = worst;
}

double worst_of(const R::SearchState& st) {
    double w = 1.0;
    for (double c : st.last_selection.best_cosine) w = std::min(w, c);
    return w;
}

// One step of one KV head for all its query heads; mirrors session.cpp:46-99.
void group_step(Group& g, const float* q, const float* key, const float* value,
                uint32_t* selected, uint64_t sel_stride, float* out, float* weights,
                csattn_step_report* reps, const uint64_t* k_override) {
    R::Session& s = g.session;
    const std::size_t d = s.kv.dim();
    if (g.group == 1 && !(k_override && k_override[0])) {
        R::DecodeStepReport r = R::decode_step(s, {q, d}, {key, d}, {value, d}, false);
        if (selected) std::copy(r.selected.begin(), r.selected.end(), selected);
        if (weights)
            std::copy(r.attention.weights.begin(), r.attention.weights.end(), weights);
        if (out) std::copy(r.attention.output.begin(), r.attention.output.end(), out);
        if (reps) fill_report(reps, r, worst_of(s.search_state));
        return;
    }
    const std::size_t n = s.kv.size();
    std::vector<R::DecodeStepReport> rs(g.group);
    for (uint64_t h = 0; h < g.group; ++h) {
        R::SearchState& st = g.group == 1 ? s.search_state : g.states[h];
        R::RetrievalConfig cfg = s.cfg;
        if (k_override && k_override[h]) {
            const std::size_t ko = k_override[h];
            cfg.k_bump = [ko](std::size_t, double) { return ko; };
        }
        R::SearchResult sr = R::decode_search({q + h * d, d}, s.index, s.kv, cfg, st);
        R::DecodeStepReport& r = rs[h];
        r.selected = std::move(sr.selected);
        r.k = sr.k;
        r.searched = sr.searched;
        r.attention = R::dense_attention({q + h * d, d}, s.kv, r.selected);
        r.counters.centroid_dot_ops = sr.centroid_dot_ops;
        r.counters.gathered_entries = sr.gathered_entries;
        r.counters.reduce_ops = sr.reduce_ops;
        r.counters.attention_key_ops = r.k * d;
        r.counters.h2d_bytes_model =
            R::h2d_bytes(s.cfg.keep_ratio, n, d, s.h2d_elem_bytes, s.cfg.search_period);
        r.counters.searches = sr.searched ? 1 : 0;
        if (selected) std::copy(r.selected.begin(), r.selected.end(), selected + h * sel_stride);
        if (weights)
            std::copy(r.attention.weights.begin(), r.attention.weights.end(),
                      weights + h * sel_stride);
        if (out) std::copy(r.attention.output.begin(), r.attention.output.end(), out + h * d);
    }
    s.kv.append({key, d}, {value, d});
    const R::InsertReport ir = R::streaming_insert({key, d}, static_cast<uint32_t>(n), s.index);
    s.step += 1;
    for (uint64_t h = 0; h < g.group; ++h) {
        rs[h].counters.inserts_attempted = ir.attempted;
        rs[h].counters.inserts_applied = ir.applied;
        rs[h].counters.insert_dot_ops = ir.dot_ops;
        if (reps)
            fill_report(reps + h, rs[h], worst_of(g.group == 1 ? s.search_state : g.states[h]));
    }
}

}  // namespace

extern "C" {

const char* csref_last_error(void) { return g_err.c_str(); }

int csref_make_synthetic(const csattn_synthetic_spec* spec, float* q, float* k, float* v) {
    return guarded([&] {
        R::SyntheticSpec s;
        s.rows = spec->rows;
        s.dim = spec->dim;
        s.clusters = spec->clusters;
        s.seed = spec->seed;
        s.plant_fraction = spec->plant_fraction;
        s.plant_scale = spec->plant_scale;
        s.query_noise = spec->query_noise;
        s.dwell = spec->dwell;
        const R::SyntheticWorkload w = R::make_synthetic(s);
        std::copy(w.queries.begin(), w.queries.end(), q);
        std::copy(w.keys.begin(), w.keys.end(), k);
        std::copy(w.values.begin(), w.values.end(), v);
    });
}

uint64_t csref_mix_seed(uint64_t seed, uint64_t salt) { return R::mix_seed(seed, salt); }
uint64_t csref_ceil_ratio(double r, uint64_t n) { return R::ceil_ratio(r, n); }

// prefill (session.cpp:25-44) with n_queries possibly != p (GQA pooling goes
// through build_index directly, index.cpp:145-177).
int csref_prefill(const float* q, uint64_t nq, const float* k, const float* v, uint64_t p,
                  uint64_t d, const uint64_t* widths, uint64_t m,
                  const csattn_index_config* icfg, const csattn_retrieval_config* rcfg,
                  uint64_t group, void** out) {
    return guarded([&] {
        const R::SubspaceLayout layout = layout_of(widths, m);
        const R::IndexConfig ic = icfg_of(icfg);
        const R::RetrievalConfig rc = rcfg_of(rcfg);
        if (nq == p) {
            R::Session s = R::prefill({q, nq * d}, {k, p * d}, {v, p * d}, layout, ic, rc);
            *out = new Group(std::move(s), group);
        } else {
            R::KvStore kv(d, {k, p * d}, {v, p * d});
            R::CsIndex idx = R::build_index({q, nq * d}, nq, kv, layout, ic);
            R::Session s(std::move(kv), std::move(idx), rc);
            s.seed = ic.cluster.seed;
            *out = new Group(std::move(s), group);
        }
    });
}

// build_index_from_centroids (index.cpp:179-202); centroids packed per subspace.
int csref_prefill_from_centroids(const float* cent, uint64_t c, const float* k, const float* v,
                                 uint64_t p, uint64_t d, const uint64_t* widths, uint64_t m,
                                 const csattn_index_config* icfg,
                                 const csattn_retrieval_config* rcfg, uint64_t group,
                                 void** out) {
    return guarded([&] {
        const R::SubspaceLayout layout = layout_of(widths, m);
        std::vector<R::CentroidSet> sets(m);
        const float* src = cent;
        for (uint64_t b = 0; b < m; ++b) {
            sets[b].subspace_id = b;
            sets[b].count = c;
            sets[b].dim = widths[b];
            sets[b].centroids.assign(src, src + c * widths[b]);
            src += c * widths[b];
        }
        R::KvStore kv(d, {k, p * d}, {v, p * d});
        R::CsIndex idx =
            R::build_index_from_centroids(std::move(sets), kv, layout, icfg_of(icfg));
        R::Session s(std::move(kv), std::move(idx), rcfg_of(rcfg));
        *out = new Group(std::move(s), group);
    });
}

// A reference Session over a given CsIndex image (TopList order) — used by
// bench.py's cpu_baseline leg to run the reference's decode path on exactly
// the tables the GPU built (tests pin them bit-identical to build_index).
int csref_import(const float* cent, uint64_t c, const uint32_t* lens, const uint32_t* idx,
                 const float* scores, uint64_t stride, uint64_t L, double alpha,
                 int32_t normalize_keys, const float* k, const float* v, uint64_t p, uint64_t d,
                 const uint64_t* widths, uint64_t m, const csattn_retrieval_config* rcfg,
                 uint64_t group, void** out) {
    return guarded([&] {
        R::CsIndex ix(layout_of(widths, m));
        const float* src = cent;
        for (uint64_t b = 0; b < m; ++b) {
            R::CentroidSet cs;
            cs.subspace_id = b;
            cs.count = c;
            cs.dim = widths[b];
            cs.centroids.assign(src, src + c * widths[b]);
            src += c * widths[b];
            ix.centroid_sets.push_back(std::move(cs));
        }
        for (uint64_t t = 0; t < m * c; ++t) {
            R::TopList tl;
            tl.capacity = static_cast<uint32_t>(L);
            tl.indices.assign(idx + t * stride, idx + t * stride + lens[t]);
            tl.scores.assign(scores + t * stride, scores + t * stride + lens[t]);
            ix.tables.push_back(std::move(tl));
        }
        ix.alpha = alpha;
        ix.list_capacity = static_cast<uint32_t>(L);
        ix.prefill_len = p;
        ix.normalize_keys = normalize_keys != 0;
        ix.score_bits = 32;
        R::KvStore kv(d, {k, p * d}, {v, p * d});
        R::Session s(std::move(kv), std::move(ix), rcfg_of(rcfg));
        *out = new Group(std::move(s), group);
    });
}

void csref_free(void* h) { delete static_cast<Group*>(h); }

// Session::cfg is a public member (session.hpp:19-31): change it between steps.
int csref_set_retrieval(void* h, const csattn_retrieval_config* rc) {
    return guarded([&] { static_cast<Group*>(h)->session.cfg = rcfg_of(rc); });
}

// A copy of a session (Session is a value type, session.hpp:19-31): KvStore,
// CsIndex and every query head's SearchState — one more independent sequence
// over the same prefill (the batch-decode sequences of config c3).
int csref_fork(void* h, void** out) {
    return guarded([&] { *out = new Group(*static_cast<Group*>(h)); });
}

int csref_info(void* h, uint64_t* n, uint64_t* l, uint64_t* c, uint64_t* m) {
    return guarded([&] {
        const Group* g = static_cast<Group*>(h);
        *n = g->session.kv.size();
        *l = g->session.index.list_capacity;
        *c = g->session.index.centroids_per_subspace();
        *m = g->session.index.subspaces();
    });
}

int csref_export(void* h, uint32_t* lens, uint32_t* idx, float* scores, uint64_t stride,
                 float* centroids) {
    return guarded([&] {
        const R::CsIndex& ix = static_cast<Group*>(h)->session.index;
        for (std::size_t t = 0; t < ix.tables.size(); ++t) {
            const R::TopList& tl = ix.tables[t];
            if (tl.indices.size() > stride) throw R::ParameterError("export stride too small");
            lens[t] = static_cast<uint32_t>(tl.indices.size());
            std::copy(tl.indices.begin(), tl.indices.end(), idx + t * stride);
            std::copy(tl.scores.begin(), tl.scores.end(), scores + t * stride);
        }
        if (centroids) {
            float* dst = centroids;
            for (const R::CentroidSet& cs : ix.centroid_sets) {
                std::copy(cs.centroids.begin(), cs.centroids.end(), dst);
                dst += cs.centroids.size();
            }
        }
    });
}

// One decode step of a KV head for its `group` query heads.
int csref_step(void* h, const float* q, const float* key, const float* value,
               uint32_t* selected, uint64_t sel_stride, float* out, float* weights,
               csattn_step_report* reps, const uint64_t* k_override) {
    return guarded([&] {
        group_step(*static_cast<Group*>(h), q, key, value, selected, sel_stride, out, weights,
                   reps, k_override);
    });
}

// SearchState::cached of query head `head` (the last reduce_by_key result).
int csref_candidates(void* h, uint64_t head, uint32_t* idx, double* scores, uint64_t cap,
                     uint64_t* n) {
    return guarded([&] {
        Group& g = *static_cast<Group*>(h);
        const R::SearchState& st = g.group == 1 ? g.session.search_state : g.states.at(head);
        const R::CandidateSet& c = st.cached;
        if (c.size() > cap) throw R::ParameterError("candidate buffer too small");
        std::copy(c.indices.begin(), c.indices.end(), idx);
        std::copy(c.scores.begin(), c.scores.end(), scores);
        *n = c.size();
    });
}

// decode_step with compare_dense = true (session.cpp:66-78): recall + l2 error.
int csref_step_compare(void* h, const float* q, const float* key, const float* value,
                       uint32_t* selected, float* out, float* dense_out, double* recall,
                       double* l2_error) {
    return guarded([&] {
        R::Session& s = static_cast<Group*>(h)->session;
        const std::size_t d = s.kv.dim();
        R::DecodeStepReport r = R::decode_step(s, {q, d}, {key, d}, {value, d}, true);
        if (selected) std::copy(r.selected.begin(), r.selected.end(), selected);
        if (out) std::copy(r.attention.output.begin(), r.attention.output.end(), out);
        if (dense_out)
            std::copy(r.dense_reference->output.begin(), r.dense_reference->output.end(),
                      dense_out);
        *recall = *r.recall;
        *l2_error = *r.l2_error;
    });
}

// Wall-clock timing of `steps` decode steps over `n` independent KV heads on
// `threads` host threads (SPEC.md:452 allows concurrent heads). Inputs per head
// h and step t: q at q + (h*steps + t)*group*d, key/value at (h*steps + t)*d.
// Returns seconds for the whole run (every head completing every step).
int csref_bench(void** hs, uint64_t n, const float* q, const float* k, const float* v,
                uint64_t steps, uint64_t threads, double* seconds) {
    return guarded([&] {
        if (threads == 0) threads = 1;
        std::vector<Group*> gs(n);
        for (uint64_t i = 0; i < n; ++i) gs[i] = static_cast<Group*>(hs[i]);
        const std::size_t d = gs[0]->session.kv.dim();
        std::atomic<uint64_t> next{0};
        std::vector<std::string> errs(threads);
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (uint64_t w = 0; w < threads; ++w) {
            pool.emplace_back([&, w] {
                try {
                    for (;;) {
                        const uint64_t i = next.fetch_add(1);
                        if (i >= n) break;
                        Group& g = *gs[i];
                        for (uint64_t t = 0; t < steps; ++t)
                            group_step(g, q + (i * steps + t) * g.group * d,
                                       k + (i * steps + t) * d, v + (i * steps + t) * d,
                                       nullptr, 0, nullptr, nullptr, nullptr, nullptr);
                    }
                } catch (const std::exception& e) {
                    errs[w] = e.what();
                }
            });
        }
        for (auto& t : pool) t.join();
        const auto t1 = std::chrono::steady_clock::now();
        for (const auto& e : errs)
            if (!e.empty()) throw R::Error(e);
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// Dense oracle helpers (core.cpp:118-192) on an arbitrary store.
// ---- CSAT v1 (serialize_index / deserialize_index, index.cpp:289-396) ----

uint16_t csref_f32_to_f16(float x) { return R::f32_to_f16(x); }
float csref_f16_to_f32(uint16_t h) { return R::f16_to_f32(h); }

namespace {
R::CsIndex index_of(const float* cent, uint64_t c, const uint32_t* lens, const uint32_t* idx,
                    const float* scores, uint64_t stride, uint64_t L, uint64_t prefill,
                    int32_t normalize_keys, int32_t score_bits, const uint64_t* widths, uint64_t m) {
    R::CsIndex ix(layout_of(widths, m));
    const float* src = cent;
    for (uint64_t b = 0; b < m; ++b) {
        R::CentroidSet cs;
        cs.subspace_id = b;
        cs.count = c;
        cs.dim = widths[b];
        cs.centroids.assign(src, src + c * widths[b]);
        src += c * widths[b];
        ix.centroid_sets.push_back(std::move(cs));
    }
    for (uint64_t t = 0; t < m * c; ++t) {
        R::TopList tl;
        tl.capacity = static_cast<uint32_t>(L);
        tl.indices.assign(idx + t * stride, idx + t * stride + lens[t]);
        tl.scores.assign(scores + t * stride, scores + t * stride + lens[t]);
        ix.tables.push_back(std::move(tl));
    }
    ix.alpha = static_cast<double>(L) / static_cast<double>(prefill);
    ix.list_capacity = static_cast<uint32_t>(L);
    ix.prefill_len = prefill;
    ix.normalize_keys = normalize_keys != 0;
    ix.score_bits = score_bits;
    return ix;
}
int copy_bytes(const std::vector<std::uint8_t>& b, uint8_t* out, uint64_t cap, uint64_t* size) {
    *size = b.size();
    if (out) {
        if (cap < b.size()) return CSATTN_ERR_PARAMETER;
        std::memcpy(out, b.data(), b.size());
    }
    return CSATTN_OK;
}
}  // namespace

// serialize_index of a host index given as arrays (TopList order)
int csref_encode(const float* cent, uint64_t c, const uint32_t* lens, const uint32_t* idx,
                 const float* scores, uint64_t stride, uint64_t L, uint64_t prefill,
                 int32_t normalize_keys, int32_t score_bits, const uint64_t* widths, uint64_t m,
                 uint8_t* out, uint64_t cap, uint64_t* size) {
    int st = CSATTN_OK;
    const int g = guarded([&] {
        const auto b = R::serialize_index(index_of(cent, c, lens, idx, scores, stride, L, prefill,
                                                   normalize_keys, score_bits, widths, m));
        st = copy_bytes(b, out, cap, size);
    });
    return g != CSATTN_OK ? g : st;
}

// serialize_index of a reference session's current index
int csref_serialize(void* h, int32_t score_bits, uint8_t* out, uint64_t cap, uint64_t* size) {
    int st = CSATTN_OK;
    const int g = guarded([&] {
        R::CsIndex& ix = static_cast<Group*>(h)->session.index;
        const int keep = ix.score_bits;
        ix.score_bits = score_bits;
        const auto b = R::serialize_index(ix);
        ix.score_bits = keep;
        st = copy_bytes(b, out, cap, size);
    });
    return g != CSATTN_OK ? g : st;
}

// deserialize_index -> status (+ csref_last_error) and the re-serialized image
int csref_roundtrip(const uint8_t* bytes, uint64_t n, uint8_t* out, uint64_t cap, uint64_t* size) {
    int st = CSATTN_OK;
    const int g = guarded([&] {
        const R::CsIndex ix = R::deserialize_index({bytes, n});
        st = copy_bytes(R::serialize_index(ix), out, cap, size);
    });
    return g != CSATTN_OK ? g : st;
}

// index_footprint of a deserialized image
int csref_footprint(const uint8_t* bytes, uint64_t n, uint64_t* header, uint64_t* centroid,
                    uint64_t* entry) {
    return guarded([&] {
        const auto fp = R::index_footprint(R::deserialize_index({bytes, n}));
        *header = fp.header_bytes;
        *centroid = fp.centroid_bytes;
        *entry = fp.entry_bytes;
    });
}

// load_index + KvStore + Session over the image's prefill rows
int csref_load(const uint8_t* bytes, uint64_t n, const float* k, const float* v, uint64_t d,
               const csattn_retrieval_config* rcfg, uint64_t group, void** out) {
    return guarded([&] {
        R::CsIndex ix = R::deserialize_index({bytes, n});
        const uint64_t p = ix.prefill_len;
        R::KvStore kv(d, {k, p * d}, {v, p * d});
        R::Session s(std::move(kv), std::move(ix), rcfg_of(rcfg));
        *out = new Group(std::move(s), group);
    });
}

int csref_dense_attention(const float* q, const float* keys, const float* values, uint64_t n,
                          uint64_t d, const uint32_t* mask, uint64_t n_mask, float* out,
                          float* weights) {
    return guarded([&] {
        R::KvStore kv(d, {keys, n * d}, {values, n * d});
        R::AttentionOutput o =
            mask ? R::dense_attention({q, d}, kv, std::span<const uint32_t>(mask, n_mask))
                 : R::dense_attention({q, d}, kv);
        std::copy(o.output.begin(), o.output.end(), out);
        if (weights) std::copy(o.weights.begin(), o.weights.end(), weights);
    });
}

int csref_dense_topk(const float* q, const float* keys, uint64_t n, uint64_t d, uint64_t k,
                     uint32_t* out) {
    return guarded([&] {
        std::vector<float> vals(n * d, 0.0f);
        R::KvStore kv(d, {keys, n * d}, {vals.data(), n * d});
        const auto t = R::dense_topk({q, d}, kv, k);
        std::copy(t.begin(), t.end(), out);
    });
}

}  // extern "C"
