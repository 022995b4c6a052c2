// test_fn.cpp — the reference's function-level tests (test_index.cpp:60-300,
// test_retrieval.cpp:134-577) ported onto the B200 facade's free functions
// (include/csattn_b200.hpp: TopList / score_keys / build_index /
// build_index_from_centroids / select_centroids / gather_lists /
// reduce_by_key / select_topk / decode_search / streaming_insert /
// dense_topk, each computing on the GPU). Every case keeps the reference
// test's assertions and, where the reference library can run the same call,
// also checks the facade's result against it exactly (csattn_ref from
// oracle/_ref). TEST INFRASTRUCTURE, built by tests/cpp/Makefile, run on a
// B200 by tests/test_cpp_facade.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "csattn/index.hpp"  // reference (compiled with -Dcsattn=csattn_ref)
#include "csattn/retrieval.hpp"
#include "csattn/util.hpp"
#include "csattn_b200.hpp"  // B200 facade

namespace R = csattn_ref;
namespace B = csattn_b200;

static int failures = 0, checks = 0;
#define CHECK(cond, ...)                                     \
    do {                                                     \
        ++checks;                                            \
        if (!(cond)) {                                       \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                        \
            std::printf("\n");                               \
            ++failures;                                      \
        }                                                    \
    } while (0)
#define CASE(name) std::printf("case: %s\n", name)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static bool approx(double a, double b, double eps = 1e-6) {
    return std::fabs(a - b) <= eps * std::max(1.0, std::max(std::fabs(a), std::fabs(b)));
}

// ---- the reference tests' input helpers (same Rng draws) ----
static std::vector<float> random_rows(std::size_t n, std::size_t d, std::uint64_t seed) {
    R::Rng rng(seed);
    std::vector<float> v(n * d);
    for (float& x : v) x = static_cast<float>(rng.next_normal());
    return v;
}
struct Store {  // the same rows as a reference KvStore and a facade KvStore
    R::KvStore r;
    B::KvStore b;
};
static Store random_store(std::size_t n, std::size_t d, std::uint64_t seed) {
    const auto k = random_rows(n, d, R::mix_seed(seed, 1));
    const auto v = random_rows(n, d, R::mix_seed(seed, 2));
    return {R::KvStore(d, k, v), B::KvStore(d, k, v)};
}
static void append(Store& s, std::span<const float> k, std::span<const float> v) {
    s.r.append(k, v);
    s.b.append(k, v);
}
static std::vector<B::CentroidSet> random_centroids(const B::SubspaceLayout& layout, std::size_t c,
                                                    std::uint64_t seed) {
    std::vector<B::CentroidSet> sets(layout.count());
    for (std::size_t b = 0; b < layout.count(); ++b) {
        B::CentroidSet& cs = sets[b];
        cs.subspace_id = b;
        cs.count = c;
        cs.dim = layout.sizes[b];
        cs.centroids = random_rows(c, cs.dim, R::mix_seed(seed, b));
        for (std::size_t j = 0; j < c; ++j) B::l2_normalize(std::span<float>(cs.centroids.data() + j * cs.dim, cs.dim));
    }
    return sets;
}
static std::vector<R::CentroidSet> to_ref(const std::vector<B::CentroidSet>& s) {
    std::vector<R::CentroidSet> out(s.size());
    for (std::size_t b = 0; b < s.size(); ++b) {
        out[b].subspace_id = s[b].subspace_id;
        out[b].count = s[b].count;
        out[b].dim = s[b].dim;
        out[b].centroids = s[b].centroids;
    }
    return out;
}
static B::CentroidSet explicit_set(std::size_t b, std::size_t dim, std::vector<float> rows) {
    B::CentroidSet cs;
    cs.subspace_id = b;
    cs.dim = dim;
    cs.count = rows.size() / dim;
    cs.centroids = std::move(rows);
    return cs;
}
static B::IndexConfig injected_config(std::size_t c, double alpha) {
    B::IndexConfig cfg;
    cfg.alpha = alpha;
    cfg.score_bits = 32;
    cfg.cluster.centroids = c;
    return cfg;
}
static R::IndexConfig ref_cfg(const B::IndexConfig& c) {
    R::IndexConfig r;
    r.alpha = c.alpha;
    r.list_capacity = c.list_capacity;
    r.normalize_keys = c.normalize_keys;
    r.score_bits = c.score_bits;
    r.cluster.centroids = c.cluster.centroids;
    r.cluster.iterations = c.cluster.iterations;
    r.cluster.batch_size = c.cluster.batch_size;
    r.cluster.seed = c.cluster.seed;
    r.cluster.tolerance = c.cluster.tolerance;
    return r;
}
static B::IndexConfig config_for(std::size_t c, double alpha, std::uint64_t seed, int bits = 32) {
    B::IndexConfig cfg;
    cfg.alpha = alpha;
    cfg.score_bits = bits;
    cfg.cluster.centroids = c;
    cfg.cluster.seed = seed;
    cfg.cluster.batch_size = 1u << 20;
    return cfg;
}
static B::CsIndex random_index(const Store& kv, const B::SubspaceLayout& layout, std::size_t c, double alpha,
                               std::uint64_t seed) {
    return B::build_index_from_centroids(random_centroids(layout, c, seed), kv.b, layout, injected_config(c, alpha));
}
// d=4, m=2, axis-aligned centroids {[1,0],[0,1]} in both subspaces
static B::CsIndex axis_index(const Store& kv) {
    const B::SubspaceLayout layout({2, 2});
    std::vector<B::CentroidSet> sets;
    sets.push_back(explicit_set(0, 2, {1, 0, 0, 1}));
    sets.push_back(explicit_set(1, 2, {1, 0, 0, 1}));
    return B::build_index_from_centroids(std::move(sets), kv.b, layout, injected_config(2, 0.5));
}
static B::CandidateSet candidates_of(std::vector<std::uint32_t> idx, std::vector<double> scores) {
    B::CandidateSet cs;
    cs.indices = std::move(idx);
    cs.scores = std::move(scores);
    cs.source_counts.assign(cs.indices.size(), 1);
    return cs;
}
static B::TopList list_of(std::vector<std::uint32_t> idx, std::vector<float> scores) {
    B::TopList l;
    l.capacity = static_cast<std::uint32_t>(idx.size());
    l.indices = std::move(idx);
    l.scores = std::move(scores);
    return l;
}
static B::RetrievalConfig cfg_of(double rho, std::size_t period, std::size_t window) {
    B::RetrievalConfig cfg;
    cfg.keep_ratio = rho;
    cfg.search_period = period;
    cfg.recent_window = window;
    return cfg;
}
static R::RetrievalConfig ref_rc(const B::RetrievalConfig& c) {
    R::RetrievalConfig r;
    r.keep_ratio = c.keep_ratio;
    r.search_period = c.search_period;
    r.recent_window = c.recent_window;
    r.weights = c.weights;
    r.backoff_tau = c.backoff_tau;
    r.backoff_threshold = c.backoff_threshold;
    r.recent_passthrough = c.recent_passthrough;
    return r;
}
static bool same_tables(const B::CsIndex& a, const R::CsIndex& b) {
    if (a.tables.size() != b.tables.size() || a.list_capacity != b.list_capacity) return false;
    for (std::size_t t = 0; t < a.tables.size(); ++t)
        if (a.tables[t].indices != b.tables[t].indices || a.tables[t].scores != b.tables[t].scores) return false;
    return true;
}
static R::CsIndex ref_index_from(const std::vector<B::CentroidSet>& sets, const Store& kv,
                                 const B::SubspaceLayout& layout, const B::IndexConfig& cfg) {
    return R::build_index_from_centroids(to_ref(sets), kv.r, R::SubspaceLayout(layout.sizes), ref_cfg(cfg));
}

// =================== test_index.cpp ===================

static void toplist_cases() {
    CASE("top list keeps sorted order and evicts only on a strict win (test_index.cpp:60-86)");
    B::TopList list;
    list.capacity = 2;
    CHECK(list.min_score() == -std::numeric_limits<float>::infinity(), "empty min");
    CHECK(list.try_insert(0, 2.0f) && list.try_insert(1, 0.0f) && list.full(), "fill");
    CHECK(list.min_score() == 0.0f, "min");
    CHECK(list.try_insert(3, 1.0f), "strict win");
    CHECK((list.indices == std::vector<std::uint32_t>{0, 3}) && (list.scores == std::vector<float>{2.0f, 1.0f}),
          "evicted");
    CHECK(!list.try_insert(9, -0.5f) && (list.indices == std::vector<std::uint32_t>{0, 3}), "below min");
    CHECK(!list.try_insert(9, 1.0f) && (list.indices == std::vector<std::uint32_t>{0, 3}), "tie is no win");
    B::TopList empty;
    empty.capacity = 2;
    CHECK(empty.try_insert(4, 0.5f) && (empty.indices == std::vector<std::uint32_t>{4}), "empty insert");

    CASE("equal scores order by ascending index (test_index.cpp:88-97)");
    B::TopList l4;
    l4.capacity = 4;
    l4.try_insert(5, 1.0f);
    l4.try_insert(2, 1.0f);
    l4.try_insert(7, 1.0f);
    l4.try_insert(1, 3.0f);
    CHECK((l4.indices == std::vector<std::uint32_t>{1, 2, 5, 7}), "tie order");
    CHECK((l4.scores == std::vector<float>{3.0f, 1.0f, 1.0f, 1.0f}), "tie scores");

    CASE("from_scores keeps the top L with ties to the lower index (test_index.cpp:99-126), on the GPU");
    const std::vector<float> scores = {2.0f, 0.0f, -1.0f};
    const auto two = B::TopList::from_scores(scores, 2);
    CHECK((two.indices == std::vector<std::uint32_t>{0, 1}) && (two.scores == std::vector<float>{2.0f, 0.0f}),
          "top 2");
    const auto full = B::TopList::from_scores(scores, 10);
    CHECK((full.indices == std::vector<std::uint32_t>{0, 1, 2}) && full.capacity == 10, "L >= N");
    R::Rng rng(15);
    for (int trial = 0; trial < 20; ++trial) {
        std::vector<float> s(1000);
        for (float& x : s) x = static_cast<float>(rng.next_normal());
        const auto got = B::TopList::from_scores(s, 200);
        const auto ref = R::TopList::from_scores(s, 200);
        CHECK(got.indices == ref.indices && got.scores == ref.scores, "trial %d vs reference", trial);
    }
    // -0.0 and +0.0 compare equal: ties by index
    const std::vector<float> z = {-0.0f, 0.0f, -0.0f, 1.0f};
    const auto gz = B::TopList::from_scores(z, 3);
    CHECK((gz.indices == std::vector<std::uint32_t>{3, 0, 1}), "signed zeros tie");
}

static void score_cases() {
    CASE("score_keys projects raw key slices onto the centroid (test_index.cpp:128-147), on the GPU");
    std::vector<float> keys = {2, 1, 0, 3, -1, 4};
    std::vector<float> values(6, 0.0f);
    B::KvStore kv(2, keys, values);
    const B::SubspaceLayout layout({2});
    std::vector<float> c = {1, 0};
    CHECK((B::score_keys(c, kv, layout, 0, false, 3) == std::vector<float>{2.0f, 0.0f, -1.0f}), "raw");
    std::vector<float> zero_keys(6, 0.0f);
    B::KvStore zkv(2, zero_keys, values);
    for (float x : B::score_keys(c, zkv, layout, 0, false, 3)) CHECK(x == 0.0f, "zero keys");
    const auto norm = B::score_keys(c, kv, layout, 0, true, 3);
    CHECK(approx(norm[0], 2.0 / std::sqrt(5.0)) && approx(norm[1], 0.0) && approx(norm[2], -1.0 / std::sqrt(17.0)),
          "normalized");
    R::KvStore rkv(2, keys, values);
    CHECK(norm == R::score_keys(c, rkv, R::SubspaceLayout({2}), 0, true, 3), "normalized == reference bits");

    CASE("score_keys matches the scalar oracle on random data (test_index.cpp:149-164)");
    const std::size_t n = 32, d = 12;
    Store st = random_store(n, d, 91);
    const auto lay = B::SubspaceLayout::uniform(d, 3);
    R::Rng rng(17);
    for (std::size_t b = 0; b < 3; ++b) {
        std::vector<float> cc(lay.sizes[b]);
        for (float& x : cc) x = static_cast<float>(rng.next_normal());
        B::l2_normalize(cc);
        const auto s = B::score_keys(cc, st.b, lay, b, false, n);
        const auto r = R::score_keys(cc, st.r, R::SubspaceLayout(lay.sizes), b, false, n);
        CHECK(s == r, "subspace %zu bits vs reference", b);
        for (std::size_t i = 0; i < n; ++i)
            CHECK(approx(s[i], B::dot(cc, lay.slice(st.b.key(i), b))), "oracle %zu", i);
    }
}

static void build_cases() {
    CASE("default sizing: alpha 0.2 over 1000 rows gives 512 lists of 200 (test_index.cpp:166-180)");
    {
        const std::size_t p = 1000, d = 64;
        Store kv = random_store(p, d, 7);
        const auto q = random_rows(p, d, 8);
        const auto layout = B::SubspaceLayout::uniform(d, 8);
        const auto ix = B::build_index(q, p, kv.b, layout, config_for(64, 0.2, 3));
        CHECK(ix.tables.size() == 512 && ix.list_capacity == 200 && ix.alpha == 0.2, "sizing");
        bool all = true;
        for (const B::TopList& t : ix.tables) all &= t.capacity == 200 && t.indices.size() == 200;
        CHECK(all, "every list fills");
        const auto ref = R::build_index(q, p, kv.r, R::SubspaceLayout(layout.sizes), ref_cfg(config_for(64, 0.2, 3)));
        CHECK(same_tables(ix, ref), "tables == reference build_index");
    }
    CASE("degenerate m=1 C=1 alpha=1 index is the full sorted score list (test_index.cpp:182-198)");
    {
        const std::size_t p = 40, d = 6;
        Store kv = random_store(p, d, 23);
        const auto q = random_rows(p, d, 24);
        const B::SubspaceLayout layout({d});
        const auto ix = B::build_index(q, p, kv.b, layout, config_for(1, 1.0, 5));
        CHECK(ix.tables.size() == 1 && ix.tables[0].indices.size() == p, "one full list");
        const B::TopList& t = ix.tables[0];
        bool sorted = true;
        for (std::size_t r = 1; r < p; ++r) sorted &= t.scores[r] <= t.scores[r - 1];
        CHECK(sorted, "descending");
        std::vector<std::uint32_t> seen(t.indices);
        std::sort(seen.begin(), seen.end());
        bool each = true;
        for (std::size_t i = 0; i < p; ++i) each &= seen[i] == i;
        CHECK(each, "every key once");
    }
    CASE("small-instance table entries all recompute from their centroid (test_index.cpp:200-219)");
    {
        const std::size_t p = 64, d = 16;
        Store kv = random_store(p, d, 41);
        const auto q = random_rows(p, d, 42);
        const auto layout = B::SubspaceLayout::uniform(d, 4);
        const auto ix = B::build_index(q, p, kv.b, layout, config_for(4, 0.25, 9));
        CHECK(ix.tables.size() == 16 && ix.list_capacity == 16, "sizes");
        bool ok = true;
        for (std::size_t b = 0; b < 4; ++b)
            for (std::size_t j = 0; j < 4; ++j) {
                const B::TopList& t = ix.table(b, j);
                for (std::size_t r = 0; r < t.indices.size(); ++r)
                    ok &= approx(t.scores[r], B::dot(ix.centroid_sets[b].centroid(j),
                                                     layout.slice(kv.b.key(t.indices[r]), b)));
            }
        CHECK(ok, "entries recompute");
    }
    CASE("membership: a key is listed iff its score ranks in the top L (test_index.cpp:221-248)");
    {
        const std::size_t p = 256, d = 8;
        Store kv = random_store(p, d, 61);
        const auto layout = B::SubspaceLayout::uniform(d, 2);
        const auto sets = random_centroids(layout, 6, 62);
        const auto ix = B::build_index_from_centroids(sets, kv.b, layout, config_for(6, 0.1, 0));
        const std::size_t l = ix.list_capacity;
        for (std::size_t b = 0; b < 2; ++b)
            for (std::size_t j = 0; j < 6; ++j) {
                const auto s = B::score_keys(sets[b].centroid(j), kv.b, layout, b, false, p);
                std::vector<std::uint32_t> order(p);
                std::iota(order.begin(), order.end(), 0u);
                std::sort(order.begin(), order.end(), [&](std::uint32_t x, std::uint32_t y) {
                    return s[x] != s[y] ? s[x] > s[y] : x < y;
                });
                order.resize(l);
                std::sort(order.begin(), order.end());
                std::vector<std::uint32_t> got(ix.table(b, j).indices);
                std::sort(got.begin(), got.end());
                CHECK(got == order, "table (%zu,%zu)", b, j);
            }
        CHECK(same_tables(ix, ref_index_from(sets, kv, layout, config_for(6, 0.1, 0))), "== reference");
    }
    CASE("capacity law holds for every table and absolute L overrides (test_index.cpp:250-266)");
    {
        const std::size_t p = 100, d = 8;
        Store kv = random_store(p, d, 3);
        const auto q = random_rows(p, d, 4);
        const auto layout = B::SubspaceLayout::uniform(d, 2);
        const auto derived = B::build_index(q, p, kv.b, layout, config_for(3, 0.33, 1));
        CHECK(derived.list_capacity == R::ceil_ratio(0.33, p), "derived L");
        B::IndexConfig cfg = config_for(3, 0.2, 1);
        cfg.list_capacity = 7;
        const auto fixed = B::build_index(q, p, kv.b, layout, cfg);
        CHECK(fixed.list_capacity == 7 && approx(fixed.alpha, 0.07), "override L");
    }
    CASE("build rejects inconsistent parameters (test_index.cpp:268-288)");
    {
        const std::size_t p = 16, d = 4;
        Store kv = random_store(p, d, 5);
        const auto q = random_rows(p, d, 6);
        const auto layout = B::SubspaceLayout::uniform(d, 2);
        CHECK(throws<B::ParameterError>([&] { B::build_index(q, p, kv.b, layout, config_for(2, 0.0, 1)); }), "alpha 0");
        CHECK(throws<B::ParameterError>([&] { B::build_index(q, p, kv.b, layout, config_for(2, 1.5, 1)); }), "alpha 1.5");
        B::IndexConfig bad = config_for(2, 0.5, 1);
        bad.score_bits = 20;
        CHECK(throws<B::ParameterError>([&] { B::build_index(q, p, kv.b, layout, bad); }), "bits");
        CHECK(throws<B::DimensionError>([&] { B::build_index(q, p - 1, kv.b, layout, config_for(2, 0.5, 1)); }),
              "count");
        const auto wide = B::SubspaceLayout::uniform(d + 2, 2);
        CHECK(throws<B::DimensionError>([&] { B::build_index(q, p, kv.b, wide, config_for(2, 0.5, 1)); }), "width");
    }
    CASE("build is deterministic for a fixed seed (test_index.cpp:290-301)");
    {
        const std::size_t p = 128, d = 16;
        Store kv = random_store(p, d, 81);
        const auto q = random_rows(p, d, 82);
        const auto layout = B::SubspaceLayout::uniform(d, 4);
        const auto a = B::build_index(q, p, kv.b, layout, config_for(8, 0.2, 77));
        const auto b = B::build_index(q, p, kv.b, layout, config_for(8, 0.2, 77));
        const auto c = B::build_index(q, p, kv.b, layout, config_for(8, 0.2, 78));
        CHECK(B::serialize_index(a) == B::serialize_index(b), "same seed");
        CHECK(B::serialize_index(a) != B::serialize_index(c), "other seed");
    }
}

// =================== test_retrieval.cpp ===================

static void routing_cases() {
    const double ninf = -std::numeric_limits<double>::infinity();
    CASE("centroid selection takes the cosine argmax per subspace (test_retrieval.cpp:134-149)");
    {
        Store kv = random_store(8, 4, 1);
        const auto ix = axis_index(kv);
        std::vector<float> q = {0.6f, 0.8f, 1.0f, 0.0f};
        const auto sel = B::select_centroids(q, ix, 1, ninf);
        CHECK(sel.per_subspace.size() == 2, "m");
        CHECK((sel.per_subspace[0] == std::vector<std::uint32_t>{1}) && approx(sel.best_cosine[0], 0.8), "b0");
        CHECK((sel.per_subspace[1] == std::vector<std::uint32_t>{0}) && approx(sel.best_cosine[1], 1.0), "b1");
        CHECK(sel.dot_ops == 2 * 2 + 2 * 2, "dot ops");
    }
    CASE("an impossible threshold forces top-tau backoff everywhere (test_retrieval.cpp:151-166)");
    {
        Store kv = random_store(8, 4, 2);
        const auto ix = axis_index(kv);
        std::vector<float> q = {0.6f, 0.8f, 0.6f, 0.8f};
        const auto sel = B::select_centroids(q, ix, 2, 1.1);
        for (std::size_t b = 0; b < 2; ++b)
            CHECK((sel.per_subspace[b] == std::vector<std::uint32_t>{1, 0}), "backoff order b%zu", b);
        CHECK(B::select_centroids(q, ix, 9, 1.1).per_subspace[0].size() == 2, "tau clips to C");
    }
    CASE("a zero query slice matches centroid 0 without backoff (test_retrieval.cpp:168-176)");
    {
        Store kv = random_store(8, 4, 3);
        const auto ix = axis_index(kv);
        std::vector<float> q = {0.0f, 0.0f, 0.3f, 0.4f};
        const auto sel = B::select_centroids(q, ix, 2, 1.1);
        CHECK((sel.per_subspace[0] == std::vector<std::uint32_t>{0}) && sel.best_cosine[0] == 1.0, "zero slice");
        CHECK(sel.per_subspace[1].size() == 2, "real slice backs off");
    }
    CASE("top-1 selection matches an exhaustive argmax over 64 centroids (test_retrieval.cpp:178-201)");
    {
        const std::size_t d = 8;
        Store kv = random_store(16, d, 4);
        const auto layout = B::SubspaceLayout::uniform(d, 2);
        const auto ix = B::build_index_from_centroids(random_centroids(layout, 64, 5), kv.b, layout,
                                                      injected_config(64, 0.5));
        R::Rng rng(6);
        for (int trial = 0; trial < 20; ++trial) {
            std::vector<float> q(d);
            for (float& x : q) x = static_cast<float>(rng.next_normal());
            const auto sel = B::select_centroids(q, ix, 1, ninf);
            for (std::size_t b = 0; b < 2; ++b) {
                std::vector<float> slice(layout.slice(q, b).begin(), layout.slice(q, b).end());
                B::l2_normalize(slice);
                const auto sc = B::centroid_scores(slice, ix.centroid_sets[b]);
                std::size_t best = 0;
                for (std::size_t j = 1; j < sc.size(); ++j)
                    if (sc[j] > sc[best]) best = j;
                CHECK((sel.per_subspace[b] == std::vector<std::uint32_t>{static_cast<std::uint32_t>(best)}),
                      "trial %d b%zu", trial, b);
            }
        }
    }
    CASE("gathering returns m lists, or m*tau under backoff (test_retrieval.cpp:203-218)");
    {
        Store kv = random_store(8, 4, 7);
        const auto ix = axis_index(kv);
        std::vector<float> q = {0.6f, 0.8f, 1.0f, 0.0f};
        const auto one = B::gather_lists(ix, B::select_centroids(q, ix, 1, ninf));
        CHECK(one.lists.size() == 2 && (one.subspace == std::vector<std::size_t>{0, 1}) &&
                  one.lists[0] == &ix.table(0, 1),
              "one");
        const auto two = B::gather_lists(ix, B::select_centroids(q, ix, 2, 1.1));
        CHECK(two.lists.size() == 4 && two.total_entries() == 4 * ix.tables[0].indices.size(), "two");
    }
}

static void reduce_cases() {
    CASE("reduce_by_key sums weighted partial scores, missing lists give 0 (test_retrieval.cpp:220-245)");
    {
        B::GatheredLists g;
        const B::TopList l1 = list_of({3, 7}, {0.9f, 0.4f});
        const B::TopList l2 = list_of({7, 1}, {0.5f, 0.2f});
        g.lists = {&l1, &l2};
        g.subspace = {0, 1};
        const std::vector<double> ones = {1.0, 1.0};
        const auto flat = B::reduce_by_key(g, ones);
        CHECK((flat.indices == std::vector<std::uint32_t>{1, 3, 7}), "keys");
        CHECK(approx(flat.scores[0], 0.2) && approx(flat.scores[1], 0.9) && approx(flat.scores[2], 0.9), "sums");
        CHECK((flat.source_counts == std::vector<std::uint32_t>{1, 1, 2}), "counts");
        // exact doubles: the reference's own sums
        R::TopList r1, r2;
        r1.capacity = 2;
        r1.indices = {3, 7};
        r1.scores = {0.9f, 0.4f};
        r2.capacity = 2;
        r2.indices = {7, 1};
        r2.scores = {0.5f, 0.2f};
        R::GatheredLists rg;
        rg.lists = {&r1, &r2};
        rg.subspace = {0, 1};
        CHECK(flat.scores == R::reduce_by_key(rg, ones).scores, "bits == reference");
        const std::vector<double> weighted = {2.0, 1.0};
        const auto scaled = B::reduce_by_key(g, weighted);
        CHECK(approx(scaled.scores[0], 0.2) && approx(scaled.scores[1], 1.8) && approx(scaled.scores[2], 1.3),
              "weighted");
        CHECK(scaled.scores == R::reduce_by_key(rg, weighted).scores, "weighted bits == reference");
        const std::vector<double> short_w = {1.0};
        CHECK(throws<B::DimensionError>([&] { B::reduce_by_key(g, short_w); }), "short weights");
    }
    CASE("disjoint lists reduce to their union (test_retrieval.cpp:247-259)");
    {
        B::GatheredLists g;
        const B::TopList l1 = list_of({0, 2}, {1.0f, 0.5f});
        const B::TopList l2 = list_of({5, 9}, {0.7f, 0.1f});
        g.lists = {&l1, &l2};
        g.subspace = {0, 1};
        const std::vector<double> ones = {1.0, 1.0};
        const auto out = B::reduce_by_key(g, ones);
        CHECK((out.indices == std::vector<std::uint32_t>{0, 2, 5, 9}), "keys");
        CHECK((out.scores == std::vector<double>{1.0, 0.5, 0.699999988079071044921875, 0.100000001490116119384765625}),
              "exact doubles");
        for (auto c : out.source_counts) CHECK(c == 1, "counts");
    }
}

static void topk_cases() {
    CASE("passthrough keeps the window and fills the rest by score (test_retrieval.cpp:261-266)");
    {
        Store kv = random_store(10, 2, 8);
        CHECK((B::select_topk(candidates_of({0, 1, 7}, {9.0, 8.0, 0.1}), kv.b, cfg_of(0.5, 1, 3)) ==
               std::vector<std::uint32_t>{0, 1, 7, 8, 9}),
              "{0,1,7,8,9}");
    }
    CASE("full keep selects every index regardless of candidates (test_retrieval.cpp:268-275)");
    {
        Store kv = random_store(10, 2, 9);
        std::vector<std::uint32_t> all(10);
        std::iota(all.begin(), all.end(), 0u);
        CHECK(B::select_topk(candidates_of({4}, {1.0}), kv.b, cfg_of(1.0, 1, 3)) == all, "all");
    }
    CASE("a budget below the window keeps only the newest K (test_retrieval.cpp:277-282)");
    {
        Store kv = random_store(10, 2, 10);
        CHECK((B::select_topk(candidates_of({0, 1}, {9.0, 8.0}), kv.b, cfg_of(0.2, 1, 3)) ==
               std::vector<std::uint32_t>{8, 9}),
              "{8,9}");
    }
    CASE("with no window the selection is a plain top-K sort (test_retrieval.cpp:284-305)");
    {
        const std::size_t n = 200;
        Store kv = random_store(n, 2, 11);
        R::Rng rng(12);
        std::vector<std::uint32_t> idx(n);
        std::iota(idx.begin(), idx.end(), 0u);
        std::vector<double> scores(n);
        for (double& s : scores) s = rng.next_normal();
        const auto got = B::select_topk(candidates_of(idx, scores), kv.b, cfg_of(0.05, 1, 0));
        std::vector<std::uint32_t> order(n);
        std::iota(order.begin(), order.end(), 0u);
        std::sort(order.begin(), order.end(),
                  [&](std::uint32_t a, std::uint32_t b) { return scores[a] != scores[b] ? scores[a] > scores[b] : a < b; });
        order.resize(10);
        std::sort(order.begin(), order.end());
        CHECK(got == order, "top-10");
    }
    CASE("no candidates and no window falls back to the newest positions (test_retrieval.cpp:307-312)");
    {
        Store kv = random_store(10, 2, 13);
        CHECK((B::select_topk(B::CandidateSet{}, kv.b, cfg_of(0.3, 1, 0)) == std::vector<std::uint32_t>{7, 8, 9}),
              "{7,8,9}");
    }
    CASE("without passthrough the window competes at its accumulated score (test_retrieval.cpp:314-321)");
    {
        Store kv = random_store(6, 2, 14);
        B::RetrievalConfig cfg = cfg_of(0.5, 1, 2);
        cfg.recent_passthrough = false;
        CHECK((B::select_topk(candidates_of({0, 1, 4}, {5.0, 0.5, -1.0}), kv.b, cfg) ==
               std::vector<std::uint32_t>{0, 1, 5}),
              "{0,1,5}");
    }
    CASE("selection always returns exactly K ascending unique indices (test_retrieval.cpp:323-345), == reference");
    {
        R::Rng rng(15);
        for (int trial = 0; trial < 40; ++trial) {
            const std::size_t n = 1 + rng.next_index(64);
            Store kv = random_store(n, 2, R::mix_seed(15, trial));
            B::CandidateSet cand;
            R::CandidateSet rc;
            for (std::size_t i = 0; i < n; ++i)
                if (rng.next_unit() < 0.3) {
                    const double s = rng.next_normal();
                    cand.indices.push_back(static_cast<std::uint32_t>(i));
                    cand.scores.push_back(s);
                    cand.source_counts.push_back(1);
                    rc.indices.push_back(static_cast<std::uint32_t>(i));
                    rc.scores.push_back(s);
                    rc.source_counts.push_back(1);
                }
            B::RetrievalConfig cfg = cfg_of(0.05 + 0.9 * rng.next_unit(), 1, rng.next_index(8));
            cfg.recent_passthrough = rng.next_unit() < 0.5;
            const auto got = B::select_topk(cand, kv.b, cfg);
            CHECK(got.size() == B::keep_count(cfg.keep_ratio, n) && std::is_sorted(got.begin(), got.end()) &&
                      std::adjacent_find(got.begin(), got.end()) == got.end(),
                  "trial %d shape", trial);
            CHECK(got == R::select_topk(rc, kv.r, ref_rc(cfg)), "trial %d == reference", trial);
        }
    }
    CASE("weight rescaling leaves the selected set unchanged (test_retrieval.cpp:347-363)");
    {
        const std::size_t d = 8, n = 96;
        Store kv = random_store(n, d, 16);
        const auto layout = B::SubspaceLayout::uniform(d, 2);
        const auto ix = random_index(kv, layout, 6, 0.25, 17);
        std::vector<float> q = random_rows(1, d, 18);
        const auto g = B::gather_lists(ix, B::select_centroids(q, ix, 1, -std::numeric_limits<double>::infinity()));
        const std::vector<double> w1 = {1.0, 2.0}, w3 = {3.0, 6.0};
        CHECK(B::select_topk(B::reduce_by_key(g, w1), kv.b, cfg_of(0.1, 1, 4)) ==
                  B::select_topk(B::reduce_by_key(g, w3), kv.b, cfg_of(0.1, 1, 4)),
              "rescaled");
    }
}

static void search_cases() {
    CASE("decode_search follows the period and recomputes K per step (test_retrieval.cpp:365-396), == reference");
    {
        const std::size_t d = 4, p = 32;
        Store kv = random_store(p, d, 19);
        const auto layout = B::SubspaceLayout::uniform(d, 2);
        const auto sets = random_centroids(layout, 2, 20);
        const auto ix = B::build_index_from_centroids(sets, kv.b, layout, injected_config(2, 0.5));
        const auto rix = ref_index_from(sets, kv, layout, injected_config(2, 0.5));
        const B::RetrievalConfig cfg = cfg_of(0.25, 4, 2);
        B::SearchState state;
        R::SearchState rstate;
        R::Rng rng(21);
        for (std::size_t t = 0; t < 8; ++t) {
            std::vector<float> q(d), k(d), v(d);
            for (float& x : q) x = static_cast<float>(rng.next_normal());
            for (float& x : k) x = static_cast<float>(rng.next_normal());
            for (float& x : v) x = static_cast<float>(rng.next_normal());
            const auto res = B::decode_search(q, ix, kv.b, cfg, state);
            const auto ref = R::decode_search(q, rix, kv.r, ref_rc(cfg), rstate);
            CHECK(res.searched == (t % 4 == 0) && res.k == B::keep_count(0.25, p + t) && res.selected.size() == res.k,
                  "step %zu shape", t);
            if (!res.searched)
                CHECK(res.centroid_dot_ops == 0 && res.gathered_entries == 0 && res.reduce_ops == 0, "reuse");
            else
                CHECK(res.centroid_dot_ops > 0, "searched");
            CHECK(std::find(res.selected.begin(), res.selected.end(), static_cast<std::uint32_t>(p + t - 1)) !=
                      res.selected.end(),
                  "newest kept");
            CHECK(res.selected == ref.selected && res.centroid_dot_ops == ref.centroid_dot_ops &&
                      res.gathered_entries == ref.gathered_entries,
                  "step %zu == reference", t);
            append(kv, k, v);
        }
    }
    CASE("reuse steps ignore keys appended after the last search (test_retrieval.cpp:398-418)");
    {
        const std::size_t d = 4, p = 32;
        Store kv = random_store(p, d, 22);
        const auto layout = B::SubspaceLayout::uniform(d, 2);
        const auto ix = random_index(kv, layout, 2, 0.5, 23);
        const B::RetrievalConfig cfg = cfg_of(0.25, 100, 0);
        B::SearchState state;
        std::vector<float> q = random_rows(1, d, 24);
        (void)B::decode_search(q, ix, kv.b, cfg, state);
        for (int t = 0; t < 5; ++t) {
            std::vector<float> k(q.begin(), q.end());
            for (float& x : k) x *= 50.0f;
            append(kv, k, k);
            const auto res = B::decode_search(q, ix, kv.b, cfg, state);
            CHECK(!res.searched, "reuse");
            for (auto i : res.selected) CHECK(i < p, "stale cache");
        }
    }
    CASE("gathered work is bounded by m*tau*L and constant across steps (test_retrieval.cpp:420-446)");
    {
        const std::size_t d = 6, p = 60;
        Store kv = random_store(p, d, 25);
        const auto layout = B::SubspaceLayout::uniform(d, 3);
        const auto ix = random_index(kv, layout, 5, 0.2, 26);
        const std::size_t l = ix.list_capacity;
        B::RetrievalConfig cfg = cfg_of(0.1, 1, 2);
        cfg.backoff_tau = 2;
        cfg.backoff_threshold = 2.0;
        B::SearchState state;
        R::Rng rng(27);
        std::size_t first = 0;
        for (std::size_t t = 0; t < 6; ++t) {
            std::vector<float> q(d);
            for (float& x : q) x = static_cast<float>(rng.next_normal());
            const auto res = B::decode_search(q, ix, kv.b, cfg, state);
            CHECK(res.gathered_entries == 3 * 2 * l, "bounded");
            if (t == 0) first = res.centroid_dot_ops;
            else CHECK(res.centroid_dot_ops == first, "constant");
        }
    }
}

static void insert_cases() {
    CASE("streaming insert offers the key to every table (test_retrieval.cpp:448-471)");
    {
        const std::size_t p = 20;
        Store kv = random_store(p, 4, 28);
        auto ix = axis_index(kv);
        const std::size_t l = ix.list_capacity;
        std::vector<float> key = {9.0f, 0.0f, 0.1f, 0.1f};
        const auto rep = B::streaming_insert(key, static_cast<std::uint32_t>(p), ix);
        CHECK(rep.attempted == 4 && rep.dot_ops == 2 * 2 + 2 * 2 && rep.applied_mask.size() == 4, "report");
        CHECK(rep.applied_mask[0] == 1 && ix.table(0, 0).indices.front() == p && ix.table(0, 0).scores.front() == 9.0f,
              "table (0,0)");
        std::size_t applied = 0;
        for (auto f : rep.applied_mask) applied += f;
        CHECK(applied == rep.applied, "mask sum");
        for (const B::TopList& t : ix.tables)
            CHECK(t.indices.size() <= t.capacity && t.capacity == l && std::is_sorted(t.scores.rbegin(), t.scores.rend()),
                  "invariants");
    }
    CASE("incremental inserts equal a batch scoring pass over all keys (test_retrieval.cpp:473-510), 50 seeds");
    {
        int bad = 0;
        for (std::uint64_t seed = 0; seed < 50; ++seed) {
            R::Rng rng(R::mix_seed(900, seed));
            const std::size_t d = 4 * (1 + rng.next_index(3));
            const std::size_t m = 1 + rng.next_index(std::min<std::size_t>(4, d));
            const std::size_t c = 1 + rng.next_index(6);
            const std::size_t p = 16 + rng.next_index(113);
            const std::size_t extra = 1 + rng.next_index(128);
            const double alpha = 0.1 + 0.9 * rng.next_unit();
            const auto layout = B::SubspaceLayout::uniform(d, m);
            const auto all_k = random_rows(p + extra, d, R::mix_seed(901, seed));
            const auto all_v = random_rows(p + extra, d, R::mix_seed(902, seed));
            const auto sets = random_centroids(layout, c, R::mix_seed(903, seed));
            B::KvStore kv_inc(d, std::span<const float>(all_k.data(), p * d), std::span<const float>(all_v.data(), p * d));
            B::CsIndex inc = B::build_index_from_centroids(sets, kv_inc, layout, injected_config(c, alpha));
            for (std::size_t t = 0; t < extra; ++t)
                B::streaming_insert(std::span<const float>(all_k.data() + (p + t) * d, d),
                                    static_cast<std::uint32_t>(p + t), inc);
            B::KvStore kv_all(d, all_k, all_v);
            B::IndexConfig bc = injected_config(c, alpha);
            bc.list_capacity = inc.list_capacity;
            const B::CsIndex batch = B::build_index_from_centroids(sets, kv_all, layout, bc);
            bool same = inc.tables.size() == batch.tables.size();
            for (std::size_t t = 0; same && t < inc.tables.size(); ++t)
                same = inc.tables[t].indices == batch.tables[t].indices && inc.tables[t].scores == batch.tables[t].scores;
            bad += same ? 0 : 1;
        }
        CHECK(bad == 0, "%d of 50 seeds differ", bad);
    }
}

static void exactness_cases() {
    CASE("query-matched centroids make retrieval exactly dense (test_retrieval.cpp:512-543)");
    {
        R::Rng rng(31);
        for (int trial = 0; trial < 20; ++trial) {
            const std::size_t d = 4 * (1 + rng.next_index(3));
            const std::size_t m = 1 + rng.next_index(2);
            const std::size_t n = 32 + rng.next_index(225);
            const auto layout = B::SubspaceLayout::uniform(d, m);
            Store kv = random_store(n, d, R::mix_seed(32, trial));
            std::vector<float> q = random_rows(1, d, R::mix_seed(33, trial));
            std::vector<float> qn;
            std::vector<B::CentroidSet> sets;
            for (std::size_t b = 0; b < m; ++b) {
                std::vector<float> slice(layout.slice(q, b).begin(), layout.slice(q, b).end());
                B::l2_normalize(slice);
                qn.insert(qn.end(), slice.begin(), slice.end());
                sets.push_back(explicit_set(b, layout.sizes[b], slice));
            }
            const auto ix = B::build_index_from_centroids(sets, kv.b, layout, injected_config(1, 1.0));
            B::RetrievalConfig cfg = cfg_of(0.05 + 0.5 * rng.next_unit(), 1, 0);
            cfg.recent_passthrough = false;
            B::SearchState state;
            const auto res = B::decode_search(q, ix, kv.b, cfg, state);
            CHECK(res.selected == B::dense_topk(qn, kv.b, res.k), "trial %d == dense_topk", trial);
            CHECK(res.selected == R::dense_topk(qn, kv.r, res.k), "trial %d == reference dense_topk", trial);
        }
    }
    CASE("recall grows with list capacity on a planted workload (test_retrieval.cpp:545-577)");
    {
        const std::size_t d = 8, n = 160;
        auto keys = random_rows(n, d, 41);
        const auto values = random_rows(n, d, 42);
        std::vector<float> dir = random_rows(1, d, 43);
        B::l2_normalize(dir);
        for (std::size_t i = 0; i < n; i += 10)
            for (std::size_t t = 0; t < d; ++t) keys[i * d + t] = 5.0f * dir[t] + 0.3f * keys[i * d + t];
        B::KvStore kvb(d, keys, values);
        R::KvStore kvr(d, keys, values);
        Store kv{std::move(kvr), std::move(kvb)};
        const auto layout = B::SubspaceLayout::uniform(d, 2);
        std::vector<float> q(d);
        for (std::size_t t = 0; t < d; ++t) q[t] = 4.0f * dir[t];
        const auto truth = B::dense_topk(q, kv.b, 16);
        double last = -1.0;
        for (double alpha : {0.05, 0.25, 1.0}) {
            const auto ix = random_index(kv, layout, 4, alpha, 44);
            B::SearchState state;
            const auto res = B::decode_search(q, ix, kv.b, cfg_of(0.1, 1, 0), state);
            double hits = 0;
            for (auto i : res.selected) hits += std::binary_search(truth.begin(), truth.end(), i) ? 1 : 0;
            const double recall = hits / 16.0;
            CHECK(recall >= last, "alpha %.2f recall %.3f", alpha, recall);
            last = recall;
        }
        CHECK(last > 0.5, "full lists recover most planted rows (%.3f)", last);
    }
    CASE("dense_attention over host rows matches the reference (core.cpp:118-169)");
    {
        Store kv = random_store(300, 16, 55);
        std::vector<float> q = random_rows(1, 16, 56);
        const std::vector<std::uint32_t> mask = {3, 7, 100, 299, 0};
        const auto a = B::dense_attention(q, kv.b, std::span<const std::uint32_t>(mask));
        const auto r = R::dense_attention(q, kv.r, std::span<const std::uint32_t>(mask));
        double err = 0, nrm = 0;
        for (std::size_t t = 0; t < 16; ++t) {
            err += (a.output[t] - r.output[t]) * (a.output[t] - r.output[t]);
            nrm += r.output[t] * r.output[t];
        }
        CHECK(std::sqrt(err / nrm) <= 1e-6 && a.weights.size() == mask.size(), "masked rel err %.3g", std::sqrt(err / nrm));
        CHECK(throws<B::ParameterError>([&] { B::dense_attention(q, kv.b, std::span<const std::uint32_t>()); }),
              "empty mask");
    }
}

int main() {
    toplist_cases();
    score_cases();
    build_cases();
    routing_cases();
    reduce_cases();
    topk_cases();
    search_cases();
    insert_cases();
    exactness_cases();
    std::printf("%d checks, %d failures\n", checks, failures);
    if (failures == 0) std::printf("ALL OK\n");
    return failures ? 1 : 0;
}
