// test_facade.cpp — the reference's own session-level checks, run twice with
// the same calls: once through the UNMODIFIED reference library (namespace
// csattn_ref, oracle/_ref) and once through the B200 drop-in facade
// (include/csattn_b200.hpp -> C ABI -> sm_100a kernels). TEST INFRASTRUCTURE:
// it links the checker; it is built by tests/cpp/Makefile where
// /root/reference exists and run by tests/test_cpp_facade.py on a B200.
//
// Mirrors test_session.cpp: prefill validation (:222-267), full lifecycle vs
// reference with exact selected sets and output agreement (:113-151),
// counters (:66-82, :153-168), stream exhaustion message (:179-196), and
// table equality after streaming inserts (acceptance.cpp:229-267).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "csattn/session.hpp"    // reference (compiled with -Dcsattn=csattn_ref)
#include "csattn/synthetic.hpp"
#include "csattn_b200.hpp"       // B200 facade

namespace R = csattn_ref;
namespace B = csattn_b200;

static int failures = 0;
#define CHECK(cond, ...)                                   \
    do {                                                   \
        if (!(cond)) {                                     \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                      \
            std::printf("\n");                             \
            ++failures;                                    \
        }                                                  \
    } while (0)

template <class E, class F>
static std::string thrown(F&& f) {
    try {
        f();
    } catch (const E& e) {
        return e.what();
    } catch (...) {
        return "<other exception>";
    }
    return "<none>";
}

static void lifecycle(std::size_t P, std::size_t T, std::size_t d, std::size_t m, std::uint64_t seed,
                      const char* schedule, bool passthrough) {
    R::SyntheticSpec spec;
    spec.rows = P + T;
    spec.dim = d;
    spec.seed = seed;
    const R::SyntheticWorkload w = R::make_synthetic(spec);
    const std::span<const float> q(w.queries), k(w.keys), v(w.values);
    auto pre = [&](std::span<const float> x) { return x.subspan(0, P * d); };
    auto tail = [&](std::span<const float> x) { return x.subspan(P * d, T * d); };

    R::IndexConfig ric;
    ric.cluster.seed = 1;
    ric.score_bits = 32;
    B::IndexConfig bic;
    bic.cluster.seed = 1;
    bic.score_bits = 32;
    const auto [rho, period] = R::parse_schedule(schedule);
    const auto [brho, bperiod] = B::parse_schedule(schedule);
    CHECK(rho == brho && period == bperiod, "parse_schedule(%s)", schedule);
    R::RetrievalConfig rrc;
    rrc.keep_ratio = rho;
    rrc.search_period = period;
    rrc.recent_passthrough = passthrough;
    B::RetrievalConfig brc;
    brc.keep_ratio = brho;
    brc.search_period = bperiod;
    brc.recent_passthrough = passthrough;

    R::Session rs = R::prefill(pre(q), pre(k), pre(v), R::SubspaceLayout::uniform(d, m), ric, rrc);
    B::Session bs = B::prefill(pre(q), pre(k), pre(v), B::SubspaceLayout::uniform(d, m), bic, brc, T);
    B::Session bg = bs.fork(T);  // decoded below as one CUDA graph (run_decode_graph)

    // offline build: identical tables (membership, order, scores)
    {
        const B::CsIndex bi = bs.export_index();
        CHECK(bi.tables.size() == rs.index.tables.size(), "table count");
        std::size_t diff = 0;
        for (std::size_t t = 0; t < bi.tables.size(); ++t)
            diff += (bi.tables[t].indices != rs.index.tables[t].indices ||
                     bi.tables[t].scores != rs.index.tables[t].scores);
        CHECK(diff == 0, "P=%zu: %zu of %zu prefill tables differ", P, diff, bi.tables.size());
        CHECK(bi.list_capacity == rs.index.list_capacity, "L");
    }

    const auto rr = R::run_decode(rs, tail(q), tail(k), tail(v), T, false);
    const auto br = B::run_decode(bs, tail(q), tail(k), tail(v), T, false);
    std::size_t sel_diff = 0;
    double worst = 0.0;
    for (std::size_t t = 0; t < T; ++t) {
        sel_diff += rr[t].selected != br[t].selected;
        double e2 = 0.0, n2 = 0.0;
        for (std::size_t x = 0; x < d; ++x) {
            const double a = rr[t].attention.output[x], b = br[t].attention.output[x];
            e2 += (a - b) * (a - b);
            n2 += a * a;
        }
        worst = std::max(worst, std::sqrt(e2 / n2));
        CHECK(rr[t].k == br[t].k && rr[t].searched == br[t].searched, "step %zu k/searched", t);
        const auto& a = rr[t].counters;
        const auto& b = br[t].counters;
        CHECK(a.centroid_dot_ops == b.centroid_dot_ops && a.gathered_entries == b.gathered_entries &&
                  a.reduce_ops == b.reduce_ops && a.attention_key_ops == b.attention_key_ops &&
                  a.searches == b.searches && a.inserts_attempted == b.inserts_attempted &&
                  a.inserts_applied == b.inserts_applied && a.insert_dot_ops == b.insert_dot_ops &&
                  a.h2d_bytes_model == b.h2d_bytes_model,
              "step %zu counters differ", t);
    }
    CHECK(sel_diff == 0, "P=%zu %s: %zu of %zu selected sets differ", P, schedule, sel_diff, T);
    {
        // the graph run asks for no softmax weights, so small batches take the
        // fused cluster step (fused.cu) whose attention sums in another order
        // than attend128's chunks: same selected sets, outputs within 1e-5
        const B::GraphRun gr = B::run_decode_graph(bg, tail(q), tail(k), tail(v), T);
        std::size_t gdiff = 0;
        for (std::size_t t = 0; t < T; ++t) {
            double e2 = 0.0, n2 = 0.0;
            for (std::size_t x = 0; x < d; ++x) {
                const double a = br[t].attention.output[x], b = gr.outputs[t * d + x];
                e2 += (a - b) * (a - b);
                n2 += a * a;
            }
            gdiff += gr.selected[t] != br[t].selected || std::sqrt(e2 / n2) > 1e-5;
        }
        CHECK(gdiff == 0, "P=%zu %s: %zu of %zu graph-run steps differ", P, schedule, gdiff, T);
        CHECK(bg.serialize() == bs.serialize(), "P=%zu: graph-run tables differ", P);
    }
    CHECK(worst <= 1e-3, "P=%zu %s: output rel err %.3g", P, schedule, worst);
    CHECK(rs.totals.inserts_applied == bs.totals.inserts_applied, "totals");

    // streaming inserts: tables still identical (acceptance.cpp:229-267)
    {
        const B::CsIndex bi = bs.export_index();
        std::size_t diff = 0;
        for (std::size_t t = 0; t < bi.tables.size(); ++t)
            diff += (bi.tables[t].indices != rs.index.tables[t].indices ||
                     bi.tables[t].scores != rs.index.tables[t].scores);
        CHECK(diff == 0, "P=%zu: %zu tables differ after %zu inserts", P, diff, T);
    }
    // CSAT v1 images (index.cpp:289-433): host codec and device writer against
    // serialize_index; load -> decode identical (acceptance.cpp:425-468)
    {
        const auto ref_img = R::serialize_index(rs.index);
        CHECK(B::serialize_index(bs.export_index()) == ref_img, "P=%zu: host CSAT image differs", P);
        CHECK(bs.serialize() == ref_img, "P=%zu: device CSAT image differs", P);
        const B::CsIndex back = B::deserialize_index(ref_img);
        CHECK(B::serialize_index(back) == ref_img, "P=%zu: CSAT decode/encode round trip", P);
        const auto fp_r = R::index_footprint(rs.index);
        const auto fp_b = B::index_footprint(back);
        CHECK(fp_r.header_bytes == fp_b.header_bytes && fp_r.centroid_bytes == fp_b.centroid_bytes &&
                  fp_r.entry_bytes == fp_b.entry_bytes,
              "P=%zu: footprint", P);
        // load the image into fresh sessions on both sides and decode two more steps
        // the image indexes appended keys too: load with all P + T rows
        std::vector<float> kk, vv;
        bs.read_kv(0, P + T, kk, vv);
        B::Session bl = B::load_session(ref_img, kk, vv, brc, 4);
        R::Session rl(R::KvStore(d, k.subspan(0, (P + T) * d), v.subspan(0, (P + T) * d)),
                      R::deserialize_index(ref_img), rrc);
        const auto rr2 = R::run_decode(rl, pre(q).subspan(0, 2 * d), pre(k).subspan(0, 2 * d),
                                       pre(v).subspan(0, 2 * d), 2, false);
        const auto br2 = B::run_decode(bl, pre(q).subspan(0, 2 * d), pre(k).subspan(0, 2 * d),
                                       pre(v).subspan(0, 2 * d), 2, false);
        for (std::size_t t = 0; t < 2; ++t)
            CHECK(rr2[t].selected == br2[t].selected, "P=%zu: loaded-session step %zu differs", P, t);
        CHECK(bl.serialize() == R::serialize_index(rl.index), "P=%zu: loaded session image after inserts", P);
        // load errors: same class and message (test_index.cpp:361-390)
        auto bad = ref_img;
        bad[4] = 9;
        const std::string a = thrown<R::VersionError>([&] { R::deserialize_index(bad); });
        const std::string b = thrown<B::VersionError>([&] { B::deserialize_index(bad); });
        CHECK(a == b, "version error: '%s' vs '%s'", a.c_str(), b.c_str());
        bad = ref_img;
        bad.resize(bad.size() / 3);
        const std::string c = thrown<R::TruncatedError>([&] { R::deserialize_index(bad); });
        const std::string e = thrown<B::TruncatedError>([&] { B::deserialize_index(bad); });
        CHECK(c == e, "truncation error: '%s' vs '%s'", c.c_str(), e.c_str());
    }
    std::printf("lifecycle P=%zu T=%zu d=%zu m=%zu %s pt=%d: sets equal %zu/%zu, rel err %.2e\n", P,
                T, d, m, schedule, passthrough ? 1 : 0, T - sel_diff, T, worst);
}

// compare_dense (session.cpp:66-78): the dense reference, recall@K against
// dense_topk and the l2 error, with the dense oracle on the GPU
static void dense_compare() {
    const std::size_t P = 4096, T = 4, d = 128;
    R::SyntheticSpec spec;
    spec.rows = P + T;
    spec.dim = d;
    spec.seed = 77;
    const R::SyntheticWorkload w = R::make_synthetic(spec);
    const std::span<const float> q(w.queries), k(w.keys), v(w.values);
    R::IndexConfig ric;
    ric.cluster.seed = 1;
    ric.score_bits = 32;
    B::IndexConfig bic;
    bic.cluster.seed = 1;
    bic.score_bits = 32;
    R::Session rs = R::prefill(q.subspan(0, P * d), k.subspan(0, P * d), v.subspan(0, P * d),
                               R::SubspaceLayout::uniform(d, 8), ric, R::RetrievalConfig{});
    B::Session bs = B::prefill(q.subspan(0, P * d), k.subspan(0, P * d), v.subspan(0, P * d),
                               B::SubspaceLayout::uniform(d, 8), bic, B::RetrievalConfig{}, T);
    const auto rr = R::run_decode(rs, q.subspan(P * d), k.subspan(P * d), v.subspan(P * d), T, true);
    const auto br = B::run_decode(bs, q.subspan(P * d), k.subspan(P * d), v.subspan(P * d), T, true);
    for (std::size_t t = 0; t < T; ++t) {
        CHECK(rr[t].recall && br[t].recall && *rr[t].recall == *br[t].recall, "step %zu recall %.6f vs %.6f", t,
              rr[t].recall.value_or(-1), br[t].recall.value_or(-1));
        double e2 = 0.0, n2 = 0.0;
        for (std::size_t x = 0; x < d; ++x) {
            const double a = rr[t].dense_reference->output[x], b = br[t].dense_reference->output[x];
            e2 += (a - b) * (a - b);
            n2 += a * a;
        }
        CHECK(std::sqrt(e2 / n2) < 1e-6, "step %zu dense output rel err %.3g", t, std::sqrt(e2 / n2));
        CHECK(std::fabs(*rr[t].l2_error - *br[t].l2_error) < 1e-4, "step %zu l2 %.6g vs %.6g", t,
              *rr[t].l2_error, *br[t].l2_error);
    }
    std::printf("dense compare: recall %.4f (step 0), l2 %.3g: done\n", *br[0].recall, *br[0].l2_error);
}

// k_bump (retrieval.cpp:257-263) is fed the worst best-cosine of the LAST
// SEARCH: this query's on searching steps, the last searching query's on
// reuse steps (period > 1). A cosine-dependent K makes any mix-up visible.
// Then a mid-session change of the public Session::cfg (session.hpp:19-31)
// reaches the device session before the next step.
static void kbump_and_cfg(const char* schedule) {
    const std::size_t P = 3000, T = 12, d = 64, m = 8;
    R::SyntheticSpec spec;
    spec.rows = P + T;
    spec.dim = d;
    spec.seed = 41;
    const R::SyntheticWorkload w = R::make_synthetic(spec);
    const std::span<const float> q(w.queries), k(w.keys), v(w.values);
    R::IndexConfig ric;
    ric.cluster.seed = 3;
    ric.cluster.centroids = 16;
    ric.score_bits = 32;
    B::IndexConfig bic;
    bic.cluster.seed = 3;
    bic.cluster.centroids = 16;
    bic.score_bits = 32;
    const auto [rho, period] = R::parse_schedule(schedule);
    auto bump = [](std::size_t kk, double worst) {
        return kk + static_cast<std::size_t>(std::floor(4000.0 * (1.0 - worst)));
    };
    R::RetrievalConfig rrc;
    rrc.keep_ratio = rho;
    rrc.search_period = period;
    rrc.k_bump = bump;
    B::RetrievalConfig brc;
    brc.keep_ratio = rho;
    brc.search_period = period;
    brc.k_bump = bump;
    R::Session rs = R::prefill(q.subspan(0, P * d), k.subspan(0, P * d), v.subspan(0, P * d),
                               R::SubspaceLayout::uniform(d, m), ric, rrc);
    B::Session bs = B::prefill(q.subspan(0, P * d), k.subspan(0, P * d), v.subspan(0, P * d),
                               B::SubspaceLayout::uniform(d, m), bic, brc, T);
    std::size_t diff = 0, bumped = 0;
    for (std::size_t t = 0; t < T; ++t) {
        if (t == 7) {  // public cfg change between steps: window and weights
            rs.cfg.recent_window = 8;
            bs.cfg.recent_window = 8;
            rs.cfg.weights.assign(m, 1.0);
            rs.cfg.weights[2] = 2.5;
            bs.cfg.weights = rs.cfg.weights;
        }
        const auto a = R::decode_step(rs, q.subspan((P + t) * d, d), k.subspan((P + t) * d, d),
                                      v.subspan((P + t) * d, d), false);
        const auto b = B::decode_step(bs, q.subspan((P + t) * d, d), k.subspan((P + t) * d, d),
                                      v.subspan((P + t) * d, d), false);
        diff += a.selected != b.selected || a.k != b.k || a.searched != b.searched;
        bumped += a.k != R::keep_count(rho, P + t);
    }
    CHECK(diff == 0, "k_bump %s: %zu of %zu steps differ", schedule, diff, T);
    CHECK(bumped > 0, "k_bump %s never changed K", schedule);
    // a GQA session serves `group` queries per step: the single-query calls refuse it
    std::vector<float> q4(4 * P * d);
    for (std::size_t r = 0; r < 4; ++r)
        std::copy(q.begin(), q.begin() + P * d, q4.begin() + r * P * d);
    B::Session g4 = B::prefill(q4, k.subspan(0, P * d), v.subspan(0, P * d),
                               B::SubspaceLayout::uniform(d, m), bic, B::RetrievalConfig{}, 4, 4);
    const std::string e = thrown<B::ParameterError>([&] {
        B::decode_step(g4, q.subspan(P * d, d), k.subspan(P * d, d), v.subspan(P * d, d), false);
    });
    CHECK(e.find("GQA group of 4") != std::string::npos, "group refusal: '%s'", e.c_str());
    std::printf("k_bump %s + cfg change: %zu/%zu steps equal, %zu bumped\n", schedule, T - diff, T, bumped);
}

static void errors() {
    const std::size_t d = 16, P = 64;
    std::vector<float> q(P * d, 0.5f), k(P * d, 0.25f), v(P * d, 1.0f);
    // prefill validation (session.cpp:25-44): same class, same message
    {
        std::vector<float> bad(P * d + 3, 0.0f);
        auto a = thrown<R::DimensionError>([&] {
            R::prefill(bad, k, v, R::SubspaceLayout::uniform(d, 4), R::IndexConfig{}, R::RetrievalConfig{});
        });
        auto b = thrown<B::DimensionError>([&] {
            B::prefill(bad, k, v, B::SubspaceLayout::uniform(d, 4), B::IndexConfig{}, B::RetrievalConfig{});
        });
        CHECK(a == b, "prefill width: ref '%s' vs b200 '%s'", a.c_str(), b.c_str());
        std::vector<float> half(P / 2 * d, 0.0f);
        a = thrown<R::ParameterError>([&] {
            R::prefill(q, half, v, R::SubspaceLayout::uniform(d, 4), R::IndexConfig{}, R::RetrievalConfig{});
        });
        b = thrown<B::ParameterError>([&] {
            B::prefill(q, half, v, B::SubspaceLayout::uniform(d, 4), B::IndexConfig{}, B::RetrievalConfig{});
        });
        CHECK(a == b, "prefill counts: ref '%s' vs b200 '%s'", a.c_str(), b.c_str());
    }
    // stream exhaustion (session.cpp:111-116)
    {
        R::IndexConfig ric;
        ric.cluster.centroids = 4;
        B::IndexConfig bic;
        bic.cluster.centroids = 4;
        R::Session rs = R::prefill(q, k, v, R::SubspaceLayout::uniform(d, 4), ric, R::RetrievalConfig{});
        B::Session bs = B::prefill(q, k, v, B::SubspaceLayout::uniform(d, 4), bic, B::RetrievalConfig{}, 8);
        std::vector<float> s3(3 * d, 0.1f);
        const auto a = thrown<R::StreamExhaustedError>([&] { R::run_decode(rs, s3, s3, s3, 5, false); });
        const auto b = thrown<B::StreamExhaustedError>([&] { B::run_decode(bs, s3, s3, s3, 5, false); });
        CHECK(a == b && a.find("step 3 of 5") != std::string::npos, "exhaustion: '%s' vs '%s'",
              a.c_str(), b.c_str());
    }
    // keep_count / h2d closed forms
    CHECK(R::keep_count(0.05, 8192) == B::keep_count(0.05, 8192), "keep_count");
    CHECK(R::h2d_bytes(0.05, 4096, 128, 2, 1) == B::h2d_bytes(0.05, 4096, 128, 2, 1), "h2d_bytes");
    std::printf("errors: done\n");
}

int main() {
    errors();
    dense_compare();
    lifecycle(4096, 12, 128, 8, 2026, "0.05-step-1", true);   // BASELINE config 1
    lifecycle(2000, 10, 64, 8, 7, "0.15-step-4", true);       // period reuse
    lifecycle(1500, 6, 64, 4, 11, "0.05-step-1", false);      // window competes
    kbump_and_cfg("0.05-step-1");
    kbump_and_cfg("0.15-step-4");
    if (failures) {
        std::printf("%d FAILURES\n", failures);
        return 1;
    }
    std::printf("ALL OK\n");
    return 0;
}
