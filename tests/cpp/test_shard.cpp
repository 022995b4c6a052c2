// test_shard.cpp — the native C++ sequence-sharded decode
// (include/csattn_b200_shard.hpp) against the unsharded sessions it came from,
// with both transports: LocalCollectives (3 shards in one process) and
// NcclCollectives (a real NCCL communicator; one rank here since the test box
// has one GPU, so NCCL's all-reduce / all-gather kernels run on the step's
// stream with 2 local shards). Checks per step: the union of the shards'
// selections equals the unsharded selection exactly, outputs within 1e-3;
// after the steps, the union of the shards' tables equals the unsharded
// tables. TEST INFRASTRUCTURE (run by tests/test_cpp_facade.py on a B200).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <tuple>
#include <vector>

#include "csattn/synthetic.hpp"  // reference generator (-Dcsattn=csattn_ref)
#include "csattn_b200_nccl.hpp"

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

struct Tables {
    std::vector<uint32_t> lens;
    std::vector<std::vector<std::pair<float, uint32_t>>> ent;  // TopList order
};
static Tables export_tables(csattn_session s) {
    csattn_session_info in{};
    B::check(csattn_session_info_get(s, &in));
    const std::size_t T = in.subspaces * in.centroids, L = std::max<std::size_t>(in.list_capacity, 1);
    std::vector<uint32_t> lens(T), idx(T * L);
    std::vector<float> sc(T * L);
    B::check(csattn_session_export(s, lens.data(), idx.data(), sc.data(), L, nullptr));
    Tables t;
    t.lens = lens;
    t.ent.resize(T);
    for (std::size_t x = 0; x < T; ++x)
        for (uint32_t r = 0; r < lens[x]; ++r) t.ent[x].push_back({sc[x * L + r], idx[x * L + r]});
    return t;
}

static void run(const char* name, int local_shards, bool nccl) {
    std::printf("case: %s (%d local shards)\n", name, local_shards);
    const std::size_t P = 16384, T = 6, d = 64, m = 4, n_kv = 2, group = 2;
    cudaStream_t st;
    B::cuda_check(cudaStreamCreate(&st), "stream");
    std::vector<std::unique_ptr<B::Context>> ctxs;
    for (int j = 0; j < local_shards; ++j) ctxs.push_back(std::make_unique<B::Context>(0, st));
    B::Context control_ctx(0, st);
    // two KV-head sessions (GQA 2) from the reference generator
    std::vector<R::SyntheticWorkload> w;
    for (std::size_t g = 0; g < n_kv; ++g) {
        R::SyntheticSpec spec;
        spec.rows = P + T;
        spec.dim = d;
        spec.seed = 900 + g;
        w.push_back(R::make_synthetic(spec));
    }
    B::IndexConfig ic;
    ic.alpha = 0.25;
    ic.cluster.centroids = 16;
    ic.cluster.seed = 3;
    ic.score_bits = 32;
    B::RetrievalConfig rc;
    rc.keep_ratio = 0.05;
    rc.recent_window = 16;
    std::vector<B::Session> full, control;
    for (std::size_t g = 0; g < n_kv; ++g) {
        std::vector<float> pooled;
        for (std::size_t r = 0; r < group; ++r) pooled.insert(pooled.end(), w[g].queries.begin(), w[g].queries.begin() + P * d);
        full.push_back(B::prefill(pooled, {w[g].keys.data(), P * d}, {w[g].values.data(), P * d},
                                  B::SubspaceLayout::uniform(d, m), ic, rc, T, group, control_ctx));
    }
    for (auto& s : full) control.push_back(s.fork(T));
    std::vector<const B::Session*> fp;
    for (auto& s : full) fp.push_back(&s);
    std::vector<B::Context*> cp;
    for (auto& c : ctxs) cp.push_back(c.get());

    B::LocalCollectives local;
    std::unique_ptr<B::NcclCollectives> nc;
    if (nccl) {
        ncclUniqueId id;
        B::nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
        nc.reset(B::NcclCollectives::init(id, 1, 0));
    }
    B::Collectives& coll = nccl ? static_cast<B::Collectives&>(*nc) : static_cast<B::Collectives&>(local);
    B::ShardedLayer layer(cp, fp, 0, local_shards, T, coll);
    const std::size_t nq = n_kv * group;
    const uint64_t kmax = B::keep_count(0.05, P + T);
    layer.enable_selected(kmax);
    float *dq, *dk, *dv, *dout;
    B::cuda_check(cudaMalloc(&dq, nq * d * 4), "q");
    B::cuda_check(cudaMalloc(&dk, n_kv * d * 4), "k");
    B::cuda_check(cudaMalloc(&dv, n_kv * d * 4), "v");
    B::cuda_check(cudaMalloc(&dout, nq * d * 4), "out");
    std::vector<csattn_session> ch;
    for (auto& s : control) ch.push_back(s.handle());
    for (std::size_t t = 0; t < T; ++t) {
        std::vector<float> q(nq * d), k(n_kv * d), v(n_kv * d);
        for (std::size_t g = 0; g < n_kv; ++g) {
            for (std::size_t r = 0; r < group; ++r)
                std::copy_n(w[g].queries.begin() + (P + t) * d, d, q.begin() + (g * group + r) * d);
            std::copy_n(w[g].keys.begin() + (P + t) * d, d, k.begin() + g * d);
            std::copy_n(w[g].values.begin() + (P + t) * d, d, v.begin() + g * d);
        }
        B::cuda_check(cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice), "q");
        B::cuda_check(cudaMemcpy(dk, k.data(), k.size() * 4, cudaMemcpyHostToDevice), "k");
        B::cuda_check(cudaMemcpy(dv, v.data(), v.size() * 4, cudaMemcpyHostToDevice), "v");
        layer.decode_step(dq, dk, dv, dout);
        std::vector<float> out(nq * d), ref(nq * d);
        B::cuda_check(cudaMemcpyAsync(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost, st), "out");
        B::cuda_check(cudaStreamSynchronize(st), "sync");
        const uint64_t K = B::keep_count(0.05, P + t);
        std::vector<uint32_t> sel(nq * K);
        B::check(csattn_decode_batch(control_ctx.handle(), n_kv, ch.data(), q.data(), k.data(), v.data(), ref.data(),
                                     sel.data(), K, CSATTN_HOST_BUFFERS));
        for (std::size_t h = 0; h < nq; ++h) {
            std::vector<uint32_t> uni;
            for (int j = 0; j < local_shards; ++j) {
                const auto s = layer.local_selected(j, h);
                uni.insert(uni.end(), s.begin(), s.end());
            }
            const std::vector<uint32_t> want(sel.begin() + h * K, sel.begin() + (h + 1) * K);
            CHECK(uni == want, "step %zu head %zu: union of shard selections != unsharded (%zu vs %zu)", t, h,
                  uni.size(), want.size());
            double e = 0, n = 0;
            for (std::size_t x = 0; x < d; ++x) {
                e += (out[h * d + x] - ref[h * d + x]) * (out[h * d + x] - ref[h * d + x]);
                n += ref[h * d + x] * ref[h * d + x];
            }
            CHECK(std::sqrt(e / n) <= 1e-3, "step %zu head %zu: rel err %.3g", t, h, std::sqrt(e / n));
        }
    }
    for (std::size_t g = 0; g < n_kv; ++g) {  // tables after T inserts
        const Tables want = export_tables(control[g].handle());
        Tables uni;
        uni.ent.resize(want.ent.size());
        for (int j = 0; j < local_shards; ++j) {
            const Tables part = export_tables(layer.shard(j)[g]);
            for (std::size_t x = 0; x < part.ent.size(); ++x)
                uni.ent[x].insert(uni.ent[x].end(), part.ent[x].begin(), part.ent[x].end());
        }
        bool same = true;
        for (std::size_t x = 0; x < want.ent.size(); ++x) {
            auto& e = uni.ent[x];
            std::sort(e.begin(), e.end(), [](auto& a, auto& b) { return a.first != b.first ? a.first > b.first : a.second < b.second; });
            same &= e == want.ent[x];
        }
        CHECK(same, "session %zu: union of shard tables != unsharded tables", g);
    }
    std::printf("       rescans %llu\n", static_cast<unsigned long long>(layer.rescans()));
    cudaFree(dq);
    cudaFree(dk);
    cudaFree(dv);
    cudaFree(dout);
}

int main() {
    try {
        run("local transport", 3, false);
        run("NCCL transport (1 rank, NCCL collectives on the step stream)", 2, true);
    } catch (const std::exception& e) {
        std::printf("FAIL: threw %s\n", e.what());
        ++failures;
    }
    std::printf("%d checks, %d failures\n", checks, failures);
    if (failures == 0) std::printf("ALL OK\n");
    return failures ? 1 : 0;
}
