// csattn_b200_shard.hpp — native C++ orchestration of the sequence-sharded
// decode step over the C ABI's shard phases, with
// a pluggable transport: LocalCollectives (several shards in one process, e.g.
// on one GPU) and NcclCollectives (include/csattn_b200_nccl.hpp: one process
// per GPU, NCCL over NVLink/NVSwitch). The same phase order as the Python
// ShardGroup (paper_2604_08584_b200/sharding.py):
//
//   SCAN -> all-reduce(sum) histograms -> BUCKET -> [speculation flag,
//   read asynchronously] -> all-gather buckets -> MARK -> all-gather counts
//   -> EMIT -> all-gather partials -> MERGE -> (on a flagged speculation miss:
//   RESCAN .. MERGE again) -> VICTIM -> all-reduce(min) victims -> INSERT
//
// The union of the shards' selections is exactly the unsharded selection and
// the merged output agrees within 1e-3 (tests/cpp/test_shard.cpp).
// Requirement: every local shard's context enqueues on the SAME CUDA stream
// (csattn_ctx_create(dev, stream)), so phases and collectives are ordered.
#pragma once

#include <cuda_runtime_api.h>

#include <memory>
#include <string>
#include <vector>

#include "csattn_b200.hpp"

namespace csattn_b200 {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Transport between this process's local shards and the other ranks. Buffers
// are device pointers, one per local shard; ops are enqueued on `stream`.
struct Collectives {
    virtual ~Collectives() = default;
    virtual int world() const = 0;
    virtual int rank() const = 0;
    // every local buffer becomes the sum over ALL shards (uint32)
    virtual void all_reduce_sum_u32(csattn_ctx ctx, const std::vector<uint32_t*>& local, uint64_t count) = 0;
    // every local buffer becomes the elementwise min over ALL shards (uint64)
    virtual void all_reduce_min_u64(csattn_ctx ctx, const std::vector<uint64_t*>& local, uint64_t count) = 0;
    // recv[j] (every local shard): all shards' `bytes`, global shard order
    // (rank-major, then local order)
    virtual void all_gather(csattn_ctx ctx, const std::vector<const void*>& local, uint64_t bytes,
                            const std::vector<void*>& recv) = 0;
};

namespace detail {
// local combine: buf[0] = combine(buf[0..L)), then broadcast buf[0]
inline void local_sum_u32(csattn_ctx ctx, const std::vector<uint32_t*>& b, uint64_t n) {
    for (std::size_t j = 1; j < b.size(); ++j) check(csattn_buffer_add_u32(ctx, b[0], b[j], n));
}
inline void local_min_u64(csattn_ctx ctx, const std::vector<uint64_t*>& b, uint64_t n) {
    for (std::size_t j = 1; j < b.size(); ++j) check(csattn_buffer_min_u64(ctx, b[0], b[j], n));
}
template <class T>
inline void local_broadcast(csattn_ctx ctx, const std::vector<T*>& b, uint64_t n) {
    auto st = static_cast<cudaStream_t>(csattn_ctx_stream(ctx));
    for (std::size_t j = 1; j < b.size(); ++j)
        cuda_check(cudaMemcpyAsync(b[j], b[0], n * sizeof(T), cudaMemcpyDeviceToDevice, st), "broadcast");
}
}  // namespace detail

// All shards in this process (world = 1).
struct LocalCollectives : Collectives {
    int world() const override { return 1; }
    int rank() const override { return 0; }
    void all_reduce_sum_u32(csattn_ctx ctx, const std::vector<uint32_t*>& b, uint64_t n) override {
        detail::local_sum_u32(ctx, b, n);
        detail::local_broadcast(ctx, b, n);
    }
    void all_reduce_min_u64(csattn_ctx ctx, const std::vector<uint64_t*>& b, uint64_t n) override {
        detail::local_min_u64(ctx, b, n);
        detail::local_broadcast(ctx, b, n);
    }
    void all_gather(csattn_ctx ctx, const std::vector<const void*>& local, uint64_t bytes,
                    const std::vector<void*>& recv) override {
        auto st = static_cast<cudaStream_t>(csattn_ctx_stream(ctx));
        for (void* r : recv)
            for (std::size_t i = 0; i < local.size(); ++i)
                cuda_check(cudaMemcpyAsync(static_cast<char*>(r) + i * bytes, local[i], bytes,
                                           cudaMemcpyDeviceToDevice, st),
                           "gather");
    }
};

// Shard bounds: tile-aligned key ranges, the last one (owner of appended keys)
// ends at P (sharding.shard_bounds).
inline std::vector<std::pair<uint64_t, uint64_t>> shard_bounds(uint64_t P, uint64_t n_shards) {
    constexpr uint64_t align = 4096;  // select tile
    const uint64_t tiles = (P + align - 1) / align;
    if (n_shards < 1 || n_shards > tiles)
        throw ParameterError(std::to_string(n_shards) + " shards for " + std::to_string(tiles) + " tiles");
    std::vector<std::pair<uint64_t, uint64_t>> b;
    for (uint64_t j = 0; j < n_shards; ++j) {
        const uint64_t lo = (tiles * j) / n_shards * align;
        const uint64_t hi = j + 1 == n_shards ? P : (tiles * (j + 1)) / n_shards * align;
        b.emplace_back(lo, hi);
    }
    return b;
}

// KV-head sharding (c4): rank r owns KV heads {g : g mod world = r}
// (sharding.kv_head_shard); no data-path collective.
inline std::vector<std::size_t> kv_head_shard(std::size_t n_kv_heads, std::size_t world, std::size_t rank) {
    if (world == 0 || rank >= world) throw ParameterError("rank out of range");
    std::vector<std::size_t> g;
    for (std::size_t h = rank; h < n_kv_heads; h += world) g.push_back(h);
    return g;
}

// The shards [first, first + ctxs.size()) of every full session of a layer,
// one local context per shard, decoded as one sequence-sharded step.
class ShardedLayer {
   public:
    ShardedLayer(std::vector<Context*> ctxs, const std::vector<const Session*>& full, uint64_t first_shard,
                 uint64_t n_shards, uint64_t max_decode_steps, Collectives& coll)
        : ctxs_(std::move(ctxs)), coll_(coll), first_(first_shard), n_shards_(n_shards) {
        if (ctxs_.empty() || full.empty()) throw ParameterError("no shards or no sessions");
        stream_ = static_cast<cudaStream_t>(csattn_ctx_stream(ctxs_[0]->handle()));
        for (Context* c : ctxs_)
            if (csattn_ctx_stream(c->handle()) != static_cast<void*>(stream_))
                throw ParameterError("local shard contexts must share one CUDA stream");
        const csattn_session_info in = full[0]->info();
        d_ = in.dim;
        bounds_ = shard_bounds(in.prefill_len, n_shards);
        ns_ = full.size();
        nq_ = 0;
        for (const Session* s : full) nq_ += s->info().group;
        for (std::size_t j = 0; j < ctxs_.size(); ++j) {
            const uint64_t g = first_ + j;
            std::vector<csattn_session> row;
            for (const Session* s : full) {
                csattn_session h = nullptr;
                check(csattn_shard_create(ctxs_[j]->handle(), s->handle(), bounds_[g].first, bounds_[g].second,
                                          g + 1 == n_shards ? 1 : 0, max_decode_steps, &h));
                row.push_back(h);
            }
            shards_.push_back(std::move(row));
        }
        check(csattn_shard_buffer_words(shards_[0][0], &hw_, &bw_, &pf_, &vw_));
        const std::size_t L = ctxs_.size();
        for (std::size_t j = 0; j < L; ++j) {
            Buf b;
            b.ghist = alloc<uint32_t>(nq_ * hw_);
            b.bucket = alloc<uint32_t>(nq_ * bw_);
            b.bucket_all = alloc<uint32_t>(n_shards * nq_ * bw_);
            b.counts = alloc<uint32_t>(nq_ * 2);
            b.counts_all = alloc<uint32_t>(n_shards * nq_ * 2);
            b.partial = alloc<float>(nq_ * pf_);
            b.partial_all = alloc<float>(n_shards * nq_ * pf_);
            b.victim = alloc<uint64_t>(ns_ * vw_);
            b.out = alloc<float>(nq_ * d_);
            b.fail = alloc<uint32_t>(1);
            bufs_.push_back(b);
        }
        cuda_check(cudaMallocHost(&fail_host_, sizeof(uint32_t)), "pinned flag");
        cuda_check(cudaEventCreateWithFlags(&fail_ev_, cudaEventDisableTiming), "event");
    }
    ~ShardedLayer() {
        for (auto& row : shards_)
            for (csattn_session h : row) csattn_session_destroy(h);
        for (void* p : mem_) cudaFree(p);
        if (fail_host_) cudaFreeHost(fail_host_);
        if (fail_ev_) cudaEventDestroy(fail_ev_);
    }
    ShardedLayer(const ShardedLayer&) = delete;
    ShardedLayer& operator=(const ShardedLayer&) = delete;

    uint64_t query_heads() const { return nq_; }
    const std::vector<std::pair<uint64_t, uint64_t>>& bounds() const { return bounds_; }
    // the shard sessions of local shard j (one per full session)
    const std::vector<csattn_session>& shard(std::size_t j) const { return shards_[j]; }
    uint64_t rescans() const { return rescans_; }

    // Keep each local shard's selection (up to k_max per query head) for
    // local_selected(); off by default.
    void enable_selected(uint64_t k_max) {
        k_max_ = k_max;
        for (Buf& b : bufs_) {
            b.sel = alloc<uint32_t>(nq_ * k_max);
            b.nsel = alloc<uint32_t>(nq_);
        }
    }
    // local shard j's ascending selection of query head h in the last step
    std::vector<uint32_t> local_selected(std::size_t j, std::size_t h) const {
        uint32_t n = 0;
        cuda_check(cudaStreamSynchronize(stream_), "sync");
        cuda_check(cudaMemcpy(&n, bufs_[j].nsel + h, 4, cudaMemcpyDeviceToHost), "nsel");
        std::vector<uint32_t> v(n);
        if (n) cuda_check(cudaMemcpy(v.data(), bufs_[j].sel + h * k_max_, n * 4, cudaMemcpyDeviceToHost), "sel");
        return v;
    }

    // One decode step of the layer. Device pointers: q (nq x d), keys/values
    // (n_sessions x d), out (nq x d). selected (nullable, nq x sel_stride):
    // this process's local shards' selections are NOT merged here; use
    // csattn_shard_io.n_selected of each shard for that.
    void decode_step(const float* q, const float* keys, const float* values, float* out) {
        const std::size_t L = ctxs_.size();
        std::vector<csattn_shard_io> io(L);
        for (std::size_t j = 0; j < L; ++j) {
            csattn_shard_io& x = io[j];
            x = csattn_shard_io{};
            const Buf& b = bufs_[j];
            x.q = q;
            x.new_keys = keys;
            x.new_values = values;
            x.ghist = b.ghist;
            x.bucket = b.bucket;
            x.bucket_all = b.bucket_all;
            x.counts = b.counts;
            x.counts_all = b.counts_all;
            x.partial = b.partial;
            x.partial_all = b.partial_all;
            x.out = b.out;
            x.victim = reinterpret_cast<unsigned long long*>(b.victim);
            x.spec_fail = b.fail;
            if (b.sel) {
                x.selected = b.sel;
                x.n_selected = b.nsel;
                x.sel_stride = k_max_;
            }
            x.shard_index = static_cast<uint32_t>(first_ + j);
            x.n_shards = static_cast<uint32_t>(n_shards_);
            cuda_check(cudaMemsetAsync(b.fail, 0, 4, stream_), "flag");
        }
        auto run = [&](int32_t phase) {
            for (std::size_t j = 0; j < L; ++j)
                check(csattn_shard_step(ctxs_[j]->handle(), ns_, shards_[j].data(), phase, &io[j]));
        };
        csattn_ctx c0 = ctxs_[0]->handle();
        auto sum_hist = [&] {
            std::vector<uint32_t*> v;
            for (Buf& b : bufs_) v.push_back(b.ghist);
            coll_.all_reduce_sum_u32(c0, v, nq_ * hw_);
        };
        auto gather = [&](auto member, auto member_all, uint64_t bytes) {
            std::vector<const void*> loc;
            std::vector<void*> rec;
            for (Buf& b : bufs_) {
                loc.push_back(b.*member);
                rec.push_back(b.*member_all);
            }
            coll_.all_gather(c0, loc, bytes, rec);
        };
        auto select_tail = [&] {
            gather(&Buf::bucket, &Buf::bucket_all, nq_ * bw_ * 4);
            run(CSATTN_SHARD_MARK);
            gather(&Buf::counts, &Buf::counts_all, nq_ * 2 * 4);
            run(CSATTN_SHARD_EMIT);
            gather(&Buf::partial, &Buf::partial_all, nq_ * pf_ * 4);
            run(CSATTN_SHARD_MERGE);
        };
        run(CSATTN_SHARD_SCAN);
        sum_hist();
        run(CSATTN_SHARD_BUCKET);
        {  // speculation miss anywhere? read asynchronously after MERGE is queued
            std::vector<uint32_t*> f;
            for (Buf& b : bufs_) f.push_back(b.fail);
            coll_.all_reduce_sum_u32(c0, f, 1);
            cuda_check(cudaMemcpyAsync(fail_host_, bufs_[0].fail, 4, cudaMemcpyDeviceToHost, stream_), "flag");
            cuda_check(cudaEventRecord(fail_ev_, stream_), "flag event");
        }
        select_tail();
        cuda_check(cudaEventSynchronize(fail_ev_), "flag wait");
        if (*fail_host_) {  // every shard saw the same global histogram: all rescan
            ++rescans_;
            for (Buf& b : bufs_) cuda_check(cudaMemsetAsync(b.fail, 0, 4, stream_), "flag");
            run(CSATTN_SHARD_RESCAN);
            sum_hist();
            run(CSATTN_SHARD_BUCKET);
            select_tail();
        }
        run(CSATTN_SHARD_VICTIM);
        {
            std::vector<uint64_t*> v;
            for (Buf& b : bufs_) v.push_back(b.victim);
            coll_.all_reduce_min_u64(c0, v, ns_ * vw_);
        }
        run(CSATTN_SHARD_INSERT);
        cuda_check(cudaMemcpyAsync(out, bufs_[0].out, nq_ * d_ * 4, cudaMemcpyDeviceToDevice, stream_), "out");
    }

   private:
    struct Buf {
        uint32_t *ghist, *bucket, *bucket_all, *counts, *counts_all, *fail;
        uint32_t* sel = nullptr;
        uint32_t* nsel = nullptr;
        float *partial, *partial_all, *out;
        uint64_t* victim;
    };
    template <class T>
    T* alloc(uint64_t n) {
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T)), "cudaMalloc");
        cuda_check(cudaMemset(p, 0, std::max<uint64_t>(n, 1) * sizeof(T)), "cudaMemset");
        mem_.push_back(p);
        return static_cast<T*>(p);
    }
    std::vector<Context*> ctxs_;
    Collectives& coll_;
    uint64_t first_, n_shards_, ns_ = 0, nq_ = 0, d_ = 0;
    uint64_t hw_ = 0, bw_ = 0, pf_ = 0, vw_ = 0;
    std::vector<std::pair<uint64_t, uint64_t>> bounds_;
    std::vector<std::vector<csattn_session>> shards_;
    std::vector<Buf> bufs_;
    std::vector<void*> mem_;
    cudaStream_t stream_ = nullptr;
    uint32_t* fail_host_ = nullptr;
    cudaEvent_t fail_ev_ = nullptr;
    uint64_t rescans_ = 0;
    uint64_t k_max_ = 0;
};

}  // namespace csattn_b200
