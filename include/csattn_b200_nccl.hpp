// csattn_b200_nccl.hpp — NCCL transport for the sequence-sharded decode step
// (csattn_b200_shard.hpp): one process per GPU, the ranks' communicator over
// NVLink 5 / NVSwitch. Histograms and speculation flags are summed with
// ncclAllReduce(uint32, sum), eviction victims with ncclAllReduce(uint64, min)
// (packed (score, key) eviction keys, unsigned order), buckets / counts /
// attention partials are gathered with ncclAllGather in rank-major order (=
// global shard order, shard = rank * local + j). Every message is a few KB to
// a few hundred KB per layer: latency-bound, so they run on the step's own
// stream, back to back with the phase kernels (no host round trip except the
// asynchronously read speculation flag). Link with -lnccl.
#pragma once

#include <nccl.h>

#include <string>
#include <vector>

#include "csattn_b200_shard.hpp"

namespace csattn_b200 {

inline void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + ncclGetErrorString(r));
}

class NcclCollectives : public Collectives {
   public:
    // An initialised communicator of `world` ranks (this rank's GPU current).
    NcclCollectives(ncclComm_t comm, int world, int rank) : comm_(comm), world_(world), rank_(rank) {}
    // Convenience: ncclCommInitRank from a unique id the ranks exchanged out of
    // band (rank 0 calls ncclGetUniqueId). Owns and destroys the communicator.
    static NcclCollectives* init(const ncclUniqueId& id, int world, int rank) {
        ncclComm_t c = nullptr;
        nccl_check(ncclCommInitRank(&c, world, id, rank), "ncclCommInitRank");
        auto* n = new NcclCollectives(c, world, rank);
        n->own_ = true;
        return n;
    }
    ~NcclCollectives() override {
        if (own_ && comm_) ncclCommDestroy(comm_);
        if (stage_) cudaFree(stage_);
    }
    int world() const override { return world_; }
    int rank() const override { return rank_; }

    void all_reduce_sum_u32(csattn_ctx ctx, const std::vector<uint32_t*>& b, uint64_t n) override {
        detail::local_sum_u32(ctx, b, n);
        nccl_check(ncclAllReduce(b[0], b[0], n, ncclUint32, ncclSum, comm_, stream(ctx)), "all-reduce sum");
        detail::local_broadcast(ctx, b, n);
    }
    void all_reduce_min_u64(csattn_ctx ctx, const std::vector<uint64_t*>& b, uint64_t n) override {
        detail::local_min_u64(ctx, b, n);
        nccl_check(ncclAllReduce(b[0], b[0], n, ncclUint64, ncclMin, comm_, stream(ctx)), "all-reduce min");
        detail::local_broadcast(ctx, b, n);
    }
    void all_gather(csattn_ctx ctx, const std::vector<const void*>& local, uint64_t bytes,
                    const std::vector<void*>& recv) override {
        cudaStream_t st = stream(ctx);
        const uint64_t L = local.size();
        // this rank's shards packed contiguously, then one all-gather: the
        // result is rank-major = global shard order
        ensure_stage(L * bytes);
        for (uint64_t j = 0; j < L; ++j)
            cuda_check(cudaMemcpyAsync(static_cast<char*>(stage_) + j * bytes, local[j], bytes,
                                       cudaMemcpyDeviceToDevice, st),
                       "gather pack");
        nccl_check(ncclAllGather(stage_, recv[0], L * bytes, ncclUint8, comm_, st), "all-gather");
        for (uint64_t j = 1; j < recv.size(); ++j)
            cuda_check(cudaMemcpyAsync(recv[j], recv[0], static_cast<size_t>(world_) * L * bytes,
                                       cudaMemcpyDeviceToDevice, st),
                       "gather copy");
    }

   private:
    static cudaStream_t stream(csattn_ctx ctx) { return static_cast<cudaStream_t>(csattn_ctx_stream(ctx)); }
    void ensure_stage(uint64_t bytes) {
        if (bytes <= stage_bytes_) return;
        if (stage_) cudaFree(stage_);
        cuda_check(cudaMalloc(&stage_, bytes), "gather stage");
        stage_bytes_ = bytes;
    }
    ncclComm_t comm_ = nullptr;
    int world_ = 1, rank_ = 0;
    bool own_ = false;
    void* stage_ = nullptr;
    uint64_t stage_bytes_ = 0;
};

}  // namespace csattn_b200
