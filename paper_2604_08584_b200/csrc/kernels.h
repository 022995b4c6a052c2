// kernels.h — host-callable launchers of the sm_100a kernels (csrc/*.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace csa {

// route.cu: centroid routing + per-rank gather plan, one CTA per problem
cudaError_t launch_route(const DecodeProblem* probs, RoutePlan* plans, uint32_t nprob, uint32_t cs,
                         uint32_t kpc, cudaStream_t st);

// select.cu: gather + top-K, one cluster per problem
size_t select_smem_bytes(uint32_t kpc);
cudaError_t launch_select(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                          uint32_t kpc, uint32_t cs, cudaStream_t st);

// attend.cu: split-K sparse attention over the selected rows, ATT_ROWS per CTA
constexpr uint32_t ATT_ROWS = 128;
cudaError_t launch_attend(const DecodeProblem* probs, const uint32_t* chunk_prob,
                          const uint32_t* chunk_base, uint32_t nchunks, float* part,
                          uint32_t* counters, uint32_t d, cudaStream_t st);

// insert.cu: append + streaming insert, one CTA per session
cudaError_t launch_insert(const InsertProblem* probs, uint32_t nprob, cudaStream_t st);

// build.cu: exact fp64 centroid x key scores and top-L tables
//   scores: T x P floats scratch
cudaError_t launch_build_scores(const SessionDev* s_dev, const SessionDev& s_host, float* scores,
                                cudaStream_t st);
cudaError_t launch_build_lists(const SessionDev* s_dev, const SessionDev& s_host,
                               const float* scores, cudaStream_t st);


}  // namespace csa
