// kmeans.h — one exact spherical k-means job (one subspace of one session).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace csa {

struct KmeansJob {
    const float* q;                 // n_total x d query rows; subspace slice at `off`
    uint32_t n_total, d, off, w;
    uint32_t k, iters, batch_cfg, pad;
    double tol;
    const unsigned long long* rng;  // raw mt19937_64 outputs, reference order
    float* train;                   // n_total * w   normalized non-zero rows
    double* best;                   // n_total
    double* run;                    // n_total
    uint32_t* assign;               // 2 * n_total
    double* sums;                   // k * w
    uint32_t* counts;               // k
    float* cent;                    // out: k * w
    int* status;                    // 0 ok, 4 DataError, 9 PropertyError
    uint32_t* info;                 // [0] usable rows n, [1] reseeded
};

constexpr uint32_t KM_MAX_KW = 4096;

size_t kmeans_rng_draws(uint32_t k, uint32_t iters, uint32_t n_total, uint32_t batch_cfg);
cudaError_t launch_kmeans(const KmeansJob* jobs, uint32_t njobs, cudaStream_t st);

}  // namespace csa
