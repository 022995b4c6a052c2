// dense.cu — the dense oracle on the device: masked or
// full dense_attention (core.cpp:118-169) and dense_topk (core.cpp:171-192)
// over a session's KV rows, for recall@K / l2_error at 128K-1M keys where the
// CPU oracle is too slow. Not on the decode hot path.
//
//   dense_dot_kernel     one thread per row: the reference's sequential fp64
//                        dot (float x float products are exact in fp64, so an
//                        FMA chain equals its mul-then-add), optionally scaled
//                        by 1/sqrt(d) (dense_attention) — bit-identical to dot()
//   dense_max_kernel     max logit (order-free)
//   dense_exp_kernel     e_r = exp(l_r - max) in fp64, per-CTA partial sums
//   dense_out_kernel     w_r = e_r / denom -> f32 weights (mask order); per
//                        CTA and dimension the fp64 sum of w_r * v_r[j]
//   dense_fin_kernel     partials summed in CTA order -> f32 output
//   dense_topk           keys = descending-ordered score bits, values = row;
//                        a stable radix sort keeps equal scores in row order
//                        (the reference's "lower index first"), the first K
//                        rows sorted ascending
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace csa {

constexpr int DN_THREADS = 256;
constexpr int DN_ROWS = 1024;  // rows per CTA in the exp / output passes

__device__ __forceinline__ const float* dn_row(const float* pre, const float* tail, uint32_t P, uint32_t i,
                                               uint32_t d) {
    return i < P ? pre + static_cast<size_t>(i) * d : tail + static_cast<size_t>(i - P) * d;
}

__global__ void dense_dot_kernel(const float* __restrict__ q, const float* __restrict__ kpre,
                                 const float* __restrict__ ktail, uint32_t P, const uint32_t* __restrict__ mask,
                                 uint32_t n, uint32_t d, double scale, double* __restrict__ out) {
    extern __shared__ float qs[];
    for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) qs[t] = q[t];
    __syncthreads();
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t i = mask ? mask[r] : r;
    const float* k = dn_row(kpre, ktail, P, i, d);
    double s = 0.0;
    for (uint32_t t = 0; t < d; ++t) s = fma(static_cast<double>(qs[t]), static_cast<double>(__ldg(k + t)), s);
    out[r] = scale != 0.0 ? s * scale : s;
}

__global__ void dense_max_kernel(const double* __restrict__ l, uint32_t n, double* __restrict__ mx) {
    __shared__ double red[DN_THREADS];
    double m = -INFINITY;
    for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) m = fmax(m, l[r]);
    red[threadIdx.x] = m;
    __syncthreads();
    for (int o = DN_THREADS / 2; o; o >>= 1) {
        if (static_cast<int>(threadIdx.x) < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *mx = red[0];
}

// e_r = exp(l_r - max) in place; partial[c] = sum over this CTA's rows (row order)
__global__ void dense_exp_kernel(double* __restrict__ l, uint32_t n, const double* __restrict__ mx,
                                 double* __restrict__ partial) {
    __shared__ double red[DN_THREADS];
    const uint32_t r0 = blockIdx.x * DN_ROWS;
    double s = 0.0;
    for (uint32_t r = r0 + threadIdx.x; r < min(n, r0 + DN_ROWS); r += blockDim.x) {
        const double e = exp(l[r] - *mx);
        l[r] = e;
        s += e;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = DN_THREADS / 2; o; o >>= 1) {
        if (static_cast<int>(threadIdx.x) < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// weights (f32, mask order) and per-CTA fp64 partial outputs [cta][d]
__global__ void dense_out_kernel(const double* __restrict__ e, uint32_t n, const double* __restrict__ psum,
                                 uint32_t nct, const float* __restrict__ vpre, const float* __restrict__ vtail,
                                 uint32_t P, const uint32_t* __restrict__ mask, uint32_t d,
                                 float* __restrict__ weights, double* __restrict__ pout) {
    __shared__ double denom_s;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (uint32_t c = 0; c < nct; ++c) s += psum[c];
        denom_s = s;
    }
    __syncthreads();
    const double denom = denom_s;
    const uint32_t r0 = blockIdx.x * DN_ROWS, r1 = min(n, r0 + DN_ROWS);
    if (weights)
        for (uint32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) weights[r] = static_cast<float>(e[r] / denom);
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
        double a = 0.0;
        for (uint32_t r = r0; r < r1; ++r) {
            const uint32_t i = mask ? __ldg(mask + r) : r;
            // mul then add, as the reference's acc[j] += w * v[j] (no contraction)
            a = __dadd_rn(a, __dmul_rn(e[r] / denom, static_cast<double>(__ldg(dn_row(vpre, vtail, P, i, d) + j))));
        }
        pout[static_cast<size_t>(blockIdx.x) * d + j] = a;
    }
}

__global__ void dense_fin_kernel(const double* __restrict__ pout, uint32_t nct, uint32_t d,
                                 float* __restrict__ out) {
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
        double a = 0.0;
        for (uint32_t c = 0; c < nct; ++c) a += pout[static_cast<size_t>(c) * d + j];
        out[j] = static_cast<float>(a);
    }
}

__global__ void dense_keys_kernel(const double* __restrict__ s, uint32_t n, unsigned long long* __restrict__ keys,
                                  uint32_t* __restrict__ rows) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double v = s[r] == 0.0 ? 0.0 : s[r];  // -0.0 == +0.0 in the reference's comparison
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned long long asc = (u >> 63) ? ~u : (u | (1ull << 63));
    keys[r] = ~asc;  // ascending key = descending score
    rows[r] = r;
}

size_t dense_scratch_bytes(uint32_t n, uint32_t d) {
    const uint32_t nct = div_up(n, DN_ROWS);
    size_t sort1 = 0, sort2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort1, static_cast<const unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<int>(n));
    cub::DeviceRadixSort::SortKeys(nullptr, sort2, static_cast<const uint32_t*>(nullptr),
                                   static_cast<uint32_t*>(nullptr), static_cast<int>(n));
    const size_t a = 256 + static_cast<size_t>(n) * 8 + 8 + static_cast<size_t>(nct) * 8 +
                     static_cast<size_t>(nct) * d * 8;
    // topk carves: scores, keys, sorted keys (8 B each), rows, sorted rows (4 B each), each 256-aligned
    const size_t b = static_cast<size_t>(n) * (8 + 8 + 8 + 4 + 4) + 5 * 256 + std::max(sort1, sort2) + 1024;
    return ((std::max(a, b) + 4096) + 255) & ~static_cast<size_t>(255);  // callers place buffers after it
}

static char* carve(char*& p, size_t bytes) {
    char* at = p;
    p += (bytes + 255) & ~static_cast<size_t>(255);
    return at;
}

cudaError_t launch_dense_attention(const float* q, const float* kpre, const float* ktail, const float* vpre,
                                   const float* vtail, uint32_t P, const uint32_t* mask, uint32_t n,
                                   uint32_t d, float* out, float* weights, void* scratch, cudaStream_t st) {
    const uint32_t nct = div_up(n, DN_ROWS);
    char* p = static_cast<char*>(scratch);
    double* l = reinterpret_cast<double*>(carve(p, static_cast<size_t>(n) * 8));
    double* mx = reinterpret_cast<double*>(carve(p, 8));
    double* ps = reinterpret_cast<double*>(carve(p, static_cast<size_t>(nct) * 8));
    double* po = reinterpret_cast<double*>(carve(p, static_cast<size_t>(nct) * d * 8));
    const double scale = 1.0 / sqrt(static_cast<double>(d));
    dense_dot_kernel<<<div_up(n, DN_THREADS), DN_THREADS, d * 4, st>>>(q, kpre, ktail, P, mask, n, d, scale, l);
    dense_max_kernel<<<1, DN_THREADS, 0, st>>>(l, n, mx);
    dense_exp_kernel<<<nct, DN_THREADS, 0, st>>>(l, n, mx, ps);
    dense_out_kernel<<<nct, 128, 0, st>>>(l, n, ps, nct, vpre, vtail, P, mask, d, weights, po);
    dense_fin_kernel<<<1, 128, 0, st>>>(po, nct, d, out);
    return cudaGetLastError();
}

cudaError_t launch_dense_topk(const float* q, const float* kpre, const float* ktail, uint32_t P, uint32_t n,
                              uint32_t d, uint32_t k, uint32_t* out, void* scratch, size_t scratch_bytes,
                              cudaStream_t st) {
    char* p = static_cast<char*>(scratch);
    double* s = reinterpret_cast<double*>(carve(p, static_cast<size_t>(n) * 8));
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(carve(p, static_cast<size_t>(n) * 8));
    unsigned long long* keys2 = reinterpret_cast<unsigned long long*>(carve(p, static_cast<size_t>(n) * 8));
    uint32_t* rows = reinterpret_cast<uint32_t*>(carve(p, static_cast<size_t>(n) * 4));
    uint32_t* rows2 = reinterpret_cast<uint32_t*>(carve(p, static_cast<size_t>(n) * 4));
    void* temp = carve(p, 0);
    const size_t used = static_cast<size_t>(p - static_cast<char*>(scratch));
    size_t tb = scratch_bytes > used ? scratch_bytes - used : 0;
    dense_dot_kernel<<<div_up(n, DN_THREADS), DN_THREADS, d * 4, st>>>(q, kpre, ktail, P, nullptr, n, d, 0.0, s);
    dense_keys_kernel<<<div_up(n, DN_THREADS), DN_THREADS, 0, st>>>(s, n, keys, rows);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys2, rows, rows2, static_cast<int>(n), 0, 64, st);
    if (e != cudaSuccess) return e;
    // the K best rows, ascending
    e = cub::DeviceRadixSort::SortKeys(temp, tb, rows2, out, static_cast<int>(k), 0, 32, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace csa
