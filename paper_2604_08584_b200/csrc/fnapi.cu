// fnapi.cu — device kernels behind the reference's function-level API
// (index.hpp / retrieval.hpp free functions on host value types), used by the
// C++ facade when a caller works with CsIndex / KvStore values instead of a
// device Session. Not on the decode hot path (the Session path is), but the
// arithmetic is the same bit-exact fp64 the hot-path kernels use:
//
//   score_multi_kernel   score_keys (index.cpp:68-91) and streaming_insert's
//                        scoring (retrieval.cpp:272-301): for every (centroid
//                        j, key i) the sequential fp64 FMA chain over the
//                        centroid's subspace (float x float products are exact
//                        in fp64, so FMA = mul-then-add). normalize mode 1
//                        divides by the slice norm (score_keys), mode 2 scores
//                        the l2_normalize'd slice (streaming_insert), zero
//                        slices score 0.
//   reduce_lists_kernel  reduce_by_key (retrieval.cpp:111-148): lists in
//                        gathered order, each list's keys are unique, so one
//                        CTA adds a whole list in parallel and syncs between
//                        lists — every key's fp64 sum runs in list order,
//                        starting from 0.0; source counts alongside.
//   toplist keys + sort  TopList::from_scores (index.cpp:46-62): one 64-bit key
//                        per score, ordered(score) << 32 | ~index, radix-sorted
//                        descending: (score desc, index asc), the first L kept.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace csa {

__global__ void score_multi_kernel(const float* __restrict__ cent, const uint32_t* __restrict__ coff,
                                   const uint32_t* __restrict__ kof, const uint32_t* __restrict__ wid,
                                   uint32_t ncent, const float* __restrict__ keys, uint32_t n, uint32_t d,
                                   int mode, float* __restrict__ out, double* __restrict__ out64) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t j = blockIdx.y;
    if (i >= n || j >= ncent) return;
    const float* c = cent + coff[j];
    const float* k = keys + static_cast<size_t>(i) * d + kof[j];
    const uint32_t w = wid[j];
    double s = 0.0;
    if (mode == 2) {  // l2_normalize (core.cpp:109-116) in f32 storage, then dot
        double n2 = 0.0;
        for (uint32_t t = 0; t < w; ++t) n2 = __fma_rn((double)k[t], (double)k[t], n2);
        if (n2 != 0.0) {
            const double inv = 1.0 / sqrt(n2);
            for (uint32_t t = 0; t < w; ++t) {
                const float kn = __double2float_rn(__dmul_rn((double)k[t], inv));
                s = __fma_rn((double)c[t], (double)kn, s);
            }
        }
    } else {
        for (uint32_t t = 0; t < w; ++t) s = __fma_rn((double)c[t], (double)k[t], s);
        if (mode == 1) {  // score_keys' normalize_keys: s / |slice|, zero slice -> 0
            double n2 = 0.0;
            for (uint32_t t = 0; t < w; ++t) n2 = __fma_rn((double)k[t], (double)k[t], n2);
            s = n2 == 0.0 ? 0.0 : __ddiv_rn(s, sqrt(n2));
        }
    }
    if (out) out[static_cast<size_t>(j) * n + i] = __double2float_rn(s);
    if (out64) out64[static_cast<size_t>(j) * n + i] = s;  // centroid_scores: unrounded
}

constexpr unsigned long long FN_ABSENT = 0x7ff4deadbeef0000ull;

// one CTA: acc[key] over [0, nkeys) starts absent; list l's entries (unique
// keys) add w_l * double(score) in parallel, lists in order
__global__ void reduce_lists_kernel(uint32_t nl, const uint64_t* __restrict__ off,
                                    const uint32_t* __restrict__ idx, const float* __restrict__ sc,
                                    const double* __restrict__ w, double* __restrict__ acc,
                                    uint32_t* __restrict__ cnt, uint32_t nkeys) {
    for (uint32_t i = threadIdx.x; i < nkeys; i += blockDim.x) {
        acc[i] = __longlong_as_double(static_cast<long long>(FN_ABSENT));
        cnt[i] = 0;
    }
    __syncthreads();
    for (uint32_t l = 0; l < nl; ++l) {
        const double wl = w[l];
        for (uint64_t e = off[l] + threadIdx.x; e < off[l + 1]; e += blockDim.x) {
            const uint32_t k = idx[e];
            const double x = __dmul_rn(wl, static_cast<double>(sc[e]));
            const double o = acc[k];
            const bool absent = static_cast<unsigned long long>(__double_as_longlong(o)) == FN_ABSENT;
            acc[k] = __dadd_rn(absent ? 0.0 : o, x);
            cnt[k] += 1;
        }
        __syncthreads();
    }
}

__global__ void toplist_keys_kernel(const float* __restrict__ s, uint32_t n,
                                    unsigned long long* __restrict__ keys) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t u = __float_as_uint(s[i]);
    if ((u << 1) == 0) u = 0;  // -0.0 == +0.0 (the comparison of index.cpp:52-56)
    const uint32_t o = (u >> 31) ? ~u : (u | 0x80000000u);
    keys[i] = (static_cast<unsigned long long>(o) << 32) | static_cast<uint32_t>(~i);
}

__global__ void buf_add_u32_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] += src[i];
}
__global__ void buf_min_u64_kernel(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src,
                                   uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i] < dst[i] ? src[i] : dst[i];
}

// Up to 4 (src, dst, bytes) copies in one launch: the decode step's inputs
// read straight from pinned host memory over the host link (one launch
// instead of one DMA call per buffer; the host-side cost of a copy call is
// larger than the transfer of these few hundred KB). 16-byte granules when
// every pointer and size allows, else 4-byte.
struct CopySegs {
    const void* src[4];
    void* dst[4];
    uint64_t bytes[4];
    uint32_t n, wide;
};
__global__ void copy_segs_kernel(const CopySegs c) {
    for (uint32_t k = 0; k < c.n; ++k) {
        if (c.wide) {
            const uint4* s = static_cast<const uint4*>(c.src[k]);
            uint4* d = static_cast<uint4*>(c.dst[k]);
            const uint64_t m = c.bytes[k] / 16;
            for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) d[i] = s[i];
        } else {
            const uint32_t* s = static_cast<const uint32_t*>(c.src[k]);
            uint32_t* d = static_cast<uint32_t*>(c.dst[k]);
            const uint64_t m = c.bytes[k] / 4;
            for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) d[i] = s[i];
        }
    }
}

cudaError_t launch_copy_segs(const void* const* src, void* const* dst, const uint64_t* bytes, uint32_t n,
                             cudaStream_t st) {
    CopySegs c{};
    c.n = n < 4 ? n : 4;
    c.wide = 1;
    uint64_t mx = 0;
    for (uint32_t k = 0; k < c.n; ++k) {
        c.src[k] = src[k];
        c.dst[k] = dst[k];
        c.bytes[k] = bytes[k];
        if ((reinterpret_cast<uintptr_t>(src[k]) | reinterpret_cast<uintptr_t>(dst[k]) | bytes[k]) & 15u) c.wide = 0;
        mx = bytes[k] > mx ? bytes[k] : mx;
    }
    const uint64_t items = mx / (c.wide ? 16 : 4);
    const uint64_t blocks = (items + 255) / 256;
    copy_segs_kernel<<<static_cast<unsigned>(blocks < 296 ? (blocks ? blocks : 1) : 296), 256, 0, st>>>(c);
    return cudaGetLastError();
}

cudaError_t launch_buf_add_u32(uint32_t* dst, const uint32_t* src, uint64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const uint64_t b = (n + 255) / 256;
    buf_add_u32_kernel<<<static_cast<unsigned>(b < 1184 ? b : 1184), 256, 0, st>>>(dst, src, n);
    return cudaGetLastError();
}
cudaError_t launch_buf_min_u64(unsigned long long* dst, const unsigned long long* src, uint64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const uint64_t b = (n + 255) / 256;
    buf_min_u64_kernel<<<static_cast<unsigned>(b < 1184 ? b : 1184), 256, 0, st>>>(dst, src, n);
    return cudaGetLastError();
}

cudaError_t launch_score_multi(const float* cent, const uint32_t* coff, const uint32_t* kof,
                               const uint32_t* wid, uint32_t ncent, const float* keys, uint32_t n,
                               uint32_t d, int mode, float* out, double* out64, cudaStream_t st) {
    if (n == 0 || ncent == 0) return cudaSuccess;
    dim3 grid(div_up(n, 128), ncent);
    score_multi_kernel<<<grid, 128, 0, st>>>(cent, coff, kof, wid, ncent, keys, n, d, mode, out, out64);
    return cudaGetLastError();
}

cudaError_t launch_reduce_lists(uint32_t nl, const uint64_t* off, const uint32_t* idx, const float* sc,
                                const double* w, double* acc, uint32_t* cnt, uint32_t nkeys,
                                cudaStream_t st) {
    reduce_lists_kernel<<<1, 1024, 0, st>>>(nl, off, idx, sc, w, acc, cnt, nkeys);
    return cudaGetLastError();
}

size_t toplist_scratch_bytes(uint32_t n) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeysDescending(nullptr, tb, static_cast<const unsigned long long*>(nullptr),
                                             static_cast<unsigned long long*>(nullptr), static_cast<int>(n));
    return 2 * static_cast<size_t>(n) * 8 + tb + 1024;
}

// sorted: n keys (score desc, index asc); the caller takes the first L
cudaError_t launch_toplist(const float* scores, uint32_t n, unsigned long long* sorted, void* scratch,
                           size_t scratch_bytes, cudaStream_t st) {
    unsigned long long* keys = static_cast<unsigned long long*>(scratch);
    void* temp = keys + n;
    size_t tb = scratch_bytes - static_cast<size_t>(n) * 8;
    toplist_keys_kernel<<<div_up(n, 256), 256, 0, st>>>(scores, n, keys);
    return cub::DeviceRadixSort::SortKeysDescending(temp, tb, keys, sorted, static_cast<int>(n), 0, 64, st);
}

}  // namespace csa
