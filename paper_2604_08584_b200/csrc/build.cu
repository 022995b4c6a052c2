// build.cu — offline table build (assemble_index, index.cpp:107-141) on sm_100a.
//
//   build_scores: s[b*C+j][i] = float(sum_t double(c_j^b[t]) * double(k_i^b[t]))
//                 (score_keys, index.cpp:68-91): sequential fp64 FMA chain per
//                 score (the float x float product is exact in fp64, so FMA
//                 contraction reproduces the reference's mul-then-add), keys
//                 staged per 128-key tile in shared memory with all C centroids
//                 of the subspace; optional normalize_keys.
//   build_lists:  one CTA per table: radix select of the L-th best by
//                 (score desc, index asc) on the 64-bit image
//                 ordf(score)<<32 | ~index (TopList::from_scores :46-62), an
//                 order-preserving compaction that writes the table already
//                 index-sorted, then key-block offsets and the low buffer.
// The contraction here is K = d_b (16) deep: too shallow to feed tcgen05, and
// the result must be bit-exact fp64, so it runs on the FP64 pipe; the kernel
// is bounded by the T x P score write/read.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "tables.cuh"

namespace csa {

constexpr int BS_TILE = 128;
constexpr int BS_THREADS = 256;
constexpr int BL_THREADS = 512;

__global__ void __launch_bounds__(BS_THREADS)
build_scores_kernel(const SessionDev* __restrict__ sp, float* __restrict__ scores) {
    extern __shared__ float bsm[];
    const SessionDev& sd = *sp;
    const uint32_t b = blockIdx.y, C = sd.C, P = sd.P, d = sd.d;
    const uint32_t w = sd.widths[b], off = sd.offs[b];
    const uint32_t i0 = blockIdx.x * BS_TILE;
    float* kt = bsm;                       // [BS_TILE][w+1]
    float* ct = bsm + BS_TILE * (w + 1);   // [C][w]
    const float* cb = sd.cent + static_cast<size_t>(C) * off;
    for (uint32_t x = threadIdx.x; x < C * w; x += blockDim.x) ct[x] = cb[x];
    for (uint32_t x = threadIdx.x; x < BS_TILE * w; x += blockDim.x) {
        const uint32_t r = x / w, c = x - r * w;
        const uint32_t i = i0 + r;
        kt[r * (w + 1) + c] = i < P ? sd.kpre[static_cast<size_t>(i) * d + off + c] : 0.0f;
    }
    __syncthreads();
    const uint32_t r = threadIdx.x % BS_TILE;
    const uint32_t jg = threadIdx.x / BS_TILE, ng = blockDim.x / BS_TILE;
    const uint32_t i = i0 + r;
    if (i >= P) return;
    const float* k = kt + r * (w + 1);
    double inv = 1.0;
    bool zero = false;
    if (sd.normalize_keys) {
        double n2 = 0.0;
        for (uint32_t t = 0; t < w; ++t) n2 = __fma_rn((double)k[t], (double)k[t], n2);
        zero = n2 == 0.0;
        inv = sqrt(n2);
    }
    for (uint32_t j = jg; j < C; j += ng) {
        const float* c = ct + j * w;
        double s = 0.0;
        for (uint32_t t = 0; t < w; ++t) s = __fma_rn((double)c[t], (double)k[t], s);
        if (sd.normalize_keys) s = zero ? 0.0 : __ddiv_rn(s, inv);
        scores[static_cast<size_t>(b * C + j) * P + i] = __double2float_rn(s);
    }
}

__device__ __forceinline__ unsigned long long sel_key(float s, uint32_t i) {
    uint32_t u = __float_as_uint(s);
    if ((u << 1) == 0) u = 0;  // -0.0 == +0.0
    const uint32_t o = (u >> 31) ? ~u : (u | 0x80000000u);
    return (static_cast<unsigned long long>(o) << 32) | static_cast<uint32_t>(~i);
}

struct BuildSmem {
    RefillSmem r;
    uint32_t hist[2048];  // 11-bit radix digits
    float rmin[BL_THREADS / 32], rmax[BL_THREADS / 32];
};

__global__ void __launch_bounds__(BL_THREADS)
build_lists_kernel(const SessionDev* __restrict__ sp, const float* __restrict__ scores) {
    __shared__ BuildSmem S;
    const SessionDev& sd = *sp;
    const uint32_t t = blockIdx.x, P = sd.P;
    const float* sc = scores + static_cast<size_t>(t) * P;
    const uint32_t keep = sd.L < P ? sd.L : P;
    unsigned long long thr = 0;  // select iff sel_key >= thr
    if (keep < P) {
        auto key_of = [&](uint32_t i) { return sel_key(sc[i], i); };
        unsigned long long mn, mx;
        cta_minmax(S.r, P, key_of, mn, mx);
        thr = cta_kth_largest_mm<11>(S.r, S.hist, P, keep, mn, mx, key_of);
    }
    uint2* e = sd.ent + static_cast<size_t>(t) * sd.cap2;
    float smin = INFINITY, smax = -INFINITY;  // live score bounds (SessionDev::tmm)
    const uint32_t out = cta_compact(
        S.r, P, false, [&](uint32_t i) { return sc[i]; },
        [&](uint32_t i, float s) { return sel_key(s, i) >= thr; },
        [&](uint32_t pos, uint32_t i, float s) {
            e[pos] = make_uint2(i, __float_as_uint(s));
            smin = fminf(smin, s);
            smax = fmaxf(smax, s);
        });
    for (int o = 16; o; o >>= 1) {
        smin = fminf(smin, __shfl_xor_sync(0xffffffffu, smin, o));
        smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        S.rmin[threadIdx.x >> 5] = smin;
        S.rmax[threadIdx.x >> 5] = smax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < BL_THREADS / 32; ++i) {
            smin = fminf(smin, S.rmin[i]);
            smax = fmaxf(smax, S.rmax[i]);
        }
        sd.n_used[t] = out;
        sd.live[t] = out;
        sd.tmm[t] = make_float2(smin, smax);
    }
    __syncthreads();
    refill_table(S.r, sd, t, (P - 1) >> KEY_BLOCK_SHIFT);
}

// Shard extraction (sequence sharding): table t of the shard = the entries of
// the full session's table t with keys in [key_lo, key_hi) — one contiguous
// run of the index-sorted list of a freshly built session — then key-block
// offsets and the low buffer are rebuilt over them (refill_table).
__global__ void __launch_bounds__(BL_THREADS)
shard_extract_kernel(const SessionDev* __restrict__ fp, const SessionDev* __restrict__ sp,
                     uint32_t key_lo, uint32_t key_hi) {
    __shared__ BuildSmem S;
    const SessionDev& f = *fp;
    const SessionDev& sd = *sp;
    const uint32_t t = blockIdx.x;
    const uint32_t* fbo = f.blk_off + static_cast<size_t>(t) * f.nb_stride;
    const uint32_t last_f = (f.P - 1) >> KEY_BLOCK_SHIFT;
    const uint32_t kb0 = key_lo >> KEY_BLOCK_SHIFT, kb1 = (key_hi + KEY_BLOCK - 1) >> KEY_BLOCK_SHIFT;
    const uint32_t p0 = fbo[kb0];
    const uint32_t p1 = kb1 <= last_f ? fbo[kb1] : f.n_used[t];
    const uint2* src = f.ent + static_cast<size_t>(t) * f.cap2;
    uint2* dst = sd.ent + static_cast<size_t>(t) * sd.cap2;
    for (uint32_t i = threadIdx.x; i < p1 - p0; i += blockDim.x) dst[i] = src[p0 + i];
    if (threadIdx.x == 0) {
        sd.n_used[t] = p1 - p0;
        sd.live[t] = p1 - p0;
        sd.live_g[t] = f.live[t];
        sd.tmm[t] = f.tmm[t];
    }
    __syncthreads();
    refill_table(S.r, sd, t, (sd.P - 1) >> KEY_BLOCK_SHIFT);
}

cudaError_t launch_shard_extract(const SessionDev* full_dev, const SessionDev* shard_dev,
                                 uint32_t tables, uint32_t key_lo, uint32_t key_hi, cudaStream_t st) {
    shard_extract_kernel<<<tables, BL_THREADS, 0, st>>>(full_dev, shard_dev, key_lo, key_hi);
    return cudaGetLastError();
}

cudaError_t launch_build_scores(const SessionDev* s_dev, const SessionDev& sh, float* scores,
                                cudaStream_t st) {
    uint32_t wmax = 0;
    for (uint32_t b = 0; b < sh.m; ++b) wmax = sh.widths[b] > wmax ? sh.widths[b] : wmax;
    const size_t smem = (static_cast<size_t>(BS_TILE) * (wmax + 1) + static_cast<size_t>(sh.C) * wmax) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(build_scores_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(div_up(sh.P, BS_TILE), sh.m);
    build_scores_kernel<<<grid, BS_THREADS, smem, st>>>(s_dev, scores);
    return cudaGetLastError();
}

cudaError_t launch_build_lists(const SessionDev* s_dev, const SessionDev& sh, const float* scores,
                               cudaStream_t st) {
    build_lists_kernel<<<sh.m * sh.C, BL_THREADS, 0, st>>>(s_dev, scores);
    return cudaGetLastError();
}

}  // namespace csa
