// build_tc.cu — the offline table build (assemble_index, index.cpp:107-141)
// with its centroid x key contraction on the tcgen05 tensor cores, fed by TMA.
//
// The tables must hold exactly the reference's top-L keys of every
// (subspace b, centroid j) list with exactly its scores
//     s = float(sum_t double(c_j^b[t]) * double(k_i^b[t]))   (score_keys,
// index.cpp:68-91; optional normalize_keys divides by the fp64 key norm), so
// the tensor cores only PRE-SCREEN and fp64 decides (SURVEY §7 hard part 1):
//
//   build_tc_prep    centroid rows [C][d] for the B operand (TMA source) and
//                    per-table error bounds e_t = 2^-7 ||c_t|| (fp32 norm).
//   build_tc_theta   per table: exact scores of an evenly strided sample of
//                    the keys, sorted; theta_t = the sample's value at rank
//                    q' = L/P + 4 sigma + 2/S (a guess: correctness does not
//                    depend on it, see the check below).
//   build_tc_kernel  per 128-key tile: TMA (SWIZZLE_128B tensor maps) loads the
//                    key tile and the centroid rows into shared memory; one
//                    thread issues kind::tf32 tcgen05.mma (M = 128 keys,
//                    N = C centroids, K = the subspace's width in k-steps of
//                    8) for every subspace into TMEM; 4 epilogue warps read
//                    their 32 lanes with tcgen05.ld and mark key i a CANDIDATE
//                    of table t iff  s~ + e_t ||k_i|| >= theta_t  (s~ the tf32
//                    product; normalize_keys: s~/||k_i|| + e_t >= theta_t),
//                    one ballot per (table, 32 keys) -> a bitmask word.
//   build_tc_lists   per table: candidates in ascending key order, rescored
//                    EXACTLY (the reference's sequential fp64 chain), then the
//                    exact (score desc, index asc) L-th by radix select and an
//                    order-preserving compaction into the index-sorted table,
//                    key-block offsets and low buffer (as build_lists does).
//
// Why it is exact: |s~ - s| <= (2^-9 + O(2^-23)) sum_t |c_t k_t| <=
// 2^-8.5 ||c|| ||k|| (tf32 operands keep 10 mantissa bits), so e_t ||k_i||
// (2^-7, a ~2.8x margin, covering the float rounding of s as well) bounds the
// error of every pair. Any key whose exact float score is >= theta_t is then
// a candidate. The lists kernel counts the candidates whose EXACT score is
// >= theta_t: if that count is >= L, the exact L-th best is >= theta_t, so
// every member of the true top-L (ties included) is a candidate and the radix
// select over the candidates equals the one over all P keys. If the count is
// short (theta_t guessed too high) or the candidates overflow their buffer,
// the kernel raises a flag and the host rebuilds the session with the plain
// fp64 kernels (build.cu) — never a wrong table.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "tables.cuh"
#include "tc.cuh"

namespace csa {

constexpr int BT_ROWS = 128;      // keys per tile = TMEM lanes = MMA M
constexpr int BT_THREADS = 512;   // 16 epilogue warps in 4 groups (thread 0 also issues TMA + MMA)
constexpr uint32_t BT_GROUPS = BT_THREADS / BT_ROWS;
constexpr int BT_BOX = 32;        // floats per 128-byte swizzle row
constexpr int BT_COLS = 512;      // TMEM columns (one persistent CTA per SM)
constexpr int BT_SAMPLE = 8192;   // theta sample size (power of two)
constexpr int BT_THETA_THREADS = 512;
constexpr int BT_LIST_THREADS = 512;
constexpr float BT_ERR = 0x1.0p-7f;

__device__ __forceinline__ unsigned long long bt_sel_key(float s, uint32_t i) {
    uint32_t u = __float_as_uint(s);
    if ((u << 1) == 0) u = 0;  // -0.0 == +0.0
    const uint32_t o = (u >> 31) ? ~u : (u | 0x80000000u);
    return (static_cast<unsigned long long>(o) << 32) | static_cast<uint32_t>(~i);
}

// exact score of key i against centroid c (w floats): build_scores' chain
__device__ __forceinline__ float bt_exact(const SessionDev& sd, const float* c, uint32_t w,
                                          uint32_t off, uint32_t i) {
    const float* k = sd.kpre + static_cast<size_t>(i) * sd.d + off;
    double s = 0.0, n2 = 0.0;
    for (uint32_t t = 0; t < w; t += 4) {  // the chains run in t order
        const float4 x = __ldg(reinterpret_cast<const float4*>(k + t));
        s = __fma_rn((double)c[t], (double)x.x, s);
        s = __fma_rn((double)c[t + 1], (double)x.y, s);
        s = __fma_rn((double)c[t + 2], (double)x.z, s);
        s = __fma_rn((double)c[t + 3], (double)x.w, s);
        n2 = __fma_rn((double)x.x, (double)x.x, n2);
        n2 = __fma_rn((double)x.y, (double)x.y, n2);
        n2 = __fma_rn((double)x.z, (double)x.z, n2);
        n2 = __fma_rn((double)x.w, (double)x.w, n2);
    }
    if (sd.normalize_keys) s = n2 == 0.0 ? 0.0 : __ddiv_rn(s, sqrt(n2));
    return __double2float_rn(s);
}

// U keys at once (independent chains interleaved; each chain in t order)
constexpr int BT_RU = 4;
template <int U>
__device__ __forceinline__ void bt_exact_n(const SessionDev& sd, const float* c, uint32_t w, uint32_t off,
                                           const uint32_t (&key)[U], float (&out)[U]) {
    double s[U], n2[U];
    const float* k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        s[u] = 0.0;
        n2[u] = 0.0;
        k[u] = sd.kpre + static_cast<size_t>(key[u]) * sd.d + off;
    }
    for (uint32_t t = 0; t < w; t += 4) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldg(reinterpret_cast<const float4*>(k[u] + t));
        const double c0 = c[t], c1 = c[t + 1], c2 = c[t + 2], c3 = c[t + 3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            s[u] = __fma_rn(c0, (double)x[u].x, s[u]);
            s[u] = __fma_rn(c1, (double)x[u].y, s[u]);
            s[u] = __fma_rn(c2, (double)x[u].z, s[u]);
            s[u] = __fma_rn(c3, (double)x[u].w, s[u]);
            n2[u] = __fma_rn((double)x[u].x, (double)x[u].x, n2[u]);
            n2[u] = __fma_rn((double)x[u].y, (double)x[u].y, n2[u]);
            n2[u] = __fma_rn((double)x[u].z, (double)x[u].z, n2[u]);
            n2[u] = __fma_rn((double)x[u].w, (double)x[u].w, n2[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        double v = s[u];
        if (sd.normalize_keys) v = n2[u] == 0.0 ? 0.0 : __ddiv_rn(v, sqrt(n2[u]));
        out[u] = __double2float_rn(v);
    }
}

// ---- prep: centroid rows + error bounds ----
__global__ void build_tc_prep_kernel(const SessionDev* __restrict__ sp, float* __restrict__ crow,
                                     float* __restrict__ err) {
    const SessionDev& sd = *sp;
    const uint32_t j = blockIdx.x, C = sd.C, d = sd.d;
    for (uint32_t x = threadIdx.x; x < d; x += blockDim.x) crow[static_cast<size_t>(j) * d + x] = 0.0f;
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < sd.m; b += blockDim.x) {
        const uint32_t w = sd.widths[b], off = sd.offs[b];
        const float* c = sd.cent + static_cast<size_t>(C) * off + static_cast<size_t>(j) * w;
        float n2 = 0.0f;
        for (uint32_t t = 0; t < w; ++t) {
            crow[static_cast<size_t>(j) * d + off + t] = c[t];
            n2 = fmaf(c[t], c[t], n2);
        }
        // 2^-7 ||c||, the fp32 norm nudged up (its own error is ~2^-22), plus
        // an absolute 2^-100 for operands the tensor core flushes to zero
        err[b * C + j] = BT_ERR * sqrtf(n2) * (1.0f + 0x1.0p-10f) + 0x1.0p-100f;
    }
}

// ---- theta: sample quantile per table ----
__device__ __forceinline__ uint32_t bt_ord(float s) {
    uint32_t u = __float_as_uint(s);
    if ((u << 1) == 0) u = 0;
    return (u >> 31) ? ~u : (u | 0x80000000u);
}

constexpr int BT_PER = BT_SAMPLE / BT_THETA_THREADS;  // samples per thread

__global__ void __launch_bounds__(BT_THETA_THREADS)
build_tc_theta_kernel(const SessionDev* __restrict__ sp, float qprime, float* __restrict__ theta) {
    __shared__ float c[WMAX];
    __shared__ uint32_t part[2][BT_THETA_THREADS / 32];
    const SessionDev& sd = *sp;
    const uint32_t t = blockIdx.x, C = sd.C, P = sd.P;
    const uint32_t b = t / C, j = t - b * C, w = sd.widths[b], off = sd.offs[b];
    const uint32_t S = P < BT_SAMPLE ? P : BT_SAMPLE;
    for (uint32_t x = threadIdx.x; x < w; x += blockDim.x)
        c[x] = sd.cent[static_cast<size_t>(C) * off + static_cast<size_t>(j) * w + x];
    __syncthreads();
    // ordered score bits of this thread's samples (0 = no sample; every
    // finite score maps to >= 1)
    uint32_t key[BT_PER];
#pragma unroll
    for (int y = 0; y < BT_PER; ++y) {
        const uint32_t x = y * BT_THETA_THREADS + threadIdx.x;
        const uint32_t i = static_cast<uint32_t>((static_cast<unsigned long long>(x) * P) / S);
        key[y] = x < S ? bt_ord(bt_exact(sd, c, w, off, i)) : 0u;
    }
    const float want = ceilf(qprime * static_cast<float>(S));
    uint32_t r = want < 1.0f ? 1u : static_cast<uint32_t>(want);
    if (r >= S) {
        if (threadIdx.x == 0) theta[t] = -INFINITY;  // no useful cut: every key passes
        return;
    }
    // bisection: the largest T with #(key >= T) >= r, i.e. the r-th largest
    uint32_t lo = 1u, hi = 0xffffffffu;
    for (int it = 0; lo < hi; ++it) {
        const uint32_t mid = lo + ((hi - lo) >> 1) + ((hi - lo) & 1u);
        uint32_t cnt = 0;
#pragma unroll
        for (int y = 0; y < BT_PER; ++y) cnt += key[y] >= mid ? 1u : 0u;
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if ((threadIdx.x & 31) == 0) part[it & 1][threadIdx.x >> 5] = cnt;
        __syncthreads();
        uint32_t tot = 0;
#pragma unroll
        for (int x = 0; x < BT_THETA_THREADS / 32; ++x) tot += part[it & 1][x];
        if (tot >= r)
            lo = mid;
        else
            hi = mid - 1u;
    }
    if (threadIdx.x == 0) {
        const uint32_t u = (lo & 0x80000000u) ? (lo & 0x7fffffffu) : ~lo;
        theta[t] = __uint_as_float(u);
    }
}

// ---- tcgen05 candidate screen ----
struct BtArgs {
    const SessionDev* s;
    const float* theta;  // [T]
    const float* err;    // [T]
    uint32_t* masks;     // [T][ntiles * 4]
    uint32_t ntiles, nbox, C, m, P, normalize;
};

__device__ __forceinline__ void bt_tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                          uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
        : "memory");
}

__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
    return (1u << 4)                 // D f32
           | (2u << 7) | (2u << 10)  // A, B tf32
           | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// smem: keys [2 buffers][nbox][128 rows][128 B] | centroid rows [nbox][C][128 B]
// | theta [T] | err [T] | norms [m][128] | barriers
struct BtLayout {
    uint32_t keys, cent, theta, err, nrm, bar, end;
};
__host__ __device__ inline BtLayout bt_layout(uint32_t nbox, uint32_t C, uint32_t m) {
    BtLayout L;
    L.keys = 0;
    L.cent = L.keys + 2u * nbox * BT_ROWS * 128u;
    L.theta = L.cent + nbox * C * 128u;
    L.err = L.theta + m * C * 4u;
    L.nrm = L.err + m * C * 4u;
    L.bar = (L.nrm + m * BT_ROWS * 4u + 7u) & ~7u;
    L.end = L.bar + 4u * 8u + 16u;
    return L;
}

// Persistent: one CTA per SM walks tiles blockIdx.x, += gridDim.x with the
// next tile's TMA in flight during the current tile's MMA + epilogue.
__global__ void __launch_bounds__(BT_THREADS, 1)
build_tc_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap cmap,
                const BtArgs a) {
    extern __shared__ __align__(1024) unsigned char bt_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(bt_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t nbox = a.nbox, C = a.C, m = a.m, T = m * C;
    const BtLayout L = bt_layout(nbox, C, m);
    float* th_s = reinterpret_cast<float*>(base + L.theta);
    float* er_s = reinterpret_cast<float*>(base + L.err);
    float* nrm = reinterpret_cast<float*>(base + L.nrm);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + L.bar);  // [2]
    uint64_t* mdone = full + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(full + 4);
    const SessionDev& sd = *a.s;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t r = tid & (BT_ROWS - 1), grp = tid >> 7;  // key row, subspace group
    const uint32_t kbytes = nbox * BT_ROWS * 128u;
    auto load_tile = [&](uint32_t tile, uint32_t buf, bool with_cent) {
        const uint32_t mb = tc::smem_u32(&full[buf]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                     "r"(kbytes + (with_cent ? nbox * C * 128u : 0u))
                     : "memory");
        for (uint32_t q = 0; q < nbox; ++q) {
            bt_tma_2d(tc::smem_u32(base + L.keys + buf * kbytes + q * BT_ROWS * 128u), &kmap,
                      static_cast<int>(q * BT_BOX), static_cast<int>(tile * BT_ROWS), mb);
            if (with_cent)
                bt_tma_2d(tc::smem_u32(base + L.cent + q * C * 128u), &cmap, static_cast<int>(q * BT_BOX), 0, mb);
        }
    };
    if (tid == 0) {
        tc::mbar_init(&full[0], 1);
        tc::mbar_init(&full[1], 1);
        tc::mbar_init(mdone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tc::tmem_alloc<BT_COLS>(tslot);
    for (uint32_t x = tid; x < T; x += blockDim.x) {
        th_s[x] = a.theta[x];
        er_s[x] = a.err[x];
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tslot;
    if (tid == 0) {
        load_tile(blockIdx.x, 0, true);
        if (blockIdx.x + gridDim.x < a.ntiles) load_tile(blockIdx.x + gridDim.x, 1, false);
    }
    const uint32_t idesc = idesc_tf32(BT_ROWS, C);
    const uint32_t per_pass = BT_COLS / C;  // subspaces per TMEM fill
    const uint32_t words = a.ntiles * 4u;
    uint32_t mphase = 0;
    for (uint32_t n = 0, tile = blockIdx.x; tile < a.ntiles; ++n, tile += gridDim.x) {
        const uint32_t buf = n & 1u;
        tc::mbar_wait(&full[buf], (n >> 1) & 1u);
        const unsigned char* ks = base + L.keys + buf * kbytes;
        // slice norms of this thread's key row for its group's subspaces
        // (16-byte chunk c of row r sits at chunk c ^ (r % 8))
        for (uint32_t b = grp; b < m; b += BT_GROUPS) {
            const uint32_t off = sd.offs[b], w = sd.widths[b];
            const uint32_t q = off / BT_BOX, k0 = off % BT_BOX;
            const unsigned char* row = ks + q * BT_ROWS * 128 + r * 128;
            float n2 = 0.0f;
            for (uint32_t t = 0; t < w; t += 4) {
                const uint32_t ch = (k0 + t) >> 2;
                const float4 x = *reinterpret_cast<const float4*>(row + ((ch ^ (r & 7u)) << 4));
                n2 = fmaf(x.x, x.x, fmaf(x.y, x.y, fmaf(x.z, x.z, fmaf(x.w, x.w, n2))));
            }
            nrm[b * BT_ROWS + r] = sqrtf(n2) * (1.0f + 0x1.0p-10f);
        }
        const uint32_t i = tile * BT_ROWS + r;
        const bool valid = i < a.P;
        for (uint32_t b0 = 0; b0 < m; b0 += per_pass) {
            const uint32_t b1 = b0 + per_pass < m ? b0 + per_pass : m;
            tc::fence_before();
            __syncthreads();  // previous TMEM reads done, norms visible
            if (tid == 0) {
                tc::fence_after();
                for (uint32_t b = b0; b < b1; ++b) {
                    const uint32_t off = sd.offs[b], w = sd.widths[b];
                    const uint32_t q = off / BT_BOX, k0 = off % BT_BOX;
                    const uint32_t abase = tc::smem_u32(ks + q * BT_ROWS * 128) + k0 * 4u;
                    const uint32_t bbase = tc::smem_u32(base + L.cent + q * C * 128) + k0 * 4u;
                    for (uint32_t s = 0; s < w / 8u; ++s) {
                        const uint64_t ad = tc::desc_sw128(abase + s * 32u, 16, 1024);
                        const uint64_t bd = tc::desc_sw128(bbase + s * 32u, 16, 1024);
                        mma_tf32(tmem + (b - b0) * C, ad, bd, idesc, s > 0 ? 1u : 0u);
                    }
                }
                tc::commit(mdone);
            }
            tc::mbar_wait(mdone, mphase);
            mphase ^= 1u;
            tc::fence_after();
            // the tile's operands are consumed after its last pass: refill
            if (tid == 0 && b1 == m && tile + 2u * gridDim.x < a.ntiles) load_tile(tile + 2u * gridDim.x, buf, false);
            for (uint32_t b = b0 + grp; b < b1; b += BT_GROUPS) {
                const float kn = nrm[b * BT_ROWS + r];
                const bool tiny = !(kn >= 0x1.0p-60f);
                for (uint32_t j0 = 0; j0 < C; j0 += 16) {
                    float v[16];
                    tc::tmem_ld16(tmem + (((warp & 3u) * 32u) << 16) + (b - b0) * C + j0, v);
                    uint32_t word = 0;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const uint32_t t = b * C + j0 + jj;
                        const float th = th_s[t], e = er_s[t];
                        // keys too small for the relative bound (flushed
                        // operands) and non-finite products always pass
                        bool cand = tiny || !isfinite(v[jj]);
                        if (a.normalize)
                            cand |= v[jj] / kn + e >= th;
                        else
                            cand |= fmaf(e, kn, v[jj]) >= th;
                        const uint32_t bal = __ballot_sync(0xffffffffu, cand && valid);
                        if (lane == static_cast<uint32_t>(jj)) word = bal;
                    }
                    if (lane < 16)
                        a.masks[static_cast<size_t>(b * C + j0 + lane) * words + tile * 4u + (warp & 3u)] = word;
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<BT_COLS>(tmem);
}

// ---- per-table exact rescore + selection ----
struct BtListSmem {
    RefillSmem r;
    float c[WMAX];
    uint32_t ge[BT_LIST_THREADS / 32];
    float rmin[BT_LIST_THREADS / 32], rmax[BT_LIST_THREADS / 32];
    unsigned long long kmn[BT_LIST_THREADS / 32], kmx[BT_LIST_THREADS / 32];
    uint32_t hist[2048];  // 11-bit radix digits
    uint32_t bad;
};

__global__ void __launch_bounds__(BT_LIST_THREADS)
build_tc_lists_kernel(const SessionDev* __restrict__ sp, const float* __restrict__ theta,
                      const uint32_t* __restrict__ masks, uint32_t ntiles, unsigned long long* __restrict__ cand,
                      uint32_t cap, uint32_t* __restrict__ fail) {
    __shared__ BtListSmem S;
    const SessionDev& sd = *sp;
    const uint32_t t = blockIdx.x, C = sd.C, P = sd.P;
    const uint32_t b = t / C, j = t - b * C, w = sd.widths[b], off = sd.offs[b];
    const uint32_t keep = sd.L < P ? sd.L : P;
    const float th = theta[t];
    const uint32_t words = ntiles * 4u;
    const uint32_t* mk = masks + static_cast<size_t>(t) * words;
    unsigned long long* cd = cand + static_cast<size_t>(t) * cap;
    for (uint32_t x = threadIdx.x; x < w; x += blockDim.x)
        S.c[x] = sd.cent[static_cast<size_t>(C) * off + static_cast<size_t>(j) * w + x];
    if (threadIdx.x == 0) S.bad = 0;
    __syncthreads();
    // 1. candidate keys in ascending order (positions from the popcounts)
    uint32_t out = 0;
    for (uint32_t c0 = 0; c0 < words; c0 += blockDim.x) {
        const uint32_t wi = c0 + threadIdx.x;
        uint32_t v = wi < words ? mk[wi] : 0u;
        uint32_t tot;
        const uint32_t ex = tbl_block_excl_scan(S.r, __popc(v), tot);
        if (out + tot > cap) {  // uniform: tot is the CTA total
            if (threadIdx.x == 0) S.bad = 1;
            break;
        }
        uint32_t pos = out + ex;
        const uint32_t kbase = (wi >> 2) * BT_ROWS + (wi & 3u) * 32u;
        while (v) {
            const uint32_t bit = __ffs(v) - 1;
            v &= v - 1;
            cd[pos++] = kbase + bit;
        }
        out += tot;
    }
    __syncthreads();
    // 2. exact scores -> selection keys (score desc, index asc), BT_RU
    //    candidates per thread in flight
    uint32_t ge = 0;
    unsigned long long kmn = ~0ull, kmx = 0ull;
    if (!S.bad) {
        for (uint32_t c0 = 0; c0 < out; c0 += blockDim.x * BT_RU) {
            uint32_t key[BT_RU];
#pragma unroll
            for (int u = 0; u < BT_RU; ++u) {
                const uint32_t p = c0 + u * blockDim.x + threadIdx.x;
                key[u] = p < out ? static_cast<uint32_t>(cd[p]) : 0u;
            }
            float sc[BT_RU];
            bt_exact_n<BT_RU>(sd, S.c, w, off, key, sc);
#pragma unroll
            for (int u = 0; u < BT_RU; ++u) {
                const uint32_t p = c0 + u * blockDim.x + threadIdx.x;
                if (p < out) {
                    ge += sc[u] >= th ? 1u : 0u;
                    const unsigned long long kk = bt_sel_key(sc[u], key[u]);
                    cd[p] = kk;
                    kmn = kk < kmn ? kk : kmn;
                    kmx = kk > kmx ? kk : kmx;
                }
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        ge += __shfl_xor_sync(0xffffffffu, ge, o);
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmn, o), bb = __shfl_xor_sync(0xffffffffu, kmx, o);
        kmn = a < kmn ? a : kmn;
        kmx = bb > kmx ? bb : kmx;
    }
    if ((threadIdx.x & 31) == 0) {
        S.ge[threadIdx.x >> 5] = ge;
        S.kmn[threadIdx.x >> 5] = kmn;
        S.kmx[threadIdx.x >> 5] = kmx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t g = 0;
        for (int x = 0; x < BT_LIST_THREADS / 32; ++x) g += S.ge[x];
        // fewer than `keep` keys proven >= theta: the screen may have cut a
        // member of the true top-L
        if (g < keep) S.bad = 1;
        if (S.bad) atomicAdd(fail, 1u);
    }
    __syncthreads();
    if (S.bad) return;
    for (int x = 0; x < BT_LIST_THREADS / 32; ++x) {
        kmn = S.kmn[x] < kmn ? S.kmn[x] : kmn;
        kmx = S.kmx[x] > kmx ? S.kmx[x] : kmx;
    }
    // the keep-th largest is >= theta (checked above): keys below it never
    // decide the threshold, so the radix starts from theta's key
    const unsigned long long kth = bt_sel_key(th, 0xffffffffu);
    kmn = kth > kmn ? kth : kmn;
    unsigned long long thr = 0;
    if (keep < out) thr = cta_kth_largest_mm<11>(S.r, S.hist, out, keep, kmn, kmx, [&](uint32_t p) { return cd[p]; });
    uint2* e = sd.ent + static_cast<size_t>(t) * sd.cap2;
    float smin = INFINITY, smax = -INFINITY;
    const uint32_t n = cta_compact(
        S.r, out, false, [&](uint32_t p) { return cd[p]; },
        [&](uint32_t, unsigned long long k) { return k >= thr; },
        [&](uint32_t pos, uint32_t, unsigned long long k) {
            const uint32_t idx = ~static_cast<uint32_t>(k), o = static_cast<uint32_t>(k >> 32);
            uint32_t bits = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
            // the key canonicalised -0.0 to +0.0: the table keeps the
            // reference's float(s) bits, so recover the sign
            if (bits == 0u) bits = __float_as_uint(bt_exact(sd, S.c, w, off, idx));
            e[pos] = make_uint2(idx, bits);
            smin = fminf(smin, __uint_as_float(bits));
            smax = fmaxf(smax, __uint_as_float(bits));
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
        for (int x = 0; x < BT_LIST_THREADS / 32; ++x) {
            smin = fminf(smin, S.rmin[x]);
            smax = fmaxf(smax, S.rmax[x]);
        }
        sd.n_used[t] = n;
        sd.live[t] = n;
        sd.tmm[t] = make_float2(smin, smax);
    }
    __syncthreads();
    refill_table(S.r, sd, t, (P - 1) >> KEY_BLOCK_SHIFT);
}

// ---- host side ----
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

bool make_map(CUtensorMap* map, const float* ptr, uint32_t inner, uint32_t rows, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner) * 4u};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(BT_BOX), box_rows};
    const cuuint32_t es[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t bt_smem(uint32_t nbox, uint32_t C, uint32_t m) { return 1024 + bt_layout(nbox, C, m).end; }
}  // namespace

bool build_tc_eligible(const SessionDev& sh) {
    if (!encode_fn()) return false;
    if (sh.d % 4 != 0 || sh.d > 256 || sh.C % 16 != 0 || sh.C < 16 || sh.C > BT_COLS) return false;
    if (sh.L >= sh.P) return false;
    for (uint32_t b = 0; b < sh.m; ++b) {
        const uint32_t w = sh.widths[b], off = sh.offs[b];
        if (w % 8 != 0 || (off % BT_BOX) + w > static_cast<uint32_t>(BT_BOX)) return false;
    }
    const uint32_t nbox = div_up(sh.d, BT_BOX);
    return bt_smem(nbox, sh.C, sh.m) <= 220u * 1024u;
}

size_t build_tc_scratch_bytes(const SessionDev& sh, uint32_t* cap_out) {
    const uint32_t T = sh.m * sh.C, P = sh.P;
    const uint32_t keep = sh.L < P ? sh.L : P;
    const unsigned long long capl = static_cast<unsigned long long>(keep) + keep / 4u + 2048u;
    const uint32_t cap = capl < P ? static_cast<uint32_t>(capl) : P;
    const uint32_t ntiles = div_up(P, BT_ROWS);
    if (cap_out) *cap_out = cap;
    // crow [C][d] f32, err/theta [T] f32, masks [T][ntiles*4] u32, cand [T][cap] u2, fail u32
    return (static_cast<size_t>(sh.C) * sh.d + 2u * T) * 4u + static_cast<size_t>(T) * ntiles * 16u +
           static_cast<size_t>(T) * cap * 8u + 256u;
}

cudaError_t launch_build_tc(const SessionDev* s_dev, const SessionDev& sh, void* scratch, float qmargin,
                            uint32_t* fail_dev, cudaStream_t st) {
    const uint32_t T = sh.m * sh.C, P = sh.P, C = sh.C, d = sh.d;
    uint32_t cap = 0;
    build_tc_scratch_bytes(sh, &cap);
    const uint32_t ntiles = div_up(P, BT_ROWS), nbox = div_up(d, BT_BOX);
    char* p = static_cast<char*>(scratch);
    float* crow = reinterpret_cast<float*>(p);
    p += static_cast<size_t>(C) * d * 4u;
    float* err = reinterpret_cast<float*>(p);
    p += static_cast<size_t>(T) * 4u;
    float* theta = reinterpret_cast<float*>(p);
    p += static_cast<size_t>(T) * 4u;
    p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    uint32_t* masks = reinterpret_cast<uint32_t*>(p);
    p += static_cast<size_t>(T) * ntiles * 16u;
    unsigned long long* cand = reinterpret_cast<unsigned long long*>(p);
    cudaError_t e = cudaMemsetAsync(fail_dev, 0, 4, st);
    if (e != cudaSuccess) return e;
    build_tc_prep_kernel<<<C, 32, 0, st>>>(s_dev, crow, err);
    // q' = L/P + 4 sigma + 2/S (+ the test hook's margin)
    const double S = P < static_cast<uint32_t>(BT_SAMPLE) ? P : BT_SAMPLE;
    const double q = static_cast<double>(sh.L) / P;
    const double qp = q + 4.0 * std::sqrt(q * (1.0 - q) / S) + 2.0 / S + qmargin;
    build_tc_theta_kernel<<<T, BT_THETA_THREADS, 0, st>>>(s_dev, static_cast<float>(qp), theta);
    CUtensorMap kmap, cmap;
    if (!make_map(&kmap, sh.kpre, d, P, BT_ROWS) || !make_map(&cmap, crow, d, C, C))
        return cudaErrorInvalidValue;
    BtArgs a{s_dev, theta, err, masks, ntiles, nbox, C, sh.m, P, sh.normalize_keys};
    const size_t smem = bt_smem(nbox, C, sh.m);
    e = cudaFuncSetAttribute(build_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    build_tc_kernel<<<ntiles < static_cast<uint32_t>(sms) ? ntiles : sms, BT_THREADS, smem, st>>>(kmap, cmap, a);
    build_tc_lists_kernel<<<T, BT_LIST_THREADS, 0, st>>>(s_dev, theta, masks, ntiles, cand, cap, fail_dev);
    return cudaGetLastError();
}

}  // namespace csa
