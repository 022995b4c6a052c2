// kmeans.cu — exact spherical k-means of one subspace per CTA
// (cosine_kmeans, clustering.cpp:73-240; kmeanspp_seed :13-71).
//
// Bit-exact with the reference by construction:
//   * the mt19937_64 stream is generated on the host (raw 64-bit outputs);
//     the kernel consumes it in the reference's order through a cursor:
//     next_index(n) = umulhi(u, n), next_unit = (u >> 11) * 2^-53;
//   * every dot product is a sequential fp64 FMA chain (float x float
//     products are exact in fp64, so FMA == mul-then-add);
//   * every order-sensitive fp64 sum (seeding weights, objectives, centroid
//     sums) runs in the reference's sequential order: the k-means++ prefix
//     is one sequential pass whose last value is the reference's `total`
//     (both start at 0 and add w_i in order), and the inverse-CDF pick is a
//     binary search on that monotone prefix (sums kept per 32 rows, the
//     found group's 32 adds redone); centroid sums are one thread per
//     (centroid, dim) walking the rows/samples in order.
// The seeding add chain runs at DADD latency (8 cycles on B200) on one lane
// while the other warps apply the previous seed's best-cosine update and
// stage the next weights (see the seeding pipeline below): c3 head
// (524288 pooled rows, 63 seeds): 445 -> 197 ms per launch.
// The data-parallel parts (normalization, k x n dot products, argmax
// assignment, best-cosine updates) use the whole CTA. One CTA per
// (session, subspace): a layer's 8 KV heads x 8 subspaces run as 64
// independent CTAs.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "kmeans.h"

namespace csa {

constexpr int KM_THREADS = 512;
constexpr int KM_MAXKW = KM_MAX_KW;  // k * w floats of centroid state in shared memory
constexpr uint32_t KM_STAGERS = KM_THREADS - 32;  // seeding: warp 0 chains, the rest stage
constexpr uint32_t KM_SR = 4;                      // rows per stager per block
constexpr uint32_t KM_CH = KM_STAGERS * KM_SR;     // rows per block (1920 = 60 x 32)
static_assert(KM_CH % 32 == 0, "blocks hold whole 32-row groups");


struct KmSmem {
    float cen[KM_MAXKW];
    double wbuf[2][KM_CH];  // seeding weight ring
    uint32_t wsum[KM_THREADS / 32];
    uint32_t n;
    uint32_t cursor;
    uint32_t pick;
    uint32_t stop;
    double total;
    double prev;
    uint32_t have_prev;
    double first_obj, last_obj;
};

__device__ __forceinline__ double unit_of(unsigned long long u) {
    return static_cast<double>(u >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ uint32_t index_of(unsigned long long u, uint32_t n) {
    return static_cast<uint32_t>(__umul64hi(u, static_cast<unsigned long long>(n)));
}

__device__ __forceinline__ double dotw(const float* a, const float* b, uint32_t w) {
    double acc = 0.0;
    for (uint32_t t = 0; t < w; ++t) acc = __fma_rn((double)a[t], (double)b[t], acc);
    return acc;
}

// k-means++ seeding weight of a row (clustering.cpp:37-38)
__device__ __forceinline__ double seed_weight(double best) {
    double dd = 1.0 - best;
    if (dd < 0.0) dd = 0.0;
    return __dmul_rn(dd, dd);
}

// ---- k-means++ seeding pipeline (clustering.cpp:34-60) ----
// Seed j needs the SEQUENTIAL fp64 prefix of w_i = max(0, 1 - best_i)^2 over
// all n rows (the reference's `total`, and its inverse-CDF walk), where best
// is the state after seed j-1's update. That add chain is inherently serial,
// so it runs on warp 0 at DADD latency while the other 15 warps ("stagers")
// apply seed j-1's update to best[] block by block (the reference's
// sequential fp64 dot, best = max(best, dot), best[pick] = 2.0) and write
// the block's weights into a double-buffered shared-memory ring. Named
// barriers hand blocks over (FULL: stagers arrive, warp 0 waits; EMPTY: warp
// 0 arrives, stagers wait), so the update overlaps the chain.

__device__ __forceinline__ void lds2(uint32_t a, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
// r + w rounded to nearest (the reference's `total += weight[i]`), issued in
// program order with the loads above
__device__ __forceinline__ double dadd_ordered(double r, double w) {
    double o;
    asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(o) : "d"(r), "d"(w));
    return o;
}
__device__ __forceinline__ void nb_sync(uint32_t id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(KM_THREADS) : "memory"); }
__device__ __forceinline__ void nb_arrive(uint32_t id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(KM_THREADS) : "memory"); }

// stager s: rows c0 + s + KM_STAGERS * u (u < KM_SR) of the block; upd:
// 0 = initial (best = dot), 1 = update (best = max(best, dot)), 2 = none.
template <int W4>
__device__ void stage_block(const float* __restrict__ train, const float* c, uint32_t w, uint32_t n,
                            double* __restrict__ best, uint32_t c0, uint32_t s, int upd, uint32_t pick,
                            double* wb) {
    const uint32_t w4 = w >> 2;
    float4 x[KM_SR][W4 > 0 ? W4 : 1];
    double bo[KM_SR];
#pragma unroll
    for (uint32_t u = 0; u < KM_SR; ++u) {
        const uint32_t i = c0 + s + KM_STAGERS * u;
        const uint32_t ii = i < n ? i : 0u;
        if (W4 > 0 && upd != 2) {
            const float4* row = reinterpret_cast<const float4*>(train + static_cast<size_t>(ii) * w);
#pragma unroll
            for (int q = 0; q < W4; ++q)
                if (q < static_cast<int>(w4)) x[u][q] = row[q];
        }
        bo[u] = upd != 0 ? best[ii] : 0.0;
    }
#pragma unroll
    for (uint32_t u = 0; u < KM_SR; ++u) {
        const uint32_t i = c0 + s + KM_STAGERS * u;
        double b = bo[u];
        if (upd != 2) {
            double acc = 0.0;
            if (W4 > 0) {
#pragma unroll
                for (int q = 0; q < W4; ++q) {
                    if (q < static_cast<int>(w4)) {
                        acc = __fma_rn((double)c[4 * q], (double)x[u][q].x, acc);
                        acc = __fma_rn((double)c[4 * q + 1], (double)x[u][q].y, acc);
                        acc = __fma_rn((double)c[4 * q + 2], (double)x[u][q].z, acc);
                        acc = __fma_rn((double)c[4 * q + 3], (double)x[u][q].w, acc);
                    }
                }
            } else {
                acc = dotw(train + static_cast<size_t>(i < n ? i : 0u) * w, c, w);
            }
            b = upd == 0 ? acc : (acc > b ? acc : b);
            if (i == pick) b = 2.0;
            if (i < n) best[i] = b;
        }
        wb[s + KM_STAGERS * u] = i < n ? seed_weight(b) : 0.0;  // rows past n add +0.0
    }
}

__device__ uint32_t km_excl_scan(KmSmem& S, uint32_t v, uint32_t& total) {
    const int wi = threadIdx.x >> 5, ln = threadIdx.x & 31;
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (ln >= o) inc += x;
    }
    __syncthreads();
    if (ln == 31) S.wsum[wi] = inc;
    __syncthreads();
    uint32_t pre = 0;
    total = 0;
    for (int i = 0; i < KM_THREADS / 32; ++i) {
        if (i < wi) pre += S.wsum[i];
        total += S.wsum[i];
    }
    return pre + inc - v;
}

// argmax_j dot(x, c_j) with bc starting at -inf and strict > (lower j wins)
__device__ __forceinline__ uint32_t nearest(const float* x, const float* cen, uint32_t k,
                                            uint32_t w, double& bc) {
    bc = -DBL_MAX;
    uint32_t bj = 0;
    bool any = false;
    for (uint32_t j = 0; j < k; ++j) {
        const double c = dotw(x, cen + j * w, w);
        if (!any || c > bc) {
            bc = c;
            bj = j;
            any = true;
        }
    }
    return bj;
}

__device__ void renormalize(KmSmem& S, const double* sums, const uint32_t* counts, uint32_t k,
                            uint32_t w, bool skip_empty) {
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) {
        if (skip_empty && counts[j] == 0) continue;
        const double* s = sums + static_cast<size_t>(j) * w;
        // s[t]*s[t] is not exact in fp64: keep the reference's rounded product
        double n2 = 0.0;
        for (uint32_t t = 0; t < w; ++t) n2 = __dadd_rn(n2, __dmul_rn(s[t], s[t]));
        if (n2 == 0.0) continue;
        const double inv = 1.0 / sqrt(n2);
        for (uint32_t t = 0; t < w; ++t) S.cen[j * w + t] = __double2float_rn(__dmul_rn(s[t], inv));
    }
    __syncthreads();
}

__global__ void __launch_bounds__(KM_THREADS) kmeans_kernel(const KmeansJob* __restrict__ jobs) {
    __shared__ KmSmem S;
    const KmeansJob& J = jobs[blockIdx.x];
    const uint32_t w = J.w, k = J.k, tid = threadIdx.x;
    float* train = J.train;

    // ---- normalize rows, drop zero rows (clustering.cpp:86-97), keep order ----
    uint32_t n = 0;
    for (uint32_t c0 = 0; c0 < J.n_total; c0 += blockDim.x) {
        const uint32_t i = c0 + tid;
        const float* x = J.q + static_cast<size_t>(i) * J.d + J.off;
        double n2 = 0.0;
        uint32_t keep = 0;
        if (i < J.n_total) {
            for (uint32_t t = 0; t < w; ++t) n2 = __fma_rn((double)x[t], (double)x[t], n2);
            keep = n2 != 0.0;
        }
        uint32_t tot;
        const uint32_t ex = km_excl_scan(S, keep, tot);
        if (keep) {
            const double inv = 1.0 / sqrt(n2);
            float* o = train + static_cast<size_t>(n + ex) * w;
            for (uint32_t t = 0; t < w; ++t) o[t] = __double2float_rn(__dmul_rn((double)x[t], inv));
        }
        n += tot;
    }
    __syncthreads();
    if (n == 0) {
        if (tid == 0) *J.status = 4;  // DataError: every training row is zero
        return;
    }
    if (tid == 0) J.info[0] = n;
    if (k > n) {
        // fewer usable rows than centroids: take each row once, then cycle
        for (uint32_t x = tid; x < k * w; x += blockDim.x) {
            const uint32_t j = x / w, t = x - j * w;
            J.cent[x] = train[static_cast<size_t>(j % n) * w + t];
        }
        return;
    }
    double* best = J.best;
    double* run = J.run;

    // ---- k-means++ seeding (clustering.cpp:13-71) ----
    uint32_t cursor = 0;
    const uint32_t first = index_of(J.rng[cursor++], n);
    for (uint32_t t = tid; t < w; t += blockDim.x) S.cen[t] = train[static_cast<size_t>(first) * w + t];
    __syncthreads();
    const bool vec = (w & 3u) == 0 && w <= 16 && (reinterpret_cast<uintptr_t>(train) & 15u) == 0;
    const uint32_t nblk = (n + KM_CH - 1) / KM_CH;
    uint32_t dup = 0;
    int upd = 0;               // the pending update of best: initial dot with seed 0
    uint32_t upd_c = 0;        // its centroid
    uint32_t upd_pick = first; // its row forced to best = 2.0
    for (uint32_t j = 1; j < k; ++j) {
        if (tid < 32) {
            // the chain: weights of block b in order, running sum after every
            // 32 rows to run[]; 16 weights per step via 8 LDS.128
            double r = 0.0;
            for (uint32_t b = 0; b < nblk; ++b) {
                nb_sync(1 + (b & 1u));
                if (tid == 0) {  // one active lane
                    // each half-group's loads go out 16 adds before their use;
                    // the warp syncs keep the compiler from sinking them next
                    // to the adds (which exposes the LDS latency per add)
                    const uint32_t wb = static_cast<uint32_t>(__cvta_generic_to_shared(S.wbuf[b & 1u]));
                    double a[16], c[16];
#pragma unroll
                    for (int q = 0; q < 8; ++q) lds2(wb + 16u * q, a[2 * q], a[2 * q + 1]);
                    for (uint32_t x = 0; x < KM_CH; x += 32) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) lds2(wb + 8u * (x + 16) + 16u * q, c[2 * q], c[2 * q + 1]);
                        __syncwarp(1u);  // a scheduling fence: the loads issue here
#pragma unroll
                        for (int q = 0; q < 16; ++q) r = dadd_ordered(r, a[q]);
                        if (x + 32 < KM_CH) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) lds2(wb + 8u * (x + 32) + 16u * q, a[2 * q], a[2 * q + 1]);
                        }
                        __syncwarp(1u);
#pragma unroll
                        for (int q = 0; q < 16; ++q) r = dadd_ordered(r, c[q]);
                        run[(b * KM_CH + x) / 32] = r;
                    }
                }
                __syncwarp();
                nb_arrive(3 + (b & 1u));
            }
            if (tid == 0) S.total = r;
        } else {
            const uint32_t st = tid - 32;
            const float* cc = S.cen + upd_c * w;
            for (uint32_t b = 0; b < nblk; ++b) {
                if (b >= 2) nb_sync(3 + (b & 1u));
                if (vec)
                    stage_block<4>(train, cc, w, n, best, b * KM_CH, st, upd, upd_pick, S.wbuf[b & 1u]);
                else
                    stage_block<0>(train, cc, w, n, best, b * KM_CH, st, upd, upd_pick, S.wbuf[b & 1u]);
                nb_arrive(1 + (b & 1u));
            }
            // balance the EMPTY arrivals of the last (up to) two blocks
            for (uint32_t b = nblk > 2 ? nblk - 2 : 0; b < nblk; ++b) nb_sync(3 + (b & 1u));
        }
        __syncthreads();
        const double total = S.total;
        if (total > 0.0) {
            if (tid == 0) {
                const double target = __dmul_rn(unit_of(J.rng[cursor]), total);
                // first i with target < (running sum after row i); pick = n-1
                // when none: the group whose end sum first exceeds target,
                // then that group's 32 adds redone from its start value
                const uint32_t ng = (n + 31) >> 5;
                uint32_t lo = 0, hi = ng;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (target < run[mid])
                        hi = mid;
                    else
                        lo = mid + 1;
                }
                uint32_t pick = n - 1;
                if (lo < ng) {
                    double r = lo ? run[lo - 1] : 0.0;
                    const uint32_t i1 = min(n, (lo + 1) * 32u);
                    for (uint32_t i = lo * 32u; i < i1; ++i) {
                        r = __dadd_rn(r, seed_weight(best[i]));
                        if (target < r) {
                            pick = i;
                            break;
                        }
                    }
                }
                S.pick = pick;
            }
            ++cursor;
            __syncthreads();
            const uint32_t pick = S.pick;
            for (uint32_t t = tid; t < w; t += blockDim.x)
                S.cen[j * w + t] = train[static_cast<size_t>(pick) * w + t];
            upd = 1;
            upd_c = j;
            upd_pick = pick;
        } else {
            for (uint32_t t = tid; t < w; t += blockDim.x) S.cen[j * w + t] = S.cen[(dup % j) * w + t];
            ++dup;
            upd = 2;  // no new seed row: best stays (the weights are recomputed as they are)
            upd_pick = 0xffffffffu;
        }
        __syncthreads();
    }

    // ---- refinement ----
    const uint32_t batch = J.batch_cfg == 0 ? (n < 4096u ? n : 4096u)
                                            : (J.batch_cfg < n ? J.batch_cfg : n);
    double* sums = J.sums;
    uint32_t* counts = J.counts;
    uint32_t* assign = J.assign;
    if (tid == 0) {
        S.have_prev = 0;
        S.stop = 0;
    }
    __syncthreads();
    if (batch >= n) {
        // full-batch Lloyd (clustering.cpp:125-192)
        for (uint32_t it = 0; it < J.iters; ++it) {
            for (uint32_t i = tid; i < n; i += blockDim.x) {
                double bc;
                assign[i] = nearest(train + static_cast<size_t>(i) * w, S.cen, k, w, bc);
                best[i] = bc;
            }
            __syncthreads();
            if (tid == 0) {
                double obj = 0.0;
                for (uint32_t i = 0; i < n; ++i) obj = __dadd_rn(obj, __fma_rn(-2.0, best[i], 2.0));
                obj = __ddiv_rn(obj, static_cast<double>(n));
                if (S.have_prev && obj > S.prev + J.tol) {
                    *J.status = 9;  // PropertyError: objective increased
                    S.stop = 2;
                } else {
                    const bool conv = S.have_prev && (S.prev - obj) < J.tol;
                    S.prev = obj;
                    S.have_prev = 1;
                    if (conv) S.stop = 1;
                }
            }
            __syncthreads();
            if (S.stop) break;
            for (uint32_t x = tid; x < k * w; x += blockDim.x) {
                const uint32_t j = x / w, t = x - j * w;
                double s = 0.0;
                uint32_t c = 0;
                for (uint32_t i = 0; i < n; ++i)
                    if (assign[i] == j) {
                        s = __dadd_rn(s, (double)train[static_cast<size_t>(i) * w + t]);
                        ++c;
                    }
                sums[x] = s;
                if (t == 0) counts[j] = c;
            }
            __syncthreads();
            if (tid == 0) {
                for (uint32_t j = 0; j < k; ++j) {
                    if (counts[j] != 0) continue;
                    // empty cluster: re-seed at the worst-covered row
                    uint32_t far = 0;
                    for (uint32_t i = 1; i < n; ++i)
                        if (best[i] < best[far]) far = i;
                    for (uint32_t t = 0; t < w; ++t) S.cen[j * w + t] = train[static_cast<size_t>(far) * w + t];
                    best[far] = 2.0;
                    J.info[1] += 1;
                }
            }
            __syncthreads();
            renormalize(S, sums, counts, k, w, true);
        }
    } else {
        // mini-batch streaming means (clustering.cpp:193-238)
        for (uint32_t x = tid; x < k * w; x += blockDim.x) sums[x] = (double)S.cen[x];
        __syncthreads();
        double* bcs = best;  // per-sample best cosine (seeding state is dead)
        for (uint32_t it = 0; it < J.iters; ++it) {
            for (uint32_t s = tid; s < batch; s += blockDim.x) {
                const uint32_t row = index_of(J.rng[cursor + s], n);
                double bc;
                const uint32_t bj = nearest(train + static_cast<size_t>(row) * w, S.cen, k, w, bc);
                assign[2 * s] = row;
                assign[2 * s + 1] = bj;
                bcs[s] = bc;
            }
            cursor += batch;
            __syncthreads();
            if (tid == 0) {
                double obj = 0.0;
                for (uint32_t s = 0; s < batch; ++s) obj = __dadd_rn(obj, __fma_rn(-2.0, bcs[s], 2.0));
                const double o = __ddiv_rn(obj, static_cast<double>(batch));
                if (it == 0) S.first_obj = o;
                S.last_obj = o;
            }
            for (uint32_t x = tid; x < k * w; x += blockDim.x) {
                const uint32_t j = x / w, t = x - j * w;
                double acc = sums[x];
                for (uint32_t s = 0; s < batch; ++s)
                    if (assign[2 * s + 1] == j)
                        acc = __dadd_rn(acc, (double)train[static_cast<size_t>(assign[2 * s]) * w + t]);
                sums[x] = acc;
            }
            __syncthreads();
            renormalize(S, sums, counts, k, w, false);
        }
        if (tid == 0 && J.iters >= 2 && S.last_obj > S.first_obj + 1e-3)
            *J.status = 9;  // PropertyError: mini-batch objective diverged
    }
    __syncthreads();
    for (uint32_t x = tid; x < k * w; x += blockDim.x) J.cent[x] = S.cen[x];
}

size_t kmeans_rng_draws(uint32_t k, uint32_t iters, uint32_t n_total, uint32_t batch_cfg) {
    const uint32_t batch = batch_cfg == 0 ? (n_total < 4096u ? n_total : 4096u)
                                          : (batch_cfg < n_total ? batch_cfg : n_total);
    return 1 + static_cast<size_t>(k) + static_cast<size_t>(iters) * batch;
}

cudaError_t launch_kmeans(const KmeansJob* jobs, uint32_t njobs, cudaStream_t st) {
    kmeans_kernel<<<njobs, KM_THREADS, 0, st>>>(jobs);
    return cudaGetLastError();
}

}  // namespace csa
