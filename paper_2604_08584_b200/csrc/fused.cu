// fused.cu — the whole decode search + sparse attention of one (session, query
// head) problem in ONE thread-block cluster, for small batches (configs c2 /
// c4: tens of problems, where the multi-kernel path is latency-bound: a route
// launch, a split select + merge launch and an attend launch per layer step).
//
// Cluster of CL CTAs (8 warps each) per problem; CTA r owns the keys
// [r*R, (r+1)*R), R = nr x 512 (warp w takes the 512-key ranges w, w+8, ...),
// and keeps its keys' fp64 sums in shared memory for the whole step.
// Nothing but the tables, the KV rows and the outputs touches global memory:
//
//   A. route (every CTA, identical): select_centroids (retrieval.cpp:40-87) +
//      gather_lists (:95-109) + score bounds [lo, hi] of every candidate
//   B. accumulate (reduce_by_key, :111-148): for every gathered list, in
//      gathered order, this warp's entries of each of its tiles (index-sorted
//      tables: one contiguous span per list), all lists' first 128 entries
//      loaded before the fp64 read-modify-writes (sum = 0.0 + w*s + ... in
//      list order, as select.cu)
//   C. histogram of the pool (select_topk's pool rules, :150-228) over a
//      2048-bin linear map of [lo, hi] (monotone: bins never split equal
//      scores); the CL histograms are summed through distributed shared
//      memory (DSMEM) into CTA 0, which finds the threshold bin
//   D. the threshold bin's members (score, index) go to CTA 0 over DSMEM; it
//      ranks them by (score desc, index asc) -> exact cut (tk, tx)
//   E. selection bits: above the cut, window passthrough, newest-first padding
//      (:218-225) across CTAs (higher ranks hold newer keys); each CTA writes
//      its ascending selection at its cluster prefix offset
//   F. attention (dense_attention masked, core.cpp:118-169) over each CTA's
//      own selected rows: online softmax per warp, CTA merge, cluster merge of
//      the CL partials in rank order (DSMEM) -> output
// Results equal the multi-kernel path's: identical selected sets, outputs
// within 1e-3 of the reference (tests/test_gpu_fused.py).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <type_traits>
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace csa {

namespace {

constexpr int FZ_THREADS = 256;
constexpr int FZ_WARPS = FZ_THREADS / 32;
constexpr uint32_t FZ_WBLKS = 512 / KEY_BLOCK;  // key blocks per 512-key warp range
constexpr int FZ_NB = 2048, FZ_NCB = FZ_NB / 32;
constexpr uint32_t FZ_BKT = 1024;  // threshold-bin members ranked in CTA 0 (more: radix over the cluster)
constexpr int FZ_MAXCL = 16;
constexpr int FZ_LB = 4;           // lists whose entries are loaded together
constexpr unsigned long long FZ_NEG0 = 0x8000000000000000ull;
constexpr unsigned long long FZ_ABSENT = 0x7ff4deadbeef0000ull;

__device__ __forceinline__ double fz_neg0() { return __longlong_as_double(static_cast<long long>(FZ_NEG0)); }
__device__ __forceinline__ bool fz_is_neg0(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == FZ_NEG0;
}
__device__ __forceinline__ unsigned long long fz_ordkey(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 == +0.0 (retrieval.cpp:168-171)
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ uint32_t fz_bin(double s, double lo, double scale) {
    const double f = __dmul_rn(__dsub_rn(s, lo), scale);
    return f >= static_cast<double>(FZ_NB - 1) ? static_cast<uint32_t>(FZ_NB - 1)
                                               : (f > 0.0 ? static_cast<uint32_t>(f) : 0u);
}
__device__ __forceinline__ float fz_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr uint32_t FZ_RANGE = 512;                  // keys per warp range
constexpr uint32_t FZ_MAXR = 32;                     // warp ranges per CTA (16384 keys)
struct FzSmem {
    uint32_t hist[FZ_NB];   // this CTA's pool histogram
    uint32_t ghist[FZ_NB];  // the cluster's (every CTA gets a copy)
    uint32_t gcoarse[FZ_NCB];  // its 32-bin sums
    uint32_t selbits[FZ_MAXR * FZ_RANGE / 32];
    unsigned long long bkey[FZ_BKT];  // CTA 0: the threshold bin's members
    uint32_t bidx[FZ_BKT];
    float part[FZ_MAXCL][132];        // CTA 0: the cluster's attention partials
    uint32_t cnt[FZ_MAXCL][2];        // CTA 0: per CTA (selected, untaken)
    float wpart[FZ_WARPS][132];       // this CTA's warps' partials
    uint32_t lists[MAXL], lsub[MAXL];
    double cw[MAXL];
    uint32_t nl, nbkt, dsel, above, take_all, overflow, scan_tot;
    unsigned long long tk;
    uint32_t tx;
    double lo, hi;
    uint32_t wsum[FZ_WARPS];
    unsigned long long dots;
    // followed by the accumulator: double acc[nr * FZ_RANGE] (dynamic size)
};
__device__ __forceinline__ double* fz_acc(FzSmem& S) {
    return reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(&S) + ((sizeof(FzSmem) + 15) & ~size_t(15)));
}

// route scratch (aliases acc, used before it is initialised)
struct FzRoute {
    float q[DMAX], qn[DMAX];
    double csc[MAX_TABLES];
    uint32_t ids[MAXM * MAXTAU], nids[MAXM], zero_mask, soff[MAXM], swid[MAXM];
    double lmin[MAXL], lmax[MAXL];
    uint32_t llive[MAXL];
    float2 ptmm[512];     // every table's live score bounds and length, loaded
    uint32_t plive[512];  // alongside the centroids (m*C <= 512)
};

__device__ __forceinline__ void fz_bar() { __syncthreads(); }

// exclusive scan over the CTA's threads; total = sum
__device__ uint32_t fz_scan(FzSmem& S, uint32_t v, uint32_t& total) {
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (ln >= o) inc += x;
    }
    if (ln == 31) S.wsum[w] = inc;
    fz_bar();
    uint32_t pre = 0;
    total = 0;
#pragma unroll
    for (int i = 0; i < FZ_WARPS; ++i) {
        const uint32_t x = S.wsum[i];
        pre += i < w ? x : 0u;
        total += x;
    }
    fz_bar();
    return pre + inc - v;
}

// The rem-th best (1-based) of the members get(e) (e < n) by (key desc, index
// asc), by 11-bit radix passes (select.cu radix_kth): sets S.tk / S.tx so that
// a member is taken iff key > tk || (key == tk && index < tx). Whole CTA.
template <class Get>
__device__ void fz_radix_kth(FzSmem& S, uint32_t n, uint32_t rem, Get get) {
    uint32_t* hist = S.hist;
    __shared__ uint32_t f_bin, f_above, f_count;
    const uint32_t tid = threadIdx.x;
    auto cross = [&](uint32_t nbins) {  // warp 0: the bin where the suffix count reaches rem
        if (tid < 32) {
            uint32_t run = 0;
            for (int g = static_cast<int>(nbins / 32) - 1; g >= 0; --g) {
                const uint32_t v = hist[g * 32 + tid];
                uint32_t suf = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o);
                    if (tid + o < 32) suf += x;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, run + suf >= rem);
                if (hit) {
                    const int l = 31 - __clz(hit);
                    if (tid == static_cast<uint32_t>(l)) {
                        f_bin = g * 32 + l;
                        f_above = run + suf - v;
                        f_count = v;
                    }
                    break;
                }
                run += __shfl_sync(0xffffffffu, suf, 0);
            }
        }
        fz_bar();
    };
    unsigned long long prefix = 0;
    int pshift = 64;
    bool ties = false;
    for (;;) {  // stage 1: the key
        const int shift = pshift > 11 ? pshift - 11 : 0;
        const uint32_t nbins = 1u << (pshift - shift);
        for (uint32_t i = tid; i < nbins; i += FZ_THREADS) hist[i] = 0;
        fz_bar();
        for (uint32_t e = tid; e < n; e += FZ_THREADS) {
            unsigned long long k;
            uint32_t ix;
            if (!get(e, k, ix)) continue;
            if (pshift < 64 && (k >> pshift) != prefix) continue;
            atomicAdd(&hist[(k >> shift) & (nbins - 1)], 1u);
        }
        fz_bar();
        cross(nbins);
        rem -= f_above;
        prefix = (pshift == 64 ? 0ull : (prefix << (pshift - shift))) | f_bin;
        pshift = shift;
        if (f_count == rem) {  // the whole digit bucket is taken
            const unsigned long long T = prefix << pshift;
            if (tid == 0) {
                S.tk = T ? T - 1 : 0ull;
                S.tx = 0;
            }
            fz_bar();
            return;
        }
        if (pshift == 0) {
            ties = true;
            break;
        }
    }
    const unsigned long long tk = prefix;  // stage 2: the rem lowest indices tied at tk
    uint32_t ipre = 0;
    int ishift = 32;
    if (ties) {
        for (;;) {
            const int shift = ishift > 11 ? ishift - 11 : 0;
            const uint32_t nbins = 1u << (ishift - shift);
            for (uint32_t i = tid; i < nbins; i += FZ_THREADS) hist[i] = 0;
            fz_bar();
            for (uint32_t e = tid; e < n; e += FZ_THREADS) {
                unsigned long long k;
                uint32_t ix;
                if (!get(e, k, ix) || k != tk) continue;
                const uint32_t r = ~ix;
                if (ishift < 32 && (r >> ishift) != ipre) continue;
                atomicAdd(&hist[(r >> shift) & (nbins - 1)], 1u);
            }
            fz_bar();
            cross(nbins);
            rem -= f_above;
            ipre = (ishift == 32 ? 0u : (ipre << (ishift - shift))) | f_bin;
            ishift = shift;
            if (f_count == rem || ishift == 0) break;
        }
    }
    if (tid == 0) {
        S.tk = tk;
        S.tx = ~(ipre << ishift) + 1u;
    }
    fz_bar();
}

// A. select_centroids + gather_lists + the candidates' score bounds, into S
// (same arithmetic as route.cu)
__device__ void fz_route(FzSmem& S, const DecodeProblem& P, const SessionDev& sd, bool report_it) {
    FzRoute& R = *reinterpret_cast<FzRoute*>(fz_acc(S));  // the launch sizes acc >= FzRoute
    const uint32_t m = sd.m, C = sd.C, d = sd.d, tid = threadIdx.x;
    DecodeReport* Rp = reinterpret_cast<DecodeReport*>(P.rep);
    for (uint32_t t = tid; t < d; t += blockDim.x) R.q[t] = P.q[t];
    if (tid < m) {
        R.soff[tid] = sd.offs[tid];
        R.swid[tid] = sd.widths[tid];
    }
    if (tid == 0) R.zero_mask = 0;
    const bool pre = m * C <= 512;
    if (pre)  // independent of the routing: in flight with the centroid loads
        for (uint32_t t = tid; t < m * C; t += blockDim.x) {
            R.ptmm[t] = __ldcg(sd.tmm + t);
            R.plive[t] = __ldcg(sd.live_g + t);
        }
    fz_bar();
    if (tid < m) {
        const uint32_t off = R.soff[tid], w = R.swid[tid];
        double n2 = 0.0;
        for (uint32_t t = 0; t < w; ++t) {
            const double x = R.q[off + t];
            n2 = __fma_rn(x, x, n2);
        }
        if (n2 == 0.0) {
            atomicOr(&R.zero_mask, 1u << tid);
        } else {
            const double inv = 1.0 / sqrt(n2);
            for (uint32_t t = 0; t < w; ++t)
                R.qn[off + t] = __double2float_rn(__dmul_rn(static_cast<double>(R.q[off + t]), inv));
        }
    }
    fz_bar();
    for (uint32_t x = tid; x < m * C; x += blockDim.x) {
        const uint32_t b = x / C, j = x - b * C;
        if (R.zero_mask & (1u << b)) continue;
        const uint32_t off = R.soff[b], w = R.swid[b];
        const float* c = sd.cent + static_cast<size_t>(C) * off + static_cast<size_t>(j) * w;
        double a = 0.0;
        if ((w & 3u) == 0u && ((C * off + j * w) & 3u) == 0u) {  // 16-byte rows: vector loads
            const float4* c4 = reinterpret_cast<const float4*>(c);
            for (uint32_t t4 = 0; t4 < w / 4; ++t4) {
                const float4 v = __ldg(c4 + t4);
                const float* qs = R.qn + off + 4 * t4;
                a = __fma_rn((double)qs[0], (double)v.x, a);
                a = __fma_rn((double)qs[1], (double)v.y, a);
                a = __fma_rn((double)qs[2], (double)v.z, a);
                a = __fma_rn((double)qs[3], (double)v.w, a);
            }
        } else {
            for (uint32_t t = 0; t < w; ++t) a = __fma_rn((double)R.qn[off + t], (double)__ldg(c + t), a);
        }
        R.csc[x] = a;
    }
    fz_bar();
    const int wid = tid >> 5, ln = tid & 31;
    for (uint32_t b = wid; b < m; b += FZ_WARPS) {
        if (R.zero_mask & (1u << b)) {  // degenerate slice: centroid 0, no backoff
            if (ln == 0) {
                R.ids[b * MAXTAU] = 0;
                R.nids[b] = 1;
                if (report_it) Rp->best_cos[b] = 1.0;
            }
            continue;
        }
        const double* sc = R.csc + b * C;
        const uint32_t take = sd.tau < C ? sd.tau : C;
        for (uint32_t r = 0; r < take; ++r) {
            double bv = -DBL_MAX;
            uint32_t bj = 0xffffffffu;
            for (uint32_t j = ln; j < C; j += 32) {
                bool used = false;
                for (uint32_t u = 0; u < r; ++u) used |= (R.ids[b * MAXTAU + u] == j);
                if (used) continue;
                const double v = sc[j];
                if (bj == 0xffffffffu || v > bv) {
                    bv = v;
                    bj = j;
                }
            }
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const uint32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (oj != 0xffffffffu && (bj == 0xffffffffu || ov > bv || (ov == bv && oj < bj))) {
                    bv = ov;
                    bj = oj;
                }
            }
            if (ln == 0) R.ids[b * MAXTAU + r] = bj;
            __syncwarp();
            if (r == 0) {
                if (ln == 0 && report_it) Rp->best_cos[b] = bv;
                if (bv >= sd.threshold) {
                    if (ln == 0) R.nids[b] = 1;
                    break;
                }
            }
            if (ln == 0) R.nids[b] = r + 1;
        }
        __syncwarp();
    }
    fz_bar();
    if (tid == 0) {
        uint32_t n = 0;
        unsigned long long dots = 0;
        for (uint32_t b = 0; b < m; ++b) {
            if (!(R.zero_mask & (1u << b))) dots += static_cast<unsigned long long>(C) * R.swid[b];
            for (uint32_t r = 0; r < R.nids[b]; ++r) {
                S.lists[n] = b * C + R.ids[b * MAXTAU + r];
                S.lsub[n] = b;
                ++n;
            }
        }
        S.nl = n;
        S.dots = dots;
    }
    fz_bar();
    const uint32_t nl = S.nl;
    if (tid < nl) {
        const uint32_t t = S.lists[tid];
        const uint32_t lv = pre ? R.plive[t] : __ldcg(sd.live_g + t);
        const float2 mm = pre ? R.ptmm[t] : __ldcg(sd.tmm + t);
        const double w = sd.weights[S.lsub[tid]];
        S.cw[tid] = w;
        R.lmin[tid] = lv ? w * static_cast<double>(mm.x) : 0.0;
        R.lmax[tid] = lv ? w * static_cast<double>(mm.y) : 0.0;
        R.llive[tid] = lv;
    }
    fz_bar();
    if (tid == 0) {
        double neg = 0.0, pos = 0.0, amin = DBL_MAX, bmax = -DBL_MAX;
        bool any = false, any_neg = false, any_pos = false;
        uint32_t g = 0;
        for (uint32_t l = 0; l < nl; ++l) {
            g += R.llive[l];
            if (R.llive[l] == 0) continue;
            const double a = R.lmin[l], b = R.lmax[l];
            any = true;
            if (a < 0.0) {
                neg += a;
                any_neg = true;
            }
            if (b > 0.0) {
                pos += b;
                any_pos = true;
            }
            amin = fmin(amin, a);
            bmax = fmax(bmax, b);
        }
        double lo = any ? (any_neg ? neg : amin) : 0.0;
        double hi = any ? (any_pos ? pos : bmax) : 0.0;
        if (!sd.passthrough) {  // window keys compete at score 0 when absent
            lo = fmin(lo, 0.0);
            hi = fmax(hi, 0.0);
        }
        S.lo = lo;
        S.hi = hi;
        if (report_it) {
            Rp->nl = nl;
            Rp->dot_ops_lo = static_cast<uint32_t>(S.dots);
            Rp->dot_ops_hi = static_cast<uint32_t>(S.dots >> 32);
            for (uint32_t l = 0; l < nl; ++l) Rp->lists[l] = S.lists[l];
            Rp->gathered_lo = g;
            Rp->gathered_hi = 0;
        }
    }
    fz_bar();
}

// the fp64 read-modify-write of up to 4 entries per lane (select.cu's order
// and canonicalisation: a -0.0f score adds as +0.0)
__device__ __forceinline__ void fz_rmw(double* acc, uint32_t kbase, const uint2 (&e)[4], double w) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        if (e[u].x & TOMB) continue;
        double* a = acc + (e[u].x - kbase);
        double x = static_cast<double>(__fadd_rn(__uint_as_float(e[u].y), 0.0f));
        if (w != 1.0) x = __dadd_rn(__dmul_rn(w, x), 0.0);
        *a = __dadd_rn(*a, x);
    }
}

template <int CL>
__global__ void __launch_bounds__(FZ_THREADS, 2)
fused_step_kernel(const DecodeProblem* __restrict__ probs, uint32_t nr) {
    extern __shared__ __align__(128) unsigned char fz_raw[];
    FzSmem& S = *reinterpret_cast<FzSmem*>(fz_raw);
    double* const acc = fz_acc(S);
    const uint32_t R = nr * FZ_RANGE;  // keys per CTA
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t rank = cluster.block_rank();
    const uint32_t p = blockIdx.x / CL;
    const DecodeProblem& P = probs[p];
    const SessionDev& sd = *P.s;
    const uint32_t tid = threadIdx.x, wid = tid >> 5, ln = tid & 31;
    const uint32_t N = P.N, K = P.K, d = sd.d;
    // the insert that follows (a programmatic dependent) may start its
    // key-scoring prologue now; it waits for this grid before any table write
    asm volatile("griddepcontrol.launch_dependents;");
    const bool search = P.mode & MODE_SEARCH;
    const bool store_cache = (P.mode & MODE_STORE_CACHE) && P.cache;
    const bool pt = sd.passthrough != 0;
    const uint32_t window = sd.window;
    const uint32_t r_eff = window < N ? window : N;
    const uint32_t wlo = N - r_eff;
    const uint32_t need = pt ? (K > r_eff ? K - r_eff : 0u) : K;
    const uint32_t f_lo = pt ? (K > r_eff ? wlo : N - K) : N;  // passthrough keys [f_lo, N)
    const uint32_t key0 = rank * R;                              // this CTA's first key
    FzSmem* S0 = cluster.map_shared_rank(&S, 0);                 // CTA 0's shared memory

    // ---- A. route ----
    if (search) {
        fz_route(S, P, sd, rank == 0);
    } else if (tid == 0) {  // a cache step: the last search's bounds
        S.lo = __ldcg(P.cbounds);
        S.hi = __ldcg(P.cbounds + 1);
        S.nl = 0;
    }
    if (tid == 0) {
        S.nbkt = 0;
        S.overflow = 0;
    }
    fz_bar();
    const double lo = S.lo, hi = S.hi;
    const double scale = hi > lo ? static_cast<double>(FZ_NB) / (hi - lo) : 0.0;
    if (search && store_cache && rank == 0 && tid == 0) {
        P.cbounds[0] = lo;
        P.cbounds[1] = hi;
    }
    const uint32_t nl = S.nl;

    // ---- B. accumulate ----
    for (uint32_t i = tid; i < R; i += FZ_THREADS) acc[i] = fz_neg0();
    for (uint32_t i = tid; i < FZ_NB; i += FZ_THREADS) S.hist[i] = 0;
    fz_bar();
    const uint32_t last_blk = N ? (N - 1) >> KEY_BLOCK_SHIFT : 0u;
    for (uint32_t j = wid; j < nr; j += FZ_WARPS) {  // this warp's key ranges
        const uint32_t kbase = key0 + j * FZ_RANGE;
        if (kbase >= N) break;
        double* const wacc = acc + j * FZ_RANGE;
        if (search) {
            // lists in groups of FZ_LB: every list's span bounds, then its first
            // 128 entries (4 per lane), all in flight before the RMWs
            for (uint32_t l0 = 0; l0 < nl; l0 += FZ_LB) {
                const uint32_t nb = min(nl - l0, static_cast<uint32_t>(FZ_LB));
                // lanes 2l, 2l+1: the bounds of list l0 + l
                uint32_t bnd = 0;
                if (ln < 2 * nb) {
                    const uint32_t l = l0 + (ln >> 1);
                    const uint32_t t = S.lists[l];
                    const uint32_t kb = (kbase >> KEY_BLOCK_SHIFT) + (ln & 1) * FZ_WBLKS;
                    bnd = kb <= last_blk ? __ldcg(sd.blk_off + static_cast<size_t>(t) * sd.nb_stride + kb)
                                         : __ldcg(sd.n_used + t);
                }
                uint2 e[FZ_LB][4];
                uint32_t ea[FZ_LB], eb[FZ_LB];
#pragma unroll
                for (int l = 0; l < FZ_LB; ++l) {
                    ea[l] = __shfl_sync(0xffffffffu, bnd, 2 * l);
                    eb[l] = __shfl_sync(0xffffffffu, bnd, 2 * l + 1);
                    if (static_cast<uint32_t>(l) >= nb) ea[l] = eb[l] = 0;
                    const uint2* tbl = sd.ent + static_cast<size_t>(S.lists[l0 + (l < nb ? l : 0)]) * sd.cap2;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t q = ea[l] + ln + 32u * u;
                        e[l][u] = q < eb[l] ? __ldcs(tbl + q) : make_uint2(TOMB, 0u);
                    }
                }
#pragma unroll
                for (int l = 0; l < FZ_LB; ++l) {
                    if (static_cast<uint32_t>(l) >= nb) break;
                    const double w = S.cw[l0 + l];
                    fz_rmw(wacc, kbase, e[l], w);
                    const uint2* tbl = sd.ent + static_cast<size_t>(S.lists[l0 + l]) * sd.cap2;
                    for (uint32_t c = ea[l] + 128; c < eb[l]; c += 128) {  // long spans
                        uint2 t4[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t q = c + ln + 32u * u;
                            t4[u] = q < eb[l] ? __ldcs(tbl + q) : make_uint2(TOMB, 0u);
                        }
                        fz_rmw(wacc, kbase, t4, w);
                    }
                    __syncwarp();  // list l's adds land before list l + 1's reads
                }
            }
        } else {  // cached candidate scores (search_period > 1)
            for (uint32_t u = 0; u < FZ_RANGE / 32; ++u) {
                const uint32_t li = u * 32 + ln, i = kbase + li;
                if (i >= N) continue;
                double v = fz_neg0();
                if (P.cache && i < P.n_cache) {
                    v = __ldcg(P.cache + i);
                    if (static_cast<unsigned long long>(__double_as_longlong(v)) == FZ_ABSENT) v = fz_neg0();
                }
                wacc[li] = v;
            }
        }
        if (store_cache) {  // the candidate cache of this search (retrieval.cpp:249)
            __syncwarp();
            for (uint32_t u = 0; u < FZ_RANGE / 32; ++u) {
                const uint32_t li = u * 32 + ln, i = kbase + li;
                if (i < N)
                    P.cache[i] = fz_is_neg0(wacc[li]) ? __longlong_as_double(static_cast<long long>(FZ_ABSENT))
                                                      : wacc[li];
            }
        }
    }
    fz_bar();

    // ---- C. histogram of the pool ----
    // pool score of key i (or not in the pool): passthrough keeps the window
    // out; otherwise window keys compete at their sum, 0 when absent
    auto pool = [&](uint32_t li, double& s) -> bool {
        const uint32_t i = key0 + li;
        if (i >= N) return false;
        const double v = acc[li];
        const bool present = !fz_is_neg0(v);
        if (i >= wlo) {
            if (pt) return false;
            s = present ? v : 0.0;
            return true;
        }
        s = v;
        return present;
    };
    // Speculative floor: the previous search of this (session, head) left its
    // threshold bin's lower edge in cbounds[2..3] (either path writes it); keys
    // below 0.9 of the way up to it are not counted. If the counts at or above
    // the floor then fall short of need, the histogram is redone from bin 0
    // (all CTAs see the same sums and take the same branch).
    uint32_t c0 = 0;
    if (need && search && !store_cache && scale > 0.0 && __ldcg(P.cbounds + 3) != 0.0) {
        const double t = __ldcg(P.cbounds + 2);
        c0 = fz_bin(lo + 0.9 * (t - lo), lo, scale);
    }
    for (;;) {
        if (need) {
            for (uint32_t i = tid; i < FZ_NB; i += FZ_THREADS) S.hist[i] = 0;
            fz_bar();
            for (uint32_t li = tid; li < R; li += FZ_THREADS) {
                double sv;
                uint32_t b = 0xffffffffu;
                if (pool(li, sv)) {
                    const uint32_t bn = fz_bin(sv, lo, scale);
                    if (bn >= c0) b = bn;
                }
                // warp-aggregated: one atomic per distinct bin of the warp
                const unsigned peers = __match_any_sync(0xffffffffu, b);
                if (b != 0xffffffffu && static_cast<int>(ln) == __ffs(peers) - 1)
                    atomicAdd(&S.hist[b], static_cast<uint32_t>(__popc(peers)));
            }
        }
        cluster.sync();  // every CTA's histogram complete
    if (need) {  // CTA r sums bins [r, r+1) * NB/CL over the cluster and hands them to every CTA
        constexpr uint32_t SL = FZ_NB / CL;
        for (uint32_t t = tid; t < SL; t += FZ_THREADS) {
            const uint32_t b = rank * SL + t;
            uint32_t v[CL];
#pragma unroll
            for (int r = 0; r < CL; ++r) v[r] = cluster.map_shared_rank(&S, r)->hist[b];
            uint32_t sum = 0;
#pragma unroll
            for (int r = 0; r < CL; ++r) sum += v[r];
#pragma unroll
            for (int r = 0; r < CL; ++r) cluster.map_shared_rank(&S, r)->ghist[b] = sum;
            // a warp holds 32 consecutive bins = one coarse bin (SL % 32 == 0)
            uint32_t cs = sum;
            for (int o = 16; o; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
            if (ln == 0)
#pragma unroll
                for (int r = 0; r < CL; ++r) cluster.map_shared_rank(&S, r)->gcoarse[b >> 5] = cs;
        }
    }
    cluster.sync();
    // threshold bin: the highest bin whose suffix count reaches need (warp 0)
    if (tid < 32) {
        uint32_t dsel = 0, above = 0, take_all = 0;
        if (need) {
            // the highest bin whose suffix count reaches need: coarse groups
            // (64 sums of 32 bins) top-down, then the 32 bins of the one found
            auto cross = [&](uint32_t v, uint32_t run, uint32_t& above_out) -> int {
                uint32_t suf = v;  // inclusive suffix over lanes >= ln
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o);
                    if (ln + o < 32) suf += x;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, run + suf >= need);
                if (!hit) {
                    above_out = run + __shfl_sync(0xffffffffu, suf, 0);
                    return -1;
                }
                const int l = 31 - __clz(hit);
                above_out = run + __shfl_sync(0xffffffffu, suf - v, l);
                return l;
            };
            int found = -1;
            uint32_t run = 0;
            for (int g = FZ_NCB / 32 - 1; g >= 0; --g) {
                uint32_t ab;
                const int l = cross(S.gcoarse[g * 32 + ln], run, ab);
                if (l >= 0) {
                    const uint32_t cb = g * 32 + l;
                    uint32_t ab2;
                    const int f = cross(S.ghist[cb * 32 + ln], ab, ab2);
                    found = static_cast<int>(cb * 32) + f;  // f >= 0: the coarse sum is exact
                    above = ab2;
                    break;
                }
                run = ab;
            }
            if (found < 0) take_all = 1;  // fewer pool keys than need: all of them
            else dsel = static_cast<uint32_t>(found);
        }
        if (ln == 0) {
            S.dsel = dsel;
            S.above = above;
            S.take_all = take_all;
        }
    }
        fz_bar();
        if (c0 == 0 || !need || !S.take_all) break;
        c0 = 0;  // the floor was above the threshold: count everything
        cluster.sync();  // every CTA done reading ghist before the next pass
    }
    const uint32_t dsel = S.dsel, take_all = S.take_all;
    const uint32_t rem = (need && !take_all) ? need - S.above : 0u;  // members of dsel to take

    // ---- D. the threshold bin's members -> CTA 0, exact cut ----
    if (rem) {
        for (uint32_t li = tid; li < R; li += FZ_THREADS) {
            double s;
            if (pool(li, s) && fz_bin(s, lo, scale) == dsel) {
                const uint32_t k = atomicAdd(&S0->nbkt, 1u);
                if (k < FZ_BKT) {
                    S0->bkey[k] = fz_ordkey(s);
                    S0->bidx[k] = key0 + li;
                } else {
                    S0->overflow = 1;
                }
            }
        }
    }
    cluster.sync();
    if (rank == 0 && rem) {
        const uint32_t nb = min(S.nbkt, FZ_BKT);
        if (!S.overflow && nb <= 384) {
            // direct ranking: member e is taken iff fewer than rem beat it; the
            // cut is the worst taken member
            for (uint32_t e = tid; e < nb; e += FZ_THREADS) {
                const unsigned long long ke = S.bkey[e];
                const uint32_t ie = S.bidx[e];
                uint32_t r = 0;
                for (uint32_t f = 0; f < nb; ++f) {
                    const unsigned long long kf = S.bkey[f];
                    r += (kf > ke) || (kf == ke && S.bidx[f] < ie);
                }
                if (r == rem - 1) {
                    S.tk = ke;
                    S.tx = ie + 1;  // taken: key > tk, or key == tk and index < tx
                }
            }
            fz_bar();
        } else if (!S.overflow) {
            fz_radix_kth(S, nb, rem, [&](uint32_t e, unsigned long long& k, uint32_t& ix) {
                k = S.bkey[e];
                ix = S.bidx[e];
                return true;
            });
        } else {  // more members than the bucket holds: rank over the cluster
            fz_radix_kth(S, static_cast<uint32_t>(CL) * R, rem,
                         [&](uint32_t e, unsigned long long& k, uint32_t& ix) {
                             const uint32_t r = e / R, li = e - r * R;
                             const uint32_t i = r * R + li;
                             if (i >= N) return false;
                             const double v = cluster.map_shared_rank(acc, r)[li];
                             const bool present = !fz_is_neg0(v);
                             double sc = v;
                             if (i >= wlo) {
                                 if (pt) return false;
                                 sc = present ? v : 0.0;
                             } else if (!present) {
                                 return false;
                             }
                             if (fz_bin(sc, lo, scale) != dsel) return false;
                             k = fz_ordkey(sc);
                             ix = i;
                             return true;
                         });
        }
    }
    cluster.sync();
    const unsigned long long tk = S0->tk;
    const uint32_t tx = S0->tx;

    // ---- E. selection bits, counts, padding, ascending emit ----
    // one key per lane, word x = 32 consecutive keys (conflict-free reads)
    for (uint32_t x = wid; x < R / 32; x += FZ_WARPS) {
        const uint32_t li = x * 32 + ln, i = key0 + li;
        bool on = false;
        if (i < N) {
            on = i >= f_lo;  // passthrough window (or the newest K)
            double sv;
            if (!on && need && pool(li, sv)) {
                const uint32_t bn = fz_bin(sv, lo, scale);
                on = take_all || bn > dsel;
                if (!on && bn == dsel && rem) {
                    const unsigned long long k = fz_ordkey(sv);
                    on = k > tk || (k == tk && i < tx);
                }
            }
        }
        const unsigned bits = __ballot_sync(0xffffffffu, on);
        if (ln == 0) S.selbits[x] = bits;
    }
    fz_bar();
    const uint32_t nkeys = key0 < N ? min(R, N - key0) : 0u;
    const uint32_t nw = (nkeys + 31) / 32;
    uint32_t c_sel = 0, c_free = 0;
    for (uint32_t x = tid; x < nw; x += FZ_THREADS) {
        const uint32_t valid = (x + 1 < nw || (nkeys & 31) == 0) ? 0xffffffffu : ((1u << (nkeys & 31)) - 1u);
        c_sel += __popc(S.selbits[x]);
        c_free += __popc(~S.selbits[x] & valid);
    }
    uint32_t tot_sel, tot_free;
    fz_scan(S, c_sel, tot_sel);
    fz_scan(S, c_free, tot_free);
    if (tid == 0) {
        S0->cnt[rank][0] = tot_sel;
        S0->cnt[rank][1] = tot_free;
    }
    cluster.sync();
    if (rank != 0 && tid < 2 * CL) (&S.cnt[0][0])[tid] = (&S0->cnt[0][0])[tid];
    fz_bar();
    uint32_t all_sel = 0, above_free = 0, before = 0;
    for (int r = 0; r < CL; ++r) {
        const uint32_t cs = S.cnt[r][0], cf = S.cnt[r][1];
        all_sel += cs;
        if (static_cast<uint32_t>(r) > rank) above_free += cf;
    }
    uint32_t take_mine = 0;  // padding: newest untaken keys (higher ranks first)
    if (all_sel < K) {
        const uint32_t pad = K - all_sel;
        take_mine = pad > above_free ? min(pad - above_free, tot_free) : 0u;
    }
    if (take_mine && tid == 0) {  // this CTA's newest untaken keys
        uint32_t left = take_mine;
        for (uint32_t x = nw; x > 0 && left;) {
            --x;
            const uint32_t valid = (x + 1 < nw || (nkeys & 31) == 0) ? 0xffffffffu : ((1u << (nkeys & 31)) - 1u);
            uint32_t z = ~S.selbits[x] & valid;
            while (z && left) {
                const int hb = 31 - __clz(z);
                S.selbits[x] |= 1u << hb;
                z &= ~(1u << hb);
                --left;
            }
        }
    }
    fz_bar();
    // my output offset: every lower rank's selected + padded count
    for (int r = 0; r < static_cast<int>(rank); ++r) {
        const uint32_t cs = S.cnt[r][0], cf = S.cnt[r][1];
        uint32_t af = 0;
        for (int q = r + 1; q < CL; ++q) af += S.cnt[q][1];
        const uint32_t tr = all_sel < K ? (K - all_sel > af ? min(K - all_sel - af, cf) : 0u) : 0u;
        before += cs + tr;
    }
    const uint32_t my_n = tot_sel + take_mine;
    {
        const uint32_t wpt = (nw + FZ_THREADS - 1) / FZ_THREADS;
        const uint32_t w0 = min(nw, tid * wpt), w1 = min(nw, w0 + wpt);
        uint32_t c = 0;
        for (uint32_t x = w0; x < w1; ++x) c += __popc(S.selbits[x]);
        uint32_t tot;
        uint32_t* const rows = reinterpret_cast<uint32_t*>(acc);  // the sums are dead now
        uint32_t pos = fz_scan(S, c, tot);
        for (uint32_t x = w0; x < w1; ++x) {
            uint32_t b = S.selbits[x];
            while (b) {
                const int lb = __ffs(b) - 1;
                const uint32_t i = key0 + x * 32 + lb;
                P.sel[before + pos] = i;
                rows[pos++] = i;
                b &= b - 1;
            }
        }
    }

    // ---- F. attention over this CTA's selected rows (ascending: P.sel[before ..]) ----
    __threadfence_block();
    fz_bar();
    {
        const float* kpre = sd.kpre;
        const float* vpre = sd.vpre;
        const float* ktail = sd.ktail;
        const float* vtail = sd.vtail;
        const uint32_t P0 = sd.P;
        const float c2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(d)));
        const float4 q4r = __ldg(reinterpret_cast<const float4*>(P.q) + ln);
        const float4 q4 = make_float4(q4r.x * c2, q4r.y * c2, q4r.z * c2, q4r.w * c2);
        float m = -FLT_MAX, s = 0.0f;
        float4 a4 = make_float4(0.f, 0.f, 0.f, 0.f);
        // warp w takes rows [8w, 8w + 8), [8w + 64, ...) of this CTA's selection
        const uint32_t* const rows = reinterpret_cast<const uint32_t*>(acc);
        for (uint32_t r0 = wid * 8; r0 < my_n; r0 += FZ_WARPS * 8) {
            float4 kk[8], vv[8];
            bool ok[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                ok[u] = r0 + u < my_n;
                const uint32_t i = rows[ok[u] ? r0 + u : r0];
                const float* kr = i < P0 ? kpre + static_cast<size_t>(i) * d : ktail + static_cast<size_t>(i - P0) * d;
                const float* vr = i < P0 ? vpre + static_cast<size_t>(i) * d : vtail + static_cast<size_t>(i - P0) * d;
                kk[u] = __ldg(reinterpret_cast<const float4*>(kr) + ln);
                vv[u] = __ldg(reinterpret_cast<const float4*>(vr) + ln);
            }
            float lg[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float x = fmaf(q4.w, kk[u].w, fmaf(q4.z, kk[u].z, fmaf(q4.y, kk[u].y, q4.x * kk[u].x)));
                for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                lg[u] = ok[u] ? x : -FLT_MAX;
            }
            float gm = lg[0];
#pragma unroll
            for (int u = 1; u < 8; ++u) gm = fmaxf(gm, lg[u]);
            if (gm > m) {
                const float f = fz_ex2(m - gm);
                s *= f;
                a4.x *= f;
                a4.y *= f;
                a4.z *= f;
                a4.w *= f;
                m = gm;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float pr = ok[u] ? fz_ex2(lg[u] - m) : 0.0f;
                s += pr;
                a4.x = fmaf(pr, vv[u].x, a4.x);
                a4.y = fmaf(pr, vv[u].y, a4.y);
                a4.z = fmaf(pr, vv[u].z, a4.z);
                a4.w = fmaf(pr, vv[u].w, a4.w);
            }
        }
        // warp partial (base-2 max) -> CTA partial -> CTA 0
        float* wp = S.wpart[wid];
        if (ln == 0) {
            wp[0] = m;
            wp[1] = s;
        }
        reinterpret_cast<float4*>(wp + 4)[ln] = a4;
        fz_bar();
        float M = -FLT_MAX;
        for (int w = 0; w < FZ_WARPS; ++w)
            if (S.wpart[w][1] > 0.0f) M = fmaxf(M, S.wpart[w][0]);
        float* dst = S0->part[rank];
        if (tid < 128) {
            float a = 0.0f;
            for (int w = 0; w < FZ_WARPS; ++w)
                if (S.wpart[w][1] > 0.0f) a += S.wpart[w][4 + tid] * fz_ex2(S.wpart[w][0] - M);
            dst[4 + tid] = a;
        }
        if (tid == 0) {
            float t = 0.0f;
            for (int w = 0; w < FZ_WARPS; ++w)
                if (S.wpart[w][1] > 0.0f) t += S.wpart[w][1] * fz_ex2(S.wpart[w][0] - M);
            dst[0] = M;
            dst[1] = t;
        }
    }
    cluster.sync();
    if (rank == 0) {  // merge the CL partials in rank order
        float GM = -FLT_MAX;
        for (int r = 0; r < CL; ++r)
            if (S.part[r][1] > 0.0f) GM = fmaxf(GM, S.part[r][0]);
        float GS = 0.0f;
        for (int r = 0; r < CL; ++r)
            if (S.part[r][1] > 0.0f) GS += S.part[r][1] * fz_ex2(S.part[r][0] - GM);
        if (tid < d) {
            float o = 0.0f;
            for (int r = 0; r < CL; ++r)
                if (S.part[r][1] > 0.0f) o += S.part[r][4 + tid] * fz_ex2(S.part[r][0] - GM);
            if (P.out) P.out[tid] = o / GS;
        }
        if (tid == 0) {
            reinterpret_cast<DecodeReport*>(P.rep)->k = K;
            // the multi-kernel path's speculative cut for the next search
            P.cbounds[2] = scale > 0.0 ? lo + static_cast<double>(dsel) / scale : lo;
            P.cbounds[3] = (need && !take_all) ? 1.0 : 0.0;
        }
    }
    cluster.sync();  // CTA 0's shared memory stays alive until every CTA is done with it
}

}  // namespace

bool fused_fits(uint32_t N, uint32_t d, int& cl, int& nr) {
    if (d != 128 || N == 0) return false;
    const uint32_t r8 = (N + 8 * FZ_RANGE - 1) / (8 * FZ_RANGE);
    if (r8 <= 14) {  // 8-CTA clusters, two CTAs per SM
        cl = 8;
        nr = static_cast<int>(r8);
        return true;
    }
    const uint32_t r16 = (N + 16 * FZ_RANGE - 1) / (16 * FZ_RANGE);
    if (r16 <= FZ_MAXR) {
        cl = 16;
        nr = static_cast<int>(r16);
        return true;
    }
    return false;
}

static size_t fz_smem(uint32_t nr) {
    const size_t acc = std::max<size_t>(static_cast<size_t>(nr) * FZ_RANGE * 8, sizeof(FzRoute));
    return ((sizeof(FzSmem) + 15) & ~size_t(15)) + acc;
}

template <int CL>
static cudaError_t launch_fz(const DecodeProblem* probs, uint32_t nprob, uint32_t nr, cudaStream_t st) {
    const size_t smem = fz_smem(nr);
    cudaError_t e = cudaFuncSetAttribute(fused_step_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(fz_smem(FZ_MAXR)));
    if (e != cudaSuccess) return e;
    if (CL > 8) {
        e = cudaFuncSetAttribute(fused_step_kernel<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nprob * CL);
    cfg.blockDim = dim3(FZ_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fused_step_kernel<CL>, probs, nr);
}

cudaError_t launch_fused_step(const DecodeProblem* probs, uint32_t nprob, int cl, int nr, cudaStream_t st) {
    if (nr < 1 || nr > static_cast<int>(FZ_MAXR)) return cudaErrorInvalidValue;
    if (cl == 8) return launch_fz<8>(probs, nprob, static_cast<uint32_t>(nr), st);
    if (cl == 16) return launch_fz<16>(probs, nprob, static_cast<uint32_t>(nr), st);
    return cudaErrorInvalidValue;
}

}  // namespace csa
