// select.cu — CSAttention decode, part 1: route + gather + top-K on sm_100a.
//
// One thread-block CLUSTER per (session, query head) "problem". CTA r of the
// cluster owns the key range [r*KPC, (r+1)*KPC) and keeps that range's fp64
// candidate scores in its own shared memory, so per-key scores never touch
// HBM. Phases (reference functions in brackets):
//   1. route     [select_centroids retrieval.cpp:40-87]  per-subspace cosine
//                argmax (or top-tau backoff) of the normalized query slice,
//                fp64 exact, m*C dot products spread over the CTA.
//   2. gather    [gather_lists :95-109, reduce_by_key :111-148]  the selected
//                index-sorted lists' key-block ranges are streamed into a
//                shared-memory ring by TMA bulk copies (cp.async.bulk +
//                mbarrier complete_tx, several chunks in flight) and
//                accumulated with a conflict-free shared-memory RMW, chunk by
//                chunk in gathered-list order:
//                score(i) = sum_l w_b(l) * double(score_l(i)).
//   3. select    [select_topk :150-228]  cluster-wide radix select on the
//                orderable 64-bit image of the fp64 score, ties by lower
//                index, recent-window passthrough and newest-first padding;
//                the K indices are written ascending for attend.cu.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace csa {

constexpr int DEC_THREADS = 512;
constexpr int RING = 4;           // TMA staging slots
constexpr int CHUNK_E = 512;      // entries per slot (4 KB)
constexpr int DEC_WARPS = DEC_THREADS / 32;
constexpr int HB_BITS = 10;
constexpr int HB = 1 << HB_BITS;  // radix histogram bins
constexpr int SURV_LOCAL = 2048;  // compacted local survivors
constexpr int SURV_MAX = 256;     // bucket size finished on CTA 0
constexpr unsigned long long ABSENT = 0x7ff4deadbeef0000ull;  // NaN box: key not gathered

struct DecSmem {
    float q[DMAX];
    float qn[DMAX];
    uint32_t lists[MAXL];
    uint32_t lsub[MAXL];
    uint32_t nids[MAXM];
    uint32_t ids[MAXM * MAXTAU];
    uint32_t zero_mask;
    uint32_t nl;
    uint32_t hist[2][HB];
    uint32_t ghist[HB];
    uint32_t gcopy[HB];
    unsigned long long skey[SURV_MAX];
    uint32_t sidx[SURV_MAX];
    uint16_t surv[SURV_LOCAL];
    // values other CTAs of the cluster read through DSMEM
    unsigned long long x_kmax, x_kmin, x_tk;
    uint32_t x_cnt, x_tx, x_slice_total, x_nsel, x_nunt;
    // block-level scratch
    unsigned long long r64a[DEC_WARPS], r64b[DEC_WARPS];
    uint32_t r32a[DEC_WARPS], r32b[DEC_WARPS];
    float rf[DEC_WARPS];
    // broadcast scalars
    unsigned long long b_prefix, b_tk;
    uint32_t b_tx, b_rem, b_bucket, b_dsel, b_done, b_nsurv, b_use_surv, b_cabove;
    int b_pshift;
    uint32_t surv_count, wpos, nsv, b_base, b_take;
    // gather stream
    unsigned long long bar[RING];
    uint32_t c_list[RING], c_cnt[RING], c_vlo[RING], c_vhi[RING];
    uint32_t l_beg[MAXL], l_cnt[MAXL], l_first[MAXL + 1], l_lo[MAXL], l_hi[MAXL];
    uint32_t nchunk, issue_l;
};

__device__ __forceinline__ unsigned long long ordkey(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 == +0.0 (retrieval.cpp:168-171)
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ bool is_absent(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == ABSENT;
}

template <class T>
__device__ __forceinline__ T* remote(cg::cluster_group& cl, T* p, int rank) {
    return cl.map_shared_rank(p, rank);
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_maxf(float v) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum of one uint32 per thread (all threads get the result).
__device__ uint32_t block_sum(DecSmem& S, uint32_t v) {
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    v = warp_sum(v);
    __syncthreads();
    if (ln == 0) S.r32a[w] = v;
    __syncthreads();
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < DEC_WARPS; ++i) t += S.r32a[i];
    return t;
}

// Block-wide exclusive scan of two counters (thread order). Returns totals.
__device__ void block_scan2(DecSmem& S, uint32_t a, uint32_t b, uint32_t& ea, uint32_t& eb,
                            uint32_t& ta, uint32_t& tb) {
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    uint32_t ia = a, ib = b;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t xa = __shfl_up_sync(0xffffffffu, ia, o);
        uint32_t xb = __shfl_up_sync(0xffffffffu, ib, o);
        if (ln >= o) {
            ia += xa;
            ib += xb;
        }
    }
    __syncthreads();
    if (ln == 31) {
        S.r32a[w] = ia;
        S.r32b[w] = ib;
    }
    __syncthreads();
    uint32_t pa = 0, pb = 0;
    ta = 0;
    tb = 0;
#pragma unroll
    for (int i = 0; i < DEC_WARPS; ++i) {
        if (i < w) {
            pa += S.r32a[i];
            pb += S.r32b[i];
        }
        ta += S.r32a[i];
        tb += S.r32b[i];
    }
    ea = pa + ia - a;
    eb = pb + ib - b;
}

struct KeyView {
    unsigned long long* keys;  // local pool keys (0 = not in pool)
    uint32_t nloc;
};

// ---------------------------------------------------------------------------
// Phase 1: centroid routing (select_centroids, retrieval.cpp:40-87)
// ---------------------------------------------------------------------------
__device__ void route(DecSmem& S, const SessionDev& sd, double* csc, uint32_t* rep, bool leader) {
    const uint32_t m = sd.m, C = sd.C, tid = threadIdx.x;
    // normalize each slice: fp64 sum of squares, inv = 1/sqrt, x = float(x*inv)
    if (tid < m) {
        const uint32_t off = sd.offs[tid], w = sd.widths[tid];
        double n2 = 0.0;
        for (uint32_t t = 0; t < w; ++t) {
            const double x = S.q[off + t];
            n2 = __fma_rn(x, x, n2);  // x*x is exact in fp64
        }
        if (n2 == 0.0) {
            atomicOr(&S.zero_mask, 1u << tid);
        } else {
            const double inv = 1.0 / sqrt(n2);
            for (uint32_t t = 0; t < w; ++t)
                S.qn[off + t] = __double2float_rn(__dmul_rn(static_cast<double>(S.q[off + t]), inv));
        }
    }
    __syncthreads();
    // all m*C fp64 centroid dot products, sequential over the slice
    for (uint32_t x = tid; x < m * C; x += blockDim.x) {
        const uint32_t b = x / C, j = x - b * C;
        if (S.zero_mask & (1u << b)) continue;
        const uint32_t off = sd.offs[b], w = sd.widths[b];
        const float* c = sd.cent + static_cast<size_t>(C) * off + static_cast<size_t>(j) * w;
        double acc = 0.0;
        for (uint32_t t = 0; t < w; ++t)
            acc = __fma_rn(static_cast<double>(S.qn[off + t]), static_cast<double>(__ldg(c + t)), acc);
        csc[x] = acc;
    }
    __syncthreads();
    // per-subspace argmax (strict >, lower j wins), or top-tau on backoff
    const int wid = tid >> 5, ln = tid & 31;
    DecodeReport* R = reinterpret_cast<DecodeReport*>(rep);
    for (uint32_t b = wid; b < m; b += DEC_WARPS) {
        if (S.zero_mask & (1u << b)) {
            if (ln == 0) {
                S.ids[b * MAXTAU] = 0;
                S.nids[b] = 1;
                if (leader) R->best_cos[b] = 1.0;
            }
            continue;
        }
        const double* sc = csc + b * C;
        const uint32_t take = sd.tau < C ? sd.tau : C;
        for (uint32_t r = 0; r < take; ++r) {
            double bv = -DBL_MAX;
            uint32_t bj = 0xffffffffu;
            for (uint32_t j = ln; j < C; j += 32) {
                bool used = false;
                for (uint32_t u = 0; u < r; ++u) used |= (S.ids[b * MAXTAU + u] == j);
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
            if (ln == 0) S.ids[b * MAXTAU + r] = bj;
            __syncwarp();
            if (r == 0) {
                if (ln == 0 && leader) R->best_cos[b] = bv;
                if (bv >= sd.threshold) {
                    if (ln == 0) S.nids[b] = 1;
                    break;
                }
            }
            if (ln == 0) S.nids[b] = r + 1;
        }
        __syncwarp();
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t nl = 0;
        unsigned long long dots = 0, gathered = 0;
        for (uint32_t b = 0; b < m; ++b) {
            if (!(S.zero_mask & (1u << b))) dots += static_cast<unsigned long long>(C) * sd.widths[b];
            for (uint32_t r = 0; r < S.nids[b]; ++r) {
                const uint32_t t = b * C + S.ids[b * MAXTAU + r];
                S.lists[nl] = t;
                S.lsub[nl] = b;
                if (leader) {
                    R->lists[nl] = t;
                    gathered += sd.live[t];
                }
                ++nl;
            }
        }
        S.nl = nl;
        if (leader) {
            R->nl = nl;
            R->dot_ops_lo = static_cast<uint32_t>(dots);
            R->dot_ops_hi = static_cast<uint32_t>(dots >> 32);
            R->gathered_lo = static_cast<uint32_t>(gathered);
            R->gathered_hi = static_cast<uint32_t>(gathered >> 32);
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Phase 2: gather + fp64 accumulate of this CTA's key range.
// The per-list key-block ranges are concatenated into a stream of <= CHUNK_E
// entry chunks; thread 0 keeps RING chunks in flight with TMA bulk copies,
// every thread consumes chunks in order (so each key sees its lists in
// gathered order: the fixed accumulation order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void acc_entry(double* acc, uint32_t key, uint32_t sbits, double w,
                                          uint32_t k0, uint32_t k1) {
    if ((key & TOMB) || key < k0 || key >= k1) return;  // tombstone / neighbour block
    const uint32_t li = key - k0;
    const double val = __dmul_rn(w, static_cast<double>(__uint_as_float(sbits)));
    const double o = acc[li];
    acc[li] = is_absent(o) ? __dadd_rn(0.0, val) : __dadd_rn(o, val);
}

// plan the chunk stream and launch the first RING bulk copies (thread 0 issues)
__device__ void gather_issue(DecSmem& S, const SessionDev& sd, uint2* stage, uint32_t k0,
                             uint32_t k1, uint32_t N) {
    const uint32_t tid = threadIdx.x;
    const uint32_t last_blk = (N - 1) >> KEY_BLOCK_SHIFT;
    const uint32_t kb0 = k0 >> KEY_BLOCK_SHIFT;
    const uint32_t kb1 = (k1 + KEY_BLOCK - 1) >> KEY_BLOCK_SHIFT;
    if (tid < S.nl) {
        const uint32_t t = S.lists[tid];
        const uint32_t* bo = sd.blk_off + static_cast<size_t>(t) * sd.nb_stride;
        const uint32_t beg = __ldg(bo + kb0);
        const uint32_t end = kb1 <= last_blk ? __ldg(bo + kb1) : __ldcg(sd.n_used + t);
        // 16-byte aligned superset [beg & ~1, (end + 1) & ~1); cap2 is even
        const uint32_t ab = beg & ~1u;
        const uint32_t ae = end > beg ? ((end + 1) & ~1u) : ab;
        S.l_beg[tid] = ab;
        S.l_cnt[tid] = ae - ab;
        S.l_lo[tid] = beg;  // the aligned superset may include one entry of a
        S.l_hi[tid] = end;  // neighbour block or one slot past n_used: masked
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t nch = 0;
        for (uint32_t l = 0; l < S.nl; ++l) {
            S.l_first[l] = nch;
            nch += div_up(S.l_cnt[l], CHUNK_E);
        }
        S.l_first[S.nl] = nch;
        S.nchunk = nch;
        S.issue_l = 0;
        for (int r = 0; r < RING; ++r) mbar_init(&S.bar[r], 1);
        fence_mbar_init();
        for (uint32_t c = 0; c < nch && c < static_cast<uint32_t>(RING); ++c) {
            // locate chunk c
            while (S.l_first[S.issue_l + 1] <= c) ++S.issue_l;
            const uint32_t l = S.issue_l;
            const uint32_t off = (c - S.l_first[l]) * CHUNK_E;
            const uint32_t n = min(static_cast<uint32_t>(CHUNK_E), S.l_cnt[l] - off);
            const uint2* src = sd.ent + static_cast<size_t>(S.lists[l]) * sd.cap2 + S.l_beg[l] + off;
            S.c_list[c % RING] = l;
            S.c_cnt[c % RING] = n;
            S.c_vlo[c % RING] = S.l_lo[l] > S.l_beg[l] + off ? S.l_lo[l] - S.l_beg[l] - off : 0u;
            S.c_vhi[c % RING] = min(n, S.l_hi[l] - S.l_beg[l] - off);
            mbar_expect_tx(&S.bar[c % RING], n * 8);
            bulk_g2s(stage + (c % RING) * CHUNK_E, src, n * 8, &S.bar[c % RING]);
        }
    }
}

__device__ void gather_consume(DecSmem& S, const SessionDev& sd, uint2* stage, double* acc,
                               uint32_t k0, uint32_t k1) {
    const uint32_t nch = S.nchunk;
    for (uint32_t c = 0; c < nch; ++c) {
        const uint32_t slot = c % RING;
        mbar_wait(&S.bar[slot], (c / RING) & 1u);
        const uint32_t l = S.c_list[slot];
        const uint32_t n = S.c_cnt[slot];
        const uint32_t vlo = S.c_vlo[slot], vhi = S.c_vhi[slot];
        const double w = sd.weights[S.lsub[l]];
        const uint4* e4 = reinterpret_cast<const uint4*>(stage + slot * CHUNK_E);
        for (uint32_t p = threadIdx.x; p < (n >> 1); p += blockDim.x) {
            const uint4 v = e4[p];
            if (2 * p >= vlo && 2 * p < vhi) acc_entry(acc, v.x, v.y, w, k0, k1);
            if (2 * p + 1 >= vlo && 2 * p + 1 < vhi) acc_entry(acc, v.z, v.w, w, k0, k1);
        }
        __syncthreads();  // slot consumed; meta of chunk c no longer needed
        if (threadIdx.x == 0 && c + RING < nch) {
            const uint32_t cn = c + RING;
            while (S.l_first[S.issue_l + 1] <= cn) ++S.issue_l;
            const uint32_t ln = S.issue_l;
            const uint32_t off = (cn - S.l_first[ln]) * CHUNK_E;
            const uint32_t nn = min(static_cast<uint32_t>(CHUNK_E), S.l_cnt[ln] - off);
            const uint2* src = sd.ent + static_cast<size_t>(S.lists[ln]) * sd.cap2 + S.l_beg[ln] + off;
            S.c_list[slot] = ln;
            S.c_cnt[slot] = nn;
            S.c_vlo[slot] = S.l_lo[ln] > S.l_beg[ln] + off ? S.l_lo[ln] - S.l_beg[ln] - off : 0u;
            S.c_vhi[slot] = min(nn, S.l_hi[ln] - S.l_beg[ln] - off);
            mbar_expect_tx(&S.bar[slot], nn * 8);
            bulk_g2s(stage + slot * CHUNK_E, src, nn * 8, &S.bar[slot]);
        }
    }
}

// ---------------------------------------------------------------------------
// Tie resolution: the rem-th smallest index among keys == tk across the cluster.
// counts come from `cnt_of(rank)`; returns tx (exclusive) on every CTA.
// ---------------------------------------------------------------------------
template <class CountOf>
__device__ void resolve_ties(cg::cluster_group& cl, DecSmem& S, const KeyView& kv, uint32_t k0,
                             unsigned long long tk, uint32_t rem, CountOf cnt_of) {
    const int rank = cl.block_rank(), cs = cl.num_blocks();
    uint32_t before = 0;
    for (int c = 0; c < rank; ++c) before += cnt_of(c);
    const uint32_t mine = cnt_of(rank);
    if (rem > before && rem <= before + mine) {
        // this CTA holds the rem-th tie: find it in ascending local order
        const uint32_t want = rem - before;  // 1-based among local ties
        const uint32_t chunk = div_up(kv.nloc, blockDim.x);
        const uint32_t c0 = min(kv.nloc, threadIdx.x * chunk), c1 = min(kv.nloc, c0 + chunk);
        uint32_t n = 0;
        for (uint32_t l = c0; l < c1; ++l) n += (kv.keys[l] == tk);
        uint32_t ex, dummy, tot, tot2;
        block_scan2(S, n, 0, ex, dummy, tot, tot2);
        if (want > ex && want <= ex + n) {
            uint32_t seen = ex;
            for (uint32_t l = c0; l < c1; ++l)
                if (kv.keys[l] == tk && ++seen == want) {
                    *remote(cl, &S.x_tx, 0) = k0 + l + 1;
                    break;
                }
        }
    }
    (void)cs;
    cl.sync();
    if (threadIdx.x == 0) {
        S.b_tk = tk;
        S.b_tx = *remote(cl, &S.x_tx, 0);
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Phase 3: cluster-wide selection of the `need` best pool keys.
// Result (on every CTA): S.b_tk / S.b_tx such that a pool key is selected iff
// key > tk || (key == tk && index < tx).
// ---------------------------------------------------------------------------
__device__ void select_threshold(cg::cluster_group& cl, DecSmem& S, const KeyView& kv,
                                 uint32_t k0, uint32_t need) {
    const int rank = cl.block_rank(), cs = cl.num_blocks();
    const uint32_t tid = threadIdx.x;
    // pool statistics: count, max, min key
    uint32_t cnt = 0;
    unsigned long long kmax = 0, kmin = ~0ull;
    for (uint32_t l = tid; l < kv.nloc; l += blockDim.x) {
        const unsigned long long k = kv.keys[l];
        if (k) {
            ++cnt;
            kmax = k > kmax ? k : kmax;
            kmin = k < kmin ? k : kmin;
        }
    }
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmax, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmin, o);
        kmax = a > kmax ? a : kmax;
        kmin = b < kmin ? b : kmin;
    }
    const int w = tid >> 5, ln = tid & 31;
    if (ln == 0) {
        S.r32a[w] = cnt;
        S.r64a[w] = kmax;
        S.r64b[w] = kmin;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t c = 0;
        unsigned long long a = 0, b = ~0ull;
        for (int i = 0; i < DEC_WARPS; ++i) {
            c += S.r32a[i];
            a = S.r64a[i] > a ? S.r64a[i] : a;
            b = S.r64b[i] < b ? S.r64b[i] : b;
        }
        S.x_cnt = c;
        S.x_kmax = a;
        S.x_kmin = b;
    }
    cl.sync();
    uint32_t total = 0;
    unsigned long long gmax = 0, gmin = ~0ull;
    for (int c = 0; c < cs; ++c) {
        total += *remote(cl, &S.x_cnt, c);
        const unsigned long long a = *remote(cl, &S.x_kmax, c);
        const unsigned long long b = *remote(cl, &S.x_kmin, c);
        gmax = a > gmax ? a : gmax;
        gmin = b < gmin ? b : gmin;
    }
    if (need == 0) {  // nothing to take from the pool
        if (tid == 0) {
            S.b_tk = ~0ull;
            S.b_tx = 0;
        }
        __syncthreads();
        return;
    }
    if (total <= need) {  // every pool key is selected
        if (tid == 0) {
            S.b_tk = 0;
            S.b_tx = 0;
        }
        __syncthreads();
        return;
    }
    if (gmax == gmin) {  // all pool keys tie: lowest indices win
        resolve_ties(cl, S, kv, k0, gmax, need,
                     [&](int c) { return *remote(cl, &S.x_cnt, c); });
        return;
    }
    // radix passes over the bits below the common prefix of [gmin, gmax]
    const unsigned long long diff = gmax ^ gmin;
    int pshift = 64 - __clzll(static_cast<long long>(diff));  // bits [pshift, 64) are common
    unsigned long long prefix = pshift == 64 ? 0ull : (gmax >> pshift);
    uint32_t rem = need;
    bool use_surv = false;
    for (int pass = 0;; ++pass) {
        const int shift = pshift > HB_BITS ? pshift - HB_BITS : 0;
        const int nbits = pshift - shift;
        const uint32_t nb = 1u << nbits;
        uint32_t* hist = S.hist[pass & 1];
        for (uint32_t i = tid; i < nb; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        if (use_surv) {
            for (uint32_t s = tid; s < S.surv_count; s += blockDim.x) {
                const unsigned long long k = kv.keys[S.surv[s]];
                atomicAdd(&hist[(k >> shift) & (nb - 1)], 1u);
            }
        } else {
            for (uint32_t l = tid; l < kv.nloc; l += blockDim.x) {
                const unsigned long long k = kv.keys[l];
                if (!k) continue;
                if (pshift < 64 && (k >> pshift) != prefix) continue;
                atomicAdd(&hist[(k >> shift) & (nb - 1)], 1u);
            }
        }
        cl.sync();  // (A) local histograms complete
        const uint32_t sl = div_up(nb, cs);
        const uint32_t lo = min(nb, rank * sl), hi = min(nb, lo + sl);
        uint32_t part = 0;
        for (uint32_t i = lo + tid; i < hi; i += blockDim.x) {
            uint32_t v = 0;
            for (int c = 0; c < cs; ++c) v += remote(cl, hist, c)[i];
            S.ghist[i] = v;
            part += v;
        }
        part = block_sum(S, part);
        if (tid == 0) S.x_slice_total = part;
        cl.sync();  // (B) reduced slices + slice totals published
        if (w == 0) {
            // locate the slice holding the rem-th largest, scanning from the top
            uint32_t st = ln < cs ? *remote(cl, &S.x_slice_total, ln) : 0;
            // suffix sums over lanes (higher slice = higher digits)
            uint32_t suf = st;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o);
                if (ln + o < 32) suf += x;
            }
            // slice s* : suf(s*) >= rem and suf(s*+1) < rem
            const uint32_t above = suf - st;
            const bool hit = (ln < cs) && st > 0 && above < rem && suf >= rem;
            const unsigned hm = __ballot_sync(0xffffffffu, hit);
            const int sstar = __ffs(hm) - 1;
            const uint32_t cab = __shfl_sync(0xffffffffu, above, sstar);
            // copy slice s* locally, then scan its bins from the top
            const uint32_t slo = min(nb, sstar * sl), shi = min(nb, slo + sl);
            const uint32_t* src = remote(cl, S.ghist, sstar);
            for (uint32_t i = slo + ln; i < shi; i += 32) S.gcopy[i] = src[i];
            __syncwarp();
            if (ln == 0) {
                uint32_t c = cab;
                uint32_t d = shi;
                while (d > slo) {
                    --d;
                    const uint32_t h = S.gcopy[d];
                    if (c + h >= rem) break;
                    c += h;
                }
                S.b_dsel = d;
                S.b_cabove = c;
                S.b_bucket = S.gcopy[d];
            }
        }
        __syncthreads();
        const uint32_t dsel = S.b_dsel;
        rem -= S.b_cabove;
        const uint32_t bucket = S.b_bucket;
        prefix = (pshift == 64 ? 0ull : (prefix << nbits)) | dsel;
        pshift = shift;
        if (bucket == rem) {  // the whole bucket is taken
            if (tid == 0) {
                S.b_tk = (prefix << pshift) - 1;
                S.b_tx = 0;
            }
            __syncthreads();
            return;
        }
        if (pshift == 0) {  // exact ties at key == prefix
            resolve_ties(cl, S, kv, k0, prefix, rem,
                         [&](int c) { return remote(cl, hist, c)[dsel]; });
            return;
        }
        if (bucket <= SURV_MAX) {
            // gather the bucket to CTA 0 and rank it there
            uint32_t off = 0;
            for (int c = 0; c < rank; ++c) off += remote(cl, hist, c)[dsel];
            unsigned long long* dk = remote(cl, S.skey, 0);
            uint32_t* di = remote(cl, S.sidx, 0);
            if (tid == 0) S.wpos = 0;
            __syncthreads();
            auto put = [&](uint32_t l) {
                const unsigned long long k = kv.keys[l];
                if (k && (k >> pshift) == prefix) {
                    const uint32_t p = off + atomicAdd(&S.wpos, 1u);
                    dk[p] = k;
                    di[p] = k0 + l;
                }
            };
            if (use_surv) {
                for (uint32_t s = tid; s < S.surv_count; s += blockDim.x) put(S.surv[s]);
            } else {
                for (uint32_t l = tid; l < kv.nloc; l += blockDim.x) put(l);
            }
            cl.sync();  // (C) bucket gathered on CTA 0
            if (rank == 0) {
                for (uint32_t e = tid; e < bucket; e += blockDim.x) {
                    const unsigned long long ke = S.skey[e];
                    const uint32_t ie = S.sidx[e];
                    uint32_t r = 0;
                    for (uint32_t f = 0; f < bucket; ++f) {
                        const unsigned long long kf = S.skey[f];
                        r += (kf > ke) || (kf == ke && S.sidx[f] < ie);
                    }
                    if (r == rem - 1) {
                        S.x_tk = ke;
                        S.x_tx = ie + 1;
                    }
                }
            }
            cl.sync();  // (D) threshold published by CTA 0
            if (tid == 0) {
                S.b_tk = *remote(cl, &S.x_tk, 0);
                S.b_tx = *remote(cl, &S.x_tx, 0);
            }
            __syncthreads();
            return;
        }
        // narrow the local candidate set for the next pass
        const uint32_t mine = hist[dsel];
        if (mine <= SURV_LOCAL) {
            if (tid == 0) S.nsv = 0;
            __syncthreads();
            if (use_surv) {
                // filter in place: read all, then write (two phases)
                const uint32_t n0 = S.surv_count;
                uint16_t keep[4];
                uint32_t nk = 0;
                for (uint32_t s = tid, u = 0; s < n0 && u < 4; s += blockDim.x, ++u) {
                    const unsigned long long k = kv.keys[S.surv[s]];
                    if ((k >> pshift) == prefix) keep[nk++] = S.surv[s];
                }
                __syncthreads();
                for (uint32_t u = 0; u < nk; ++u) S.surv[atomicAdd(&S.nsv, 1u)] = keep[u];
            } else {
                for (uint32_t l = tid; l < kv.nloc; l += blockDim.x) {
                    const unsigned long long k = kv.keys[l];
                    if (k && (k >> pshift) == prefix) S.surv[atomicAdd(&S.nsv, 1u)] = static_cast<uint16_t>(l);
                }
            }
            __syncthreads();
            if (tid == 0) S.surv_count = S.nsv;
            use_surv = true;
            __syncthreads();
        } else {
            use_surv = false;
        }
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(DEC_THREADS, 2)
select_kernel(const DecodeProblem* __restrict__ probs, uint32_t kpc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DecSmem& S = *reinterpret_cast<DecSmem*>(smem_raw);
    uint2* stage = reinterpret_cast<uint2*>(smem_raw + ((sizeof(DecSmem) + 127) & ~size_t(127)));
    double* acc = reinterpret_cast<double*>(stage + RING * CHUNK_E);
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank(), cs = cl.num_blocks();
    const DecodeProblem& P = probs[blockIdx.x / cs];
    const SessionDev& sd = *P.s;
    const uint32_t tid = threadIdx.x, N = P.N, K = P.K, d = sd.d;
    const bool leader = rank == 0;

    const uint32_t k0 = rank * kpc;
    const uint32_t k1 = min(N, k0 + kpc);
    const uint32_t nloc = k1 > k0 ? k1 - k0 : 0;

    for (uint32_t t = tid; t < d; t += blockDim.x) S.q[t] = P.q[t];
    if (tid == 0) {
        S.zero_mask = 0;
        S.nl = 0;
        S.surv_count = 0;
    }
    __syncthreads();

    // ---- 1+2: candidate scores of this CTA's key range ----
    if (P.mode & MODE_SEARCH) {
        route(S, sd, acc, P.rep, leader);  // acc doubles as the m*C score scratch
        if (nloc) gather_issue(S, sd, stage, k0, k1, N);  // TMA copies in flight ...
        for (uint32_t l = tid; l < kpc; l += blockDim.x)  // ... while acc is reset
            acc[l] = __longlong_as_double(static_cast<long long>(ABSENT));
        __syncthreads();
        if (nloc) gather_consume(S, sd, stage, acc, k0, k1);
        if (P.mode & MODE_STORE_CACHE)
            for (uint32_t l = tid; l < nloc; l += blockDim.x) P.cache[k0 + l] = acc[l];
    } else {
        for (uint32_t l = tid; l < kpc; l += blockDim.x)
            acc[l] = (l < nloc && k0 + l < P.n_cache)
                         ? P.cache[k0 + l]
                         : __longlong_as_double(static_cast<long long>(ABSENT));
    }
    __syncthreads();

    // ---- 3: pool keys, selection threshold ----
    const uint32_t r_eff = sd.window < N ? sd.window : N;
    const uint32_t wlo = N - r_eff;
    const bool pt = sd.passthrough != 0;
    uint32_t need, f_lo;
    if (pt) {
        need = K > r_eff ? K - r_eff : 0;
        f_lo = K > r_eff ? wlo : N - K;
    } else {
        need = K;
        f_lo = N;
    }
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(acc);
    for (uint32_t l = tid; l < kpc; l += blockDim.x) {
        const uint32_t i = k0 + l;
        const double v = acc[l];
        unsigned long long key = 0;
        if (l < nloc) {
            if (i < wlo)
                key = is_absent(v) ? 0ull : ordkey(v);
            else if (!pt)
                key = ordkey(is_absent(v) ? 0.0 : v);
        }
        keys[l] = key;
    }
    __syncthreads();
    KeyView kv{keys, nloc};
    select_threshold(cl, S, kv, k0, need);
    const unsigned long long tk = S.b_tk;
    const uint32_t tx = S.b_tx;

    // ---- emit the selected set in ascending order (+ newest-first padding) ----
    const uint32_t chunk = div_up(nloc, blockDim.x);
    const uint32_t c0 = min(nloc, tid * chunk), c1 = min(nloc, c0 + chunk);
    auto picked = [&](uint32_t l) {
        const uint32_t i = k0 + l;
        const unsigned long long k = keys[l];
        return i >= f_lo || (k && (k > tk || (k == tk && i < tx)));
    };
    uint32_t nsel = 0, nunt = 0;
    for (uint32_t l = c0; l < c1; ++l) {
        if (picked(l))
            ++nsel;
        else
            ++nunt;
    }
    const int w_ = tid >> 5, ln_ = tid & 31;
    uint32_t esel, eunt, tsel, tunt;
    block_scan2(S, nsel, nunt, esel, eunt, tsel, tunt);
    if (tid == 0) {
        S.x_nsel = tsel;
        S.x_nunt = tunt;
    }
    cl.sync();
    if (w_ == 0) {
        // per-CTA padding share and output base, one lane per cluster rank
        const uint32_t ns = ln_ < cs ? *remote(cl, &S.x_nsel, ln_) : 0;
        const uint32_t nu = ln_ < cs ? *remote(cl, &S.x_nunt, ln_) : 0;
        const uint32_t all_sel = warp_sum(ns);
        uint32_t suf = nu;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o);
            if (ln_ + o < 32) suf += x;
        }
        const uint32_t above = suf - nu;
        const uint32_t pad = K > all_sel ? K - all_sel : 0;
        const uint32_t tk_l = pad > above ? min(pad - above, nu) : 0;
        const uint32_t cnt = ns + tk_l;
        uint32_t inc = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
            if (ln_ >= o) inc += x;
        }
        if (ln_ == rank) {
            S.b_base = inc - cnt;
            S.b_take = tk_l;
        }
    }
    __syncthreads();
    const uint32_t base = S.b_base, take = S.b_take;
    {
        // padded keys: the `take` highest-index untaken keys of this CTA
        const uint32_t pad_from = tunt - take;  // untaken rank >= pad_from is padded
        uint32_t pos = base + esel + (eunt > pad_from ? eunt - pad_from : 0);
        uint32_t u = eunt;
        for (uint32_t l = c0; l < c1; ++l) {
            bool s = picked(l);
            if (!s) {
                s = u >= pad_from;
                ++u;
            }
            if (s) P.sel[pos++] = k0 + l;
        }
    }
    if (leader && tid == 0) reinterpret_cast<DecodeReport*>(P.rep)->k = K;
    cl.sync();  // nobody exits while a peer may still read its shared memory
}

size_t select_smem_bytes(uint32_t kpc) {
    return ((sizeof(DecSmem) + 127) & ~size_t(127)) + static_cast<size_t>(RING) * CHUNK_E * 8 +
           static_cast<size_t>(kpc) * sizeof(double);
}

cudaError_t launch_select(const DecodeProblem* probs, uint32_t nprob, uint32_t kpc, uint32_t cs,
                          cudaStream_t st) {
    const size_t smem = select_smem_bytes(kpc);
    cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (cs > 8) {
        e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nprob * cs, 1, 1);
    cfg.blockDim = dim3(DEC_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, select_kernel, probs, kpc);
}

}  // namespace csa
