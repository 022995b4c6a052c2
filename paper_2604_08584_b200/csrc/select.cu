// select.cu — CSAttention decode, part 1: route + gather + top-K on sm_100a.
//
// One thread-block CLUSTER per (session, query head) "problem". CTA r of the
// cluster owns the key range [r*KPC, (r+1)*KPC) and keeps that range's fp64
// candidate scores in its own shared memory, so per-key scores never touch
// HBM. Phases (reference functions in brackets):
//   1. plan      routing (select_centroids) is done by route.cu, which also
//                writes every rank's entry range of each gathered list.
//   2. gather    [gather_lists :95-109, reduce_by_key :111-148]  the selected
//                index-sorted lists' key-block ranges are streamed into an
//                8-slot shared-memory ring by TMA bulk copies (cp.async.bulk +
//                mbarrier complete_tx) and accumulated with a conflict-free
//                shared-memory RMW, chunk by chunk in gathered-list order:
//                score(i) = sum_l w_b(l) * double(score_l(i)).
//   3. select    [select_topk :150-228]  the `need`-th best pool key by
//                (score desc, index asc), cluster-wide: one 1024-bin
//                linear-bucket pass in the fp64 domain (monotone, so the
//                threshold bucket is exact), then the bucket's members are
//                ranked on CTA 0. Degenerate inputs (huge buckets, exact ties)
//                fall back to 64-bit radix passes and index-order tie breaks.
//   4. emit      window passthrough + newest-first padding; the K indices are
//                written ascending for attend.cu.
// Shared memory: a small header, one 32 KB region reused as (query slices |
// TMA ring | selection scratch) across phases, and KPC fp64 scores.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace csa {

constexpr int SEL_THREADS = 256;
constexpr int SEL_WARPS = SEL_THREADS / 32;
constexpr int RING = 4;           // TMA staging slots
constexpr int CHUNK_E = 1024;     // entries per slot (8 KB)
constexpr int HB_BITS = 10;
constexpr int HB = 1 << HB_BITS;  // histogram bins
constexpr int SURV_LOCAL = 2048;  // compacted local survivors (fallback radix)
constexpr int SURV_MAX = 256;     // bucket size finished on CTA 0
constexpr unsigned long long ABSENT = 0x7ff4deadbeef0000ull;  // NaN box: key not gathered

struct SelHdr {
    uint32_t lists[MAXL];
    uint32_t lsub[MAXL];
    uint32_t nids[MAXM];
    uint32_t ids[MAXM * MAXTAU];
    uint32_t zero_mask, nl;
    // gather stream
    unsigned long long bar[RING];    // full: TMA bytes landed
    unsigned long long empty[RING];  // all warps done with the slot
    uint32_t c_list[RING], c_cnt[RING], c_vlo[RING], c_vhi[RING];
    uint32_t l_beg[MAXL], l_cnt[MAXL], l_first[MAXL + 1], l_lo[MAXL], l_hi[MAXL];
    uint32_t nchunk, issue_l;
    // values other CTAs of the cluster read through DSMEM
    unsigned long long x_kmax, x_kmin, x_tk, x_bmax, x_bmin;
    uint32_t x_cnt, x_tx, x_slice_total, x_nsel, x_nunt;
    // block scratch / broadcasts
    unsigned long long r64a[SEL_WARPS], r64b[SEL_WARPS];
    uint32_t r32a[SEL_WARPS], r32b[SEL_WARPS];
    unsigned long long b_tk, b_gmax, b_gmin;
    uint32_t b_tx, b_dsel, b_cabove, b_bucket, b_base, b_take, b_total, b_off;
    uint32_t surv_count, wpos, nsv;
};

// the 32 KB multi-use region
struct SelectView {
    uint32_t hist[2][HB];
    uint32_t ghist[HB];
    uint32_t gcopy[HB];
    unsigned long long skey[SURV_MAX];
    uint32_t sidx[SURV_MAX];
    uint16_t surv[SURV_LOCAL];
};
constexpr size_t REGION_BYTES = static_cast<size_t>(RING) * CHUNK_E * sizeof(uint2);
static_assert(sizeof(SelectView) <= REGION_BYTES, "select view exceeds region");

__device__ __forceinline__ unsigned long long ordkey(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 == +0.0 (retrieval.cpp:168-171)
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_double(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
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

__device__ uint32_t block_sum(SelHdr& S, uint32_t v) {
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    v = warp_sum(v);
    __syncthreads();
    if (ln == 0) S.r32a[w] = v;
    __syncthreads();
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < SEL_WARPS; ++i) t += S.r32a[i];
    return t;
}

// Block-wide exclusive scan of two counters (thread order) + totals.
__device__ void block_scan2(SelHdr& S, uint32_t a, uint32_t b, uint32_t& ea, uint32_t& eb,
                            uint32_t& ta, uint32_t& tb) {
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    uint32_t ia = a, ib = b;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t xa = __shfl_up_sync(0xffffffffu, ia, o);
        const uint32_t xb = __shfl_up_sync(0xffffffffu, ib, o);
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
    ta = tb = 0;
#pragma unroll
    for (int i = 0; i < SEL_WARPS; ++i) {
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

// lane c of the calling warp gets f(c) for c < cs; returns the exclusive prefix
// over ranks < `rank` and the total (warp-uniform).
template <class F>
__device__ __forceinline__ void warp_rank_scan(int cs, int rank, F f, uint32_t& before,
                                               uint32_t& total) {
    const int ln = threadIdx.x & 31;
    const uint32_t v = ln < cs ? f(ln) : 0u;
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (ln >= o) inc += x;
    }
    total = __shfl_sync(0xffffffffu, inc, 31);
    before = rank > 0 ? __shfl_sync(0xffffffffu, inc, rank - 1) : 0u;
}

// ---------------------------------------------------------------------------
// Phase 1: the routing plan written by route.cu (lists, subspaces, and this
// rank's entry range of every list) — one round trip.
// ---------------------------------------------------------------------------
__device__ void load_plan(SelHdr& S, const RoutePlan& plan, int rank) {
    const uint32_t nl = __ldcg(&plan.nl);
    if (threadIdx.x < MAXL) {  // all slots at once (one round trip); slots >= nl unused
        const uint32_t l = threadIdx.x;
        S.lists[l] = __ldcg(plan.lists + l);
        S.lsub[l] = __ldcg(plan.lsub + l);
        const uint2 be = plan.bounds[rank * MAXL + l];
        S.l_lo[l] = be.x;
        S.l_hi[l] = be.y;
    }
    if (threadIdx.x == 0) S.nl = nl;
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
                                          uint32_t k0) {
    if (key & TOMB) return;  // evicted entry
    const uint32_t li = key - k0;
    const double val = __dmul_rn(w, static_cast<double>(__uint_as_float(sbits)));
    const double o = acc[li];
    acc[li] = is_absent(o) ? __dadd_rn(0.0, val) : __dadd_rn(o, val);
}

__device__ __forceinline__ void issue_chunk(SelHdr& S, const SessionDev& sd, uint2* stage,
                                            uint32_t c) {
    while (S.l_first[S.issue_l + 1] <= c) ++S.issue_l;
    const uint32_t l = S.issue_l, slot = c % RING;
    const uint32_t off = (c - S.l_first[l]) * CHUNK_E;
    const uint32_t n = min(static_cast<uint32_t>(CHUNK_E), S.l_cnt[l] - off);
    const uint2* src = sd.ent + static_cast<size_t>(S.lists[l]) * sd.cap2 + S.l_beg[l] + off;
    S.c_list[slot] = l;
    S.c_cnt[slot] = n;
    // the 16-byte aligned superset may include one entry of a neighbour block
    // or one slot past n_used: only positions inside [lo, hi) are accumulated
    const uint32_t pos = S.l_beg[l] + off;
    S.c_vlo[slot] = S.l_lo[l] > pos ? S.l_lo[l] - pos : 0u;
    S.c_vhi[slot] = min(n, S.l_hi[l] - pos);
    mbar_expect_tx(&S.bar[slot], n * 8);
    bulk_g2s(stage + slot * CHUNK_E, src, n * 8, &S.bar[slot]);
}

// plan the chunk stream (bounds prefetched by route) and launch the first RING
// bulk copies; thread 0 is the producer. Called right after route's barrier.
__device__ void gather_issue(SelHdr& S, const SessionDev& sd, uint2* stage) {
    if (threadIdx.x != 0) return;
    uint32_t nch = 0;
    for (uint32_t l = 0; l < S.nl; ++l) {
        const uint32_t beg = S.l_lo[l], end = S.l_hi[l];
        const uint32_t ab = beg & ~1u;
        const uint32_t ae = end > beg ? ((end + 1) & ~1u) : ab;  // cap2 is even
        S.l_beg[l] = ab;
        S.l_cnt[l] = ae - ab;
        S.l_first[l] = nch;
        nch += div_up(ae - ab, CHUNK_E);
    }
    S.l_first[S.nl] = nch;
    S.nchunk = nch;
    S.issue_l = 0;
    for (int r = 0; r < RING; ++r) {
        mbar_init(&S.bar[r], 1);
        mbar_init(&S.empty[r], SEL_WARPS);
    }
    fence_mbar_init();
    fence_proxy_async();  // the ring reuses bytes the generic proxy just wrote
    for (uint32_t c = 0; c < nch && c < static_cast<uint32_t>(RING); ++c) issue_chunk(S, sd, stage, c);
}

// Consumers: chunks of one list touch distinct keys, so warps only need a
// block barrier where a new list starts (fixed per-key accumulation order);
// slot reuse is tracked per slot by an `empty` mbarrier (one arrival per warp),
// which the producer waits on before refilling the slot.
__device__ void gather_consume(SelHdr& S, const SessionDev& sd, uint2* stage, double* acc,
                               uint32_t k0) {
    const uint32_t nch = S.nchunk;
    uint32_t cur = 0;  // list of chunk c
    for (uint32_t c = 0; c < nch; ++c) {
        const uint32_t slot = c % RING, par = (c / RING) & 1u;
        if (S.l_first[cur + 1] <= c) {  // chunk c opens a new list (skip empty ones)
            while (S.l_first[cur + 1] <= c) ++cur;
            if (c > 0) __syncthreads();  // previous list fully accumulated
        }
        mbar_wait(&S.bar[slot], par);
        const uint32_t n = S.c_cnt[slot];
        const uint32_t vlo = S.c_vlo[slot], vhi = S.c_vhi[slot];
        const double w = sd.weights[S.lsub[cur]];
        const uint4* e4 = reinterpret_cast<const uint4*>(stage + slot * CHUNK_E);
        for (uint32_t p = threadIdx.x; p < (n >> 1); p += blockDim.x) {
            const uint4 v = e4[p];
            if (2 * p >= vlo && 2 * p < vhi) acc_entry(acc, v.x, v.y, w, k0);
            if (2 * p + 1 >= vlo && 2 * p + 1 < vhi) acc_entry(acc, v.z, v.w, w, k0);
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&S.empty[slot]);
        if (threadIdx.x == 0 && c + RING < nch) {
            mbar_wait(&S.empty[slot], par);  // every warp is done with chunk c
            issue_chunk(S, sd, stage, c + RING);
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Phase 3: cluster-wide selection of the `need` best pool keys.
// Result (on every CTA): S.b_tk / S.b_tx such that a pool key is selected iff
// key > tk || (key == tk && index < tx).
// ---------------------------------------------------------------------------
struct Keys {
    unsigned long long* k;  // local pool keys (0 = not in pool)
    uint32_t n;
};

// Finish on CTA 0: the bucket's members (pred) from every CTA are copied to
// CTA 0, which finds the rem-th by (key desc, index asc). cnt_of(c) = members
// on CTA c. Publishes b_tk / b_tx on every CTA.
template <class Pred, class CountOf>
__device__ void rank_on_leader(cg::cluster_group& cl, SelHdr& S, SelectView& V, const Keys& kv,
                               uint32_t k0, uint32_t rem, uint32_t bucket, Pred pred,
                               CountOf cnt_of) {
    const int rank = cl.block_rank(), cs = cl.num_blocks();
    const uint32_t tid = threadIdx.x;
    if (tid < 32) {
        uint32_t before, total;
        warp_rank_scan(cs, rank, cnt_of, before, total);
        if (tid == 0) {
            S.b_off = before;
            S.wpos = 0;
        }
    }
    __syncthreads();
    unsigned long long* dk = remote(cl, V.skey, 0);
    uint32_t* di = remote(cl, V.sidx, 0);
    const uint32_t off = S.b_off;
    for (uint32_t l = tid; l < kv.n; l += blockDim.x) {
        const unsigned long long k = kv.k[l];
        if (k && pred(l, k)) {
            const uint32_t p = off + atomicAdd(&S.wpos, 1u);
            dk[p] = k;
            di[p] = k0 + l;
        }
    }
    cl.sync();  // bucket gathered on CTA 0
    if (rank == 0) {
        for (uint32_t e = tid; e < bucket; e += blockDim.x) {
            const unsigned long long ke = V.skey[e];
            const uint32_t ie = V.sidx[e];
            uint32_t r = 0;
            for (uint32_t f = 0; f < bucket; ++f) {
                const unsigned long long kf = V.skey[f];
                r += (kf > ke) || (kf == ke && V.sidx[f] < ie);
            }
            if (r == rem - 1) {
                S.x_tk = ke;
                S.x_tx = ie + 1;
            }
        }
    }
    cl.sync();  // threshold published by CTA 0
    if (tid == 0) {
        S.b_tk = *remote(cl, &S.x_tk, 0);
        S.b_tx = *remote(cl, &S.x_tx, 0);
    }
    __syncthreads();
}

// Exact ties at key == tk: the rem-th smallest index among them, cluster-wide.
template <class Pred, class CountOf>
__device__ void resolve_ties(cg::cluster_group& cl, SelHdr& S, const Keys& kv, uint32_t k0,
                             unsigned long long tk, uint32_t rem, Pred pred, CountOf cnt_of) {
    const int rank = cl.block_rank(), cs = cl.num_blocks();
    if (threadIdx.x < 32) {
        uint32_t before, total;
        warp_rank_scan(cs, rank, cnt_of, before, total);
        if (threadIdx.x == 0) S.b_off = before;
    }
    __syncthreads();
    const uint32_t before = S.b_off;
    const uint32_t mine = cnt_of(rank);
    if (rem > before && rem <= before + mine) {
        const uint32_t want = rem - before;  // 1-based among local ties
        const uint32_t chunk = div_up(kv.n, blockDim.x);
        const uint32_t c0 = min(kv.n, threadIdx.x * chunk), c1 = min(kv.n, c0 + chunk);
        uint32_t n = 0;
        for (uint32_t l = c0; l < c1; ++l) n += (kv.k[l] == tk && pred(l, tk));
        uint32_t ex, dummy, tot, tot2;
        block_scan2(S, n, 0, ex, dummy, tot, tot2);
        if (want > ex && want <= ex + n) {
            uint32_t seen = ex;
            for (uint32_t l = c0; l < c1; ++l)
                if (kv.k[l] == tk && pred(l, tk) && ++seen == want) {
                    *remote(cl, &S.x_tx, 0) = k0 + l + 1;
                    break;
                }
        }
    }
    cl.sync();
    if (threadIdx.x == 0) {
        S.b_tk = tk;
        S.b_tx = *remote(cl, &S.x_tx, 0);
    }
    __syncthreads();
}

// Distributed histogram: local hist (nb bins, already filled) -> CTA r reduces
// slice r across the cluster -> every CTA locates the bin holding the rem-th
// largest. Leaves b_dsel / b_cabove / b_bucket. Two cluster barriers.
__device__ void cluster_hist_pick(cg::cluster_group& cl, SelHdr& S, SelectView& V, uint32_t* hist,
                                  uint32_t nb, uint32_t rem) {
    const int rank = cl.block_rank(), cs = cl.num_blocks();
    const uint32_t tid = threadIdx.x;
    cl.sync();  // local histograms complete
    const uint32_t sl = div_up(nb, cs);
    const uint32_t lo = min(nb, rank * sl), hi = min(nb, lo + sl);
    uint32_t part = 0;
    for (uint32_t i = lo + tid; i < hi; i += blockDim.x) {
        uint32_t v = 0;
        for (int c = 0; c < cs; ++c) v += remote(cl, hist, c)[i];
        V.ghist[i] = v;
        part += v;
    }
    part = block_sum(S, part);
    if (tid == 0) S.x_slice_total = part;
    cl.sync();  // reduced slices + slice totals published
    if (tid < 32) {
        const int ln = tid;
        const uint32_t st = ln < cs ? *remote(cl, &S.x_slice_total, ln) : 0;
        uint32_t suf = st;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o);
            if (ln + o < 32) suf += x;
        }
        const uint32_t above = suf - st;
        const bool hit = (ln < cs) && st > 0 && above < rem && suf >= rem;
        const unsigned hm = __ballot_sync(0xffffffffu, hit);
        const int sstar = __ffs(hm) - 1;
        const uint32_t cab = __shfl_sync(0xffffffffu, above, sstar);
        const uint32_t slo = min(nb, sstar * sl), shi = min(nb, slo + sl);
        const uint32_t* src = remote(cl, V.ghist, sstar);
        for (uint32_t i = slo + ln; i < shi; i += 32) V.gcopy[i] = src[i];
        __syncwarp();
        if (ln == 0) {
            uint32_t c = cab, dd = shi;
            while (dd > slo) {
                --dd;
                const uint32_t h = V.gcopy[dd];
                if (c + h >= rem) break;
                c += h;
            }
            S.b_dsel = dd;
            S.b_cabove = c;
            S.b_bucket = V.gcopy[dd];
        }
    }
    __syncthreads();
}

// 64-bit radix refinement restricted to keys with pred(l, k) (fallback path).
template <class Pred>
__device__ void radix_refine(cg::cluster_group& cl, SelHdr& S, SelectView& V, const Keys& kv,
                             uint32_t k0, uint32_t rem, unsigned long long gmin,
                             unsigned long long gmax, Pred pred) {
    const uint32_t tid = threadIdx.x;
    if (gmin == gmax) {
        resolve_ties(cl, S, kv, k0, gmax, rem, pred, [&](int c) { return *remote(cl, &S.x_cnt, c); });
        return;
    }
    int pshift = 64 - __clzll(static_cast<long long>(gmax ^ gmin));
    unsigned long long prefix = pshift == 64 ? 0ull : (gmax >> pshift);
    bool use_surv = false;
    for (int pass = 0;; ++pass) {
        const int shift = pshift > HB_BITS ? pshift - HB_BITS : 0;
        const int nbits = pshift - shift;
        const uint32_t nb = 1u << nbits;
        uint32_t* hist = V.hist[pass & 1];
        for (uint32_t i = tid; i < nb; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        auto cand = [&](uint32_t l, unsigned long long k) {
            return k && pred(l, k) && (pshift == 64 || (k >> pshift) == prefix);
        };
        if (use_surv) {
            for (uint32_t s = tid; s < S.surv_count; s += blockDim.x) {
                const unsigned long long k = kv.k[V.surv[s]];
                atomicAdd(&hist[(k >> shift) & (nb - 1)], 1u);
            }
        } else {
            for (uint32_t l = tid; l < kv.n; l += blockDim.x) {
                const unsigned long long k = kv.k[l];
                if (cand(l, k)) atomicAdd(&hist[(k >> shift) & (nb - 1)], 1u);
            }
        }
        cluster_hist_pick(cl, S, V, hist, nb, rem);
        const uint32_t dsel = S.b_dsel;
        rem -= S.b_cabove;
        const uint32_t bucket = S.b_bucket;
        prefix = (pshift == 64 ? 0ull : (prefix << nbits)) | dsel;
        pshift = shift;
        auto member = [&](uint32_t l, unsigned long long k) {
            return pred(l, k) && (k >> pshift) == prefix;
        };
        auto cnt_of = [&](int c) { return remote(cl, hist, c)[dsel]; };
        if (bucket == rem) {  // the whole bucket is taken
            if (tid == 0) {
                S.b_tk = (prefix << pshift) - 1;
                S.b_tx = 0;
            }
            __syncthreads();
            return;
        }
        if (pshift == 0) {  // exact ties at key == prefix
            resolve_ties(cl, S, kv, k0, prefix, rem, member, cnt_of);
            return;
        }
        if (bucket <= static_cast<uint32_t>(SURV_MAX)) {
            rank_on_leader(cl, S, V, kv, k0, rem, bucket, member, cnt_of);
            return;
        }
        const uint32_t mine = hist[dsel];
        if (mine <= static_cast<uint32_t>(SURV_LOCAL)) {
            if (tid == 0) S.nsv = 0;
            __syncthreads();
            if (use_surv) {
                const uint32_t n0 = S.surv_count;
                uint16_t keep[SURV_LOCAL / SEL_THREADS];
                uint32_t nk = 0;
                for (uint32_t s = tid, u = 0; s < n0 && u < SURV_LOCAL / SEL_THREADS;
                     s += blockDim.x, ++u) {
                    const unsigned long long k = kv.k[V.surv[s]];
                    if ((k >> pshift) == prefix) keep[nk++] = V.surv[s];
                }
                __syncthreads();
                for (uint32_t u = 0; u < nk; ++u) V.surv[atomicAdd(&S.nsv, 1u)] = keep[u];
            } else {
                for (uint32_t l = tid; l < kv.n; l += blockDim.x) {
                    const unsigned long long k = kv.k[l];
                    if (k && member(l, k)) V.surv[atomicAdd(&S.nsv, 1u)] = static_cast<uint16_t>(l);
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

// (cnt, kmax, kmin): this thread's pool statistics from the key transform
__device__ void select_threshold(cg::cluster_group& cl, SelHdr& S, SelectView& V, const Keys& kv,
                                 uint32_t k0, uint32_t need, uint32_t cnt,
                                 unsigned long long kmax, unsigned long long kmin) {
    const int cs = cl.num_blocks();
    const uint32_t tid = threadIdx.x;
    // ---- pool statistics: count, max, min key ----
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
        for (int i = 0; i < SEL_WARPS; ++i) {
            c += S.r32a[i];
            a = S.r64a[i] > a ? S.r64a[i] : a;
            b = S.r64b[i] < b ? S.r64b[i] : b;
        }
        S.x_cnt = c;
        S.x_kmax = a;
        S.x_kmin = b;
    }
    cl.sync();
    if (tid < 32) {
        uint32_t c = 0;
        unsigned long long a = 0, b = ~0ull;
        if (ln < cs) {
            c = *remote(cl, &S.x_cnt, ln);
            a = *remote(cl, &S.x_kmax, ln);
            b = *remote(cl, &S.x_kmin, ln);
        }
        c = warp_sum(c);
        for (int o = 16; o; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, a, o);
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, b, o);
            a = x > a ? x : a;
            b = y < b ? y : b;
        }
        if (ln == 0) {
            S.b_total = c;
            S.b_gmax = a;
            S.b_gmin = b;
        }
    }
    __syncthreads();
    const uint32_t total = S.b_total;
    const unsigned long long gmax = S.b_gmax, gmin = S.b_gmin;
    if (need == 0 || total <= need) {  // nothing / everything from the pool
        if (tid == 0) {
            S.b_tk = need == 0 ? ~0ull : 0ull;
            S.b_tx = 0;
        }
        __syncthreads();
        return;
    }
    auto any = [](uint32_t, unsigned long long) { return true; };
    if (gmax == gmin) {  // all pool keys tie: lowest indices win
        resolve_ties(cl, S, kv, k0, gmax, need, any, [&](int c) { return *remote(cl, &S.x_cnt, c); });
        return;
    }
    // ---- one linear-bucket pass in the fp64 domain ----
    // bucket(s) = min(HB-1, floor((s - smin) * HB/(smax - smin))) is monotone
    // non-decreasing in s under IEEE rounding, so the bucket holding the
    // need-th largest key is exact; equal keys share a bucket.
    const double smin = key_double(gmin), smax = key_double(gmax);
    const double scale = static_cast<double>(HB) / (smax - smin);
    auto bucket_of = [&](unsigned long long k) {
        const double f = (key_double(k) - smin) * scale;
        return f >= static_cast<double>(HB - 1) ? static_cast<uint32_t>(HB - 1)
                                                : static_cast<uint32_t>(f);
    };
    uint32_t* hist = V.hist[0];
    for (uint32_t i = tid; i < static_cast<uint32_t>(HB); i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint32_t l = tid; l < kv.n; l += blockDim.x) {
        const unsigned long long k = kv.k[l];
        if (k) atomicAdd(&hist[bucket_of(k)], 1u);
    }
    cluster_hist_pick(cl, S, V, hist, HB, need);
    const uint32_t dsel = S.b_dsel;
    const uint32_t rem = need - S.b_cabove;
    const uint32_t bucket = S.b_bucket;
    auto member = [&](uint32_t, unsigned long long k) { return bucket_of(k) == dsel; };
    auto cnt_of = [&](int c) { return remote(cl, hist, c)[dsel]; };
    if (bucket <= static_cast<uint32_t>(SURV_MAX)) {
        rank_on_leader(cl, S, V, kv, k0, rem, bucket, member, cnt_of);
        return;
    }
    // ---- fallback: 64-bit radix within the (large) bucket ----
    unsigned long long bmax = 0, bmin = ~0ull;
    uint32_t bc = 0;
    for (uint32_t l = tid; l < kv.n; l += blockDim.x) {
        const unsigned long long k = kv.k[l];
        if (k && member(l, k)) {
            bmax = k > bmax ? k : bmax;
            bmin = k < bmin ? k : bmin;
            ++bc;
        }
    }
    for (int o = 16; o; o >>= 1) {
        bc += __shfl_xor_sync(0xffffffffu, bc, o);
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, bmax, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, bmin, o);
        bmax = a > bmax ? a : bmax;
        bmin = b < bmin ? b : bmin;
    }
    if (ln == 0) {
        S.r32a[w] = bc;
        S.r64a[w] = bmax;
        S.r64b[w] = bmin;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t c = 0;
        unsigned long long a = 0, b = ~0ull;
        for (int i = 0; i < SEL_WARPS; ++i) {
            c += S.r32a[i];
            a = S.r64a[i] > a ? S.r64a[i] : a;
            b = S.r64b[i] < b ? S.r64b[i] : b;
        }
        S.x_cnt = c;  // per-CTA member count (tie path)
        S.x_bmax = a;
        S.x_bmin = b;
    }
    cl.sync();
    if (tid < 32) {
        unsigned long long a = 0, b = ~0ull;
        if (ln < cs) {
            a = *remote(cl, &S.x_bmax, ln);
            b = *remote(cl, &S.x_bmin, ln);
        }
        for (int o = 16; o; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, a, o);
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, b, o);
            a = x > a ? x : a;
            b = y < b ? y : b;
        }
        if (ln == 0) {
            S.b_gmax = a;
            S.b_gmin = b;
        }
    }
    __syncthreads();
    radix_refine(cl, S, V, kv, k0, rem, S.b_gmin, S.b_gmax, member);
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SEL_THREADS, 2)
select_kernel(const DecodeProblem* __restrict__ probs, const RoutePlan* __restrict__ plans,
              uint32_t kpc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SelHdr& S = *reinterpret_cast<SelHdr*>(smem_raw);
    unsigned char* region = smem_raw + ((sizeof(SelHdr) + 127) & ~size_t(127));
    uint2* stage = reinterpret_cast<uint2*>(region);
    SelectView& V = *reinterpret_cast<SelectView*>(region);
    double* acc = reinterpret_cast<double*>(region + REGION_BYTES);
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank(), cs = cl.num_blocks();
    const DecodeProblem& P = probs[blockIdx.x / cs];
    const SessionDev& sd = *P.s;
    const uint32_t tid = threadIdx.x, N = P.N, K = P.K;
    const bool leader = rank == 0;
    const uint32_t k0 = rank * kpc;
    const uint32_t k1 = min(N, k0 + kpc);
    const uint32_t nloc = k1 > k0 ? k1 - k0 : 0;

    if (tid == 0) {
        S.zero_mask = 0;
        S.nl = 0;
        S.surv_count = 0;
    }
    __syncthreads();
    unsigned long long* prof = P.prof ? P.prof + rank * 8 : nullptr;
    auto phase = [&](int i) {
        if (prof && tid == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            prof[i] = t;
        }
    };
    phase(0);

    // ---- 1+2: candidate scores of this CTA's key range ----
    if (P.mode & MODE_SEARCH) {
        load_plan(S, plans[blockIdx.x / cs], rank);
        phase(1);
        if (nloc) gather_issue(S, sd, stage);  // TMA copies in flight ...
        for (uint32_t l = tid; l < kpc; l += blockDim.x)  // ... while acc is reset
            acc[l] = __longlong_as_double(static_cast<long long>(ABSENT));
        __syncthreads();
        phase(2);
        if (nloc) gather_consume(S, sd, stage, acc, k0);
        phase(3);
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
    uint32_t pcnt = 0;
    unsigned long long pmax = 0, pmin = ~0ull;
    for (uint32_t l = tid; l < nloc; l += blockDim.x) {
        const uint32_t i = k0 + l;
        const double v = acc[l];
        unsigned long long key = 0;
        if (i < wlo)
            key = is_absent(v) ? 0ull : ordkey(v);
        else if (!pt)
            key = ordkey(is_absent(v) ? 0.0 : v);
        keys[l] = key;
        if (key) {
            ++pcnt;
            pmax = key > pmax ? key : pmax;
            pmin = key < pmin ? key : pmin;
        }
    }
    __syncthreads();
    Keys kv{keys, nloc};
    phase(4);
    select_threshold(cl, S, V, kv, k0, need, pcnt, pmax, pmin);
    phase(5);
    const unsigned long long tk = S.b_tk;
    const uint32_t tx = S.b_tx;

    // ---- 4: emit the selected set in ascending order (+ newest-first padding) ----
    // Warp w owns keys [w*span, (w+1)*span), 32 at a time: ballots give each
    // key's rank among the selected / untaken keys, so index writes coalesce.
    const int w = tid >> 5, ln = tid & 31;
    const uint32_t span = div_up(div_up(nloc, SEL_WARPS), 32) * 32;
    const uint32_t wb = min(nloc, w * span), we = min(nloc, wb + span);
    auto picked = [&](uint32_t l) {
        const uint32_t i = k0 + l;
        const unsigned long long k = keys[l];
        return i >= f_lo || (k && (k > tk || (k == tk && i < tx)));
    };
    uint32_t wsel = 0, wunt = 0;
    for (uint32_t g = wb; g < we; g += 32) {
        const uint32_t l = g + ln;
        const bool in = l < we;
        const unsigned ms = __ballot_sync(0xffffffffu, in && picked(l));
        const unsigned mu = __ballot_sync(0xffffffffu, in) & ~ms;
        wsel += __popc(ms);
        wunt += __popc(mu);
    }
    if (ln == 0) {
        S.r32a[w] = wsel;
        S.r32b[w] = wunt;
    }
    __syncthreads();
    uint32_t esel = 0, eunt = 0, tsel = 0, tunt = 0;
#pragma unroll
    for (int i = 0; i < SEL_WARPS; ++i) {
        if (i < w) {
            esel += S.r32a[i];
            eunt += S.r32b[i];
        }
        tsel += S.r32a[i];
        tunt += S.r32b[i];
    }
    if (tid == 0) {
        S.x_nsel = tsel;
        S.x_nunt = tunt;
    }
    cl.sync();
    if (tid < 32) {
        // per-CTA padding share and output base, one lane per cluster rank
        const uint32_t ns = ln < cs ? *remote(cl, &S.x_nsel, ln) : 0;
        const uint32_t nu = ln < cs ? *remote(cl, &S.x_nunt, ln) : 0;
        const uint32_t all_sel = warp_sum(ns);
        uint32_t suf = nu;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o);
            if (ln + o < 32) suf += x;
        }
        const uint32_t above = suf - nu;
        const uint32_t pad = K > all_sel ? K - all_sel : 0;
        const uint32_t tk_l = pad > above ? min(pad - above, nu) : 0;
        const uint32_t cnt = ns + tk_l;
        uint32_t inc = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
            if (ln >= o) inc += x;
        }
        if (ln == rank) {
            S.b_base = inc - cnt;
            S.b_take = tk_l;
        }
    }
    __syncthreads();
    {
        // padded keys: the `take` highest-index untaken keys of this CTA
        const uint32_t pad_from = tunt - S.b_take;  // untaken rank >= pad_from is padded
        uint32_t pos = S.b_base + esel + (eunt > pad_from ? eunt - pad_from : 0);
        uint32_t u = eunt;
        const unsigned lt = (1u << ln) - 1u;
        for (uint32_t g = wb; g < we; g += 32) {
            const uint32_t l = g + ln;
            const bool in = l < we;
            const bool ps = in && picked(l);
            const unsigned mu = __ballot_sync(0xffffffffu, in && !ps);
            const uint32_t urank = u + __popc(mu & lt);  // this key's untaken rank
            const bool out = ps || (in && !ps && urank >= pad_from);
            const unsigned mo = __ballot_sync(0xffffffffu, out);
            if (out) P.sel[pos + __popc(mo & lt)] = k0 + l;
            pos += __popc(mo);
            u += __popc(mu);
        }
    }
    if (leader && tid == 0) reinterpret_cast<DecodeReport*>(P.rep)->k = K;
    phase(6);
    cl.sync();  // nobody exits while a peer may still read its shared memory
}

size_t select_smem_bytes(uint32_t kpc) {
    return ((sizeof(SelHdr) + 127) & ~size_t(127)) + REGION_BYTES +
           static_cast<size_t>(kpc) * sizeof(double);
}

cudaError_t launch_select(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                          uint32_t kpc, uint32_t cs, cudaStream_t st) {
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
    cfg.blockDim = dim3(SEL_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, select_kernel, probs, plans, kpc);
}

}  // namespace csa
