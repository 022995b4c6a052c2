// tables.cuh — maintenance of one index-sorted table (see common.cuh):
// compaction, key-block offsets and the low (eviction-order) buffer refill.
// Shared by the streaming insert (insert.cu) and the offline build (build.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace csa {

// eviction key: ascending = evicted first (score asc, then key desc)
__device__ __forceinline__ unsigned long long evkey(float score, uint32_t key) {
    uint32_t b = __float_as_uint(score);
    if ((b << 1) == 0) b = 0;  // -0.0 == +0.0
    const uint32_t o = (b >> 31) ? ~b : (b | 0x80000000u);
    return (static_cast<unsigned long long>(o) << 32) | static_cast<uint32_t>(~key);
}

// a evicted before b ?
__device__ __forceinline__ bool ev_before(float sa, uint32_t ka, float sb, uint32_t kb) {
    return sa != sb ? sa < sb : ka > kb;
}

struct RefillSmem {
    uint32_t hist[256];
    uint32_t wsum[32];
    unsigned long long bkey[LOW_Q];
    uint32_t bpos[LOW_Q];
    uint32_t cnt;
    unsigned long long b_prefix;
    uint32_t b_rem, b_done;
    int b_shift;
};

__device__ __forceinline__ uint32_t tbl_block_excl_scan(RefillSmem& S, uint32_t v, uint32_t& total) {
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (ln >= o) inc += x;
    }
    __syncthreads();
    if (ln == 31) S.wsum[w] = inc;
    __syncthreads();
    uint32_t pre = 0;
    total = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
        if (i < w) pre += S.wsum[i];
        total += S.wsum[i];
    }
    return pre + inc - v;
}

// CTA-wide min and max of n 64-bit keys (every thread gets both).
constexpr int CK_U = 8;  // independent loads in flight per thread and pass

template <class KeyOf>
__device__ void cta_minmax(RefillSmem& S, uint32_t n, KeyOf key_of, unsigned long long& mn,
                           unsigned long long& mx) {
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const uint32_t span = blockDim.x * CK_U;
    mn = ~0ull;
    mx = 0ull;
    for (uint32_t c0 = 0; c0 < n; c0 += span) {
        unsigned long long kk[CK_U];
#pragma unroll
        for (int u = 0; u < CK_U; ++u) {
            const uint32_t p = c0 + u * blockDim.x + threadIdx.x;
            kk[u] = p < n ? key_of(p) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < CK_U; ++u) {
            if (c0 + u * blockDim.x + threadIdx.x < n) {
                mn = kk[u] < mn ? kk[u] : mn;
                mx = kk[u] > mx ? kk[u] : mx;
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    __syncthreads();  // bkey may hold a previous caller's data
    if (lane == 0) {
        S.bkey[wid] = mn;
        S.bkey[32 + wid] = mx;
    }
    __syncthreads();
    for (uint32_t w = 0; w < nwarp; ++w) {
        mn = S.bkey[w] < mn ? S.bkey[w] : mn;
        mx = S.bkey[32 + w] > mx ? S.bkey[32 + w] : mx;
    }
    __syncthreads();
}

// k-th largest (1-based) of n UNIQUE 64-bit keys whose CTA-wide min and max
// are mn, mx: radix passes of <= BITS bits below the prefix all keys share
// (table scores sit in a narrow band, so the top byte alone would put nearly
// every key in one bin), early exit; returns T such that exactly k keys are
// >= T. hist holds 2^BITS counters. Histogram updates are warp-aggregated
// (one atomic per distinct digit per warp instruction), each thread keeps
// CK_U loads in flight, and warp 0 finds the threshold bin with a lane scan.
template <int BITS, class KeyOf>
__device__ unsigned long long cta_kth_largest_mm(RefillSmem& S, uint32_t* hist, uint32_t n, uint32_t k,
                                                 unsigned long long mn, unsigned long long mx, KeyOf key_of) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t span = blockDim.x * CK_U;
    if (threadIdx.x == 0) {
        const unsigned long long diff = mn ^ mx;
        const int top = diff ? 64 - __clzll(diff) : 0;  // bits below the common prefix
        S.b_prefix = top == 64 ? 0ull : (mx >> top);
        S.b_shift = top;
        S.b_rem = k;
        S.b_done = top == 0 ? 1u : 0u;  // n == 1 (keys are unique)
    }
    __syncthreads();
    while (!S.b_done) {
        const int pshift = S.b_shift, shift = pshift > BITS ? pshift - BITS : 0;
        const unsigned long long prefix = S.b_prefix;
        const uint32_t dmask = (1u << (pshift - shift)) - 1u;
        for (uint32_t i = threadIdx.x; i <= dmask; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (uint32_t c0 = 0; c0 < n; c0 += span) {
            unsigned long long kk[CK_U];
#pragma unroll
            for (int u = 0; u < CK_U; ++u) {
                const uint32_t p = c0 + u * blockDim.x + threadIdx.x;
                kk[u] = p < n ? key_of(p) : 0ull;
            }
#pragma unroll
            for (int u = 0; u < CK_U; ++u) {
                uint32_t dg = 0xffffffffu;
                if (c0 + u * blockDim.x + threadIdx.x < n && (pshift == 64 || (kk[u] >> pshift) == prefix))
                    dg = static_cast<uint32_t>(kk[u] >> shift) & dmask;
                const uint32_t peers = __match_any_sync(0xffffffffu, dg);
                if (dg != 0xffffffffu && lane == static_cast<uint32_t>(__ffs(peers) - 1))
                    atomicAdd(&hist[dg], static_cast<uint32_t>(__popc(peers)));
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // lane l holds bins [hi - per, hi), hi = nb - per * l (descending)
            const int nb = static_cast<int>(dmask) + 1, per = (nb + 31) / 32;
            const int hi = nb - per * static_cast<int>(lane), lo = hi - per > 0 ? hi - per : 0;
            uint32_t sum = 0;
            for (int b = lo; b < hi; ++b) sum += hist[b];
            uint32_t inc = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= static_cast<uint32_t>(o)) inc += x;
            }
            const uint32_t rem = S.b_rem, ex = inc - sum;
            const uint32_t hit = __ballot_sync(0xffffffffu, ex < rem && inc >= rem);
            __syncwarp();  // every lane's reads of the state before the hit lane writes it
            if (lane == static_cast<uint32_t>(__ffs(hit) - 1)) {
                uint32_t c = ex;
                int dsel;
                for (dsel = hi - 1; dsel > lo; --dsel) {
                    if (c + hist[dsel] >= rem) break;
                    c += hist[dsel];
                }
                const uint32_t bucket = hist[dsel];
                S.b_rem = rem - c;
                S.b_prefix = (pshift == 64 ? 0ull : (prefix << (pshift - shift))) | static_cast<unsigned>(dsel);
                S.b_shift = shift;
                if (bucket == rem - c || shift == 0) S.b_done = 1;
            }
        }
        __syncthreads();
    }
    return S.b_shift == 64 ? 0ull : (S.b_prefix << S.b_shift);
}

// k-th largest of n unique keys (8-bit digits over S.hist)
template <class KeyOf>
__device__ unsigned long long cta_kth_largest(RefillSmem& S, uint32_t n, uint32_t k, KeyOf key_of) {
    unsigned long long mn, mx;
    cta_minmax(S, n, key_of, mn, mx);
    return cta_kth_largest_mm<8>(S, S.hist, n, k, mn, mx, key_of);
}

// Order-preserving CTA compaction of items [0, n): thread x handles the CC_U
// consecutive items [c0 + x*CC_U, ...) of each span, so one block scan covers
// CC_U items per thread and their loads are in flight together. keep(p, v)
// decides, emit(pos, p, v) writes; in_place = every read of a span completes
// before any write (a compaction into the array it reads).
constexpr int CC_U = 4;

template <class Load, class Keep, class Emit>
__device__ uint32_t cta_compact(RefillSmem& S, uint32_t n, bool in_place, Load load, Keep keep, Emit emit) {
    using V = decltype(load(0u));
    const uint32_t span = blockDim.x * CC_U;
    uint32_t out = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += span) {
        const uint32_t p0 = c0 + threadIdx.x * CC_U;
        V v[CC_U];
        uint32_t flags = 0;
#pragma unroll
        for (int u = 0; u < CC_U; ++u)
            if (p0 + u < n) v[u] = load(p0 + u);
#pragma unroll
        for (int u = 0; u < CC_U; ++u)
            if (p0 + u < n && keep(p0 + u, v[u])) flags |= 1u << u;
        uint32_t tot;
        uint32_t pos = out + tbl_block_excl_scan(S, static_cast<uint32_t>(__popc(flags)), tot);
        if (in_place) __syncthreads();  // whole span read before any write
#pragma unroll
        for (int u = 0; u < CC_U; ++u)
            if (flags & (1u << u)) emit(pos++, p0 + u, v[u]);
        out += tot;
        if (in_place) __syncthreads();
    }
    return out;
}

// Compact table t (drop tombstones, keep key order), rebuild blk_off for
// blocks [0, last_blk], refill its low buffer with the LOW_Q lowest entries.
__device__ inline void refill_table(RefillSmem& S, const SessionDev& sd, uint32_t t, uint32_t last_blk) {
    uint2* e = sd.ent + static_cast<size_t>(t) * sd.cap2;
    uint32_t* bo = sd.blk_off + static_cast<size_t>(t) * sd.nb_stride;
    const uint32_t n = sd.n_used[t];
    // 1. in-place order-preserving compaction
    const uint32_t nlive = cta_compact(
        S, n, true, [&](uint32_t p) { return e[p]; }, [](uint32_t, uint2 v) { return !(v.x & TOMB); },
        [&](uint32_t pos, uint32_t, uint2 v) { e[pos] = v; });
    __syncthreads();
    // 2. key-block offsets: bo[kb] = first position with key >= kb*KEY_BLOCK
    for (uint32_t p = threadIdx.x; p <= nlive; p += blockDim.x) {
        const uint32_t prevb = p == 0 ? 0u : (e[p - 1].x >> KEY_BLOCK_SHIFT) + 1;
        const uint32_t curb = p == nlive ? last_blk + 1 : (e[p].x >> KEY_BLOCK_SHIFT);
        for (uint32_t kb = prevb; kb <= curb && kb <= last_blk; ++kb) bo[kb] = p;
    }
    // 3. low buffer: the LOW_Q smallest eviction keys = the LOW_Q largest of
    //    their complements
    const uint32_t want = nlive < static_cast<uint32_t>(LOW_Q) ? nlive : LOW_Q;
    unsigned long long lim = ~0ull;  // inclusive eviction-key limit
    if (want < nlive)
        lim = ~cta_kth_largest(S, nlive, want, [&](uint32_t p) {
            const uint2 v = e[p];
            return ~evkey(__uint_as_float(v.y), v.x);
        });
    if (threadIdx.x == 0) S.cnt = 0;
    __syncthreads();
    // collect entries with eviction key inside the limit (exactly `want`)
    for (uint32_t p = threadIdx.x; p < nlive; p += blockDim.x) {
        const uint2 v = e[p];
        const unsigned long long k = evkey(__uint_as_float(v.y), v.x);
        if (k <= lim) {
            const uint32_t slot = atomicAdd(&S.cnt, 1u);
            if (slot < LOW_Q) {
                S.bkey[slot] = k;
                S.bpos[slot] = p;
            }
        }
    }
    __syncthreads();
    const uint32_t cnt = S.cnt < static_cast<uint32_t>(LOW_Q) ? S.cnt : LOW_Q;
    // bitonic sort (descending eviction key) over LOW_Q slots, padding = 0
    for (uint32_t i = threadIdx.x; i < static_cast<uint32_t>(LOW_Q); i += blockDim.x)
        if (i >= cnt) {
            S.bkey[i] = 0;
            S.bpos[i] = 0;
        }
    __syncthreads();
    for (uint32_t k = 2; k <= static_cast<uint32_t>(LOW_Q); k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < static_cast<uint32_t>(LOW_Q); i += blockDim.x) {
                const uint32_t ij = i ^ j;
                if (ij > i) {
                    const bool desc = (i & k) == 0;
                    const unsigned long long a = S.bkey[i], b = S.bkey[ij];
                    if (desc ? (a < b) : (a > b)) {
                        S.bkey[i] = b;
                        S.bkey[ij] = a;
                        const uint32_t t2 = S.bpos[i];
                        S.bpos[i] = S.bpos[ij];
                        S.bpos[ij] = t2;
                    }
                }
            }
            __syncthreads();
        }
    LowEnt* lo = sd.low + static_cast<size_t>(t) * LOW_Q;
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        const uint32_t p = S.bpos[i];
        const uint2 v = e[p];
        LowEnt le;
        le.score = __uint_as_float(v.y);
        le.key = v.x;
        le.pos = p;
        le.pad = 0;
        lo[i] = le;
    }
    if (threadIdx.x == 0) {
        sd.n_used[t] = nlive;
        sd.low_cnt[t] = cnt;
    }
    __syncthreads();
}

}  // namespace csa
