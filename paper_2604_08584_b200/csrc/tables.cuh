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

// Compact table t (drop tombstones, keep key order), rebuild blk_off for
// blocks [0, last_blk], refill its low buffer with the LOW_Q lowest entries.
__device__ inline void refill_table(RefillSmem& S, const SessionDev& sd, uint32_t t, uint32_t last_blk) {
    uint2* e = sd.ent + static_cast<size_t>(t) * sd.cap2;
    uint32_t* bo = sd.blk_off + static_cast<size_t>(t) * sd.nb_stride;
    const uint32_t n = sd.n_used[t];
    // 1. in-place order-preserving compaction, chunk by chunk
    uint32_t out = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += blockDim.x) {
        const uint32_t p = c0 + threadIdx.x;
        uint2 v = make_uint2(TOMB, 0);
        if (p < n) v = e[p];
        const uint32_t keep = (p < n && !(v.x & TOMB)) ? 1u : 0u;
        uint32_t tot;
        const uint32_t ex = tbl_block_excl_scan(S, keep, tot);
        __syncthreads();  // whole chunk read before any write
        if (keep) e[out + ex] = v;
        out += tot;
        __syncthreads();
    }
    const uint32_t nlive = out;
    // 2. key-block offsets: bo[kb] = first position with key >= kb*KEY_BLOCK
    for (uint32_t p = threadIdx.x; p <= nlive; p += blockDim.x) {
        const uint32_t prevb = p == 0 ? 0u : (e[p - 1].x >> KEY_BLOCK_SHIFT) + 1;
        const uint32_t curb = p == nlive ? last_blk + 1 : (e[p].x >> KEY_BLOCK_SHIFT);
        for (uint32_t kb = prevb; kb <= curb && kb <= last_blk; ++kb) bo[kb] = p;
    }
    // 3. low buffer: the LOW_Q smallest eviction keys, via 8-bit radix passes
    const uint32_t want = nlive < static_cast<uint32_t>(LOW_Q) ? nlive : LOW_Q;
    if (threadIdx.x == 0) {
        S.b_prefix = 0;
        S.b_shift = 64;
        S.b_rem = want;
        S.b_done = (want == nlive) ? 1u : 0u;  // take everything
        S.cnt = 0;
    }
    __syncthreads();
    while (!S.b_done) {
        const int shift = S.b_shift - 8;
        const unsigned long long prefix = S.b_prefix;
        const int pshift = S.b_shift;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) S.hist[i] = 0;
        __syncthreads();
        for (uint32_t p = threadIdx.x; p < nlive; p += blockDim.x) {
            const uint2 v = e[p];
            const unsigned long long k = evkey(__uint_as_float(v.y), v.x);
            if (pshift < 64 && (k >> pshift) != prefix) continue;
            atomicAdd(&S.hist[(k >> shift) & 0xff], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t c = 0, dsel = 0;
            for (dsel = 0; dsel < 256; ++dsel) {
                if (c + S.hist[dsel] >= S.b_rem) break;
                c += S.hist[dsel];
            }
            const uint32_t bucket = S.hist[dsel];
            S.b_rem -= c;
            S.b_prefix = (pshift == 64 ? 0ull : (prefix << 8)) | dsel;
            S.b_shift = shift;
            if (bucket == S.b_rem || shift == 0) S.b_done = 2;
        }
        __syncthreads();
    }
    // collect entries with eviction key inside the threshold
    const unsigned long long lim =
        S.b_done == 1 ? ~0ull : (((S.b_prefix + 1) << S.b_shift) - 1);  // inclusive
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

namespace csa {

// k-th largest (1-based) of n UNIQUE 64-bit keys, CTA-wide 8-bit radix passes
// from the top bit with early exit; returns T such that exactly k keys are >= T.
template <class KeyOf>
__device__ unsigned long long cta_kth_largest(RefillSmem& S, uint32_t n, uint32_t k, KeyOf key_of) {
    if (threadIdx.x == 0) {
        S.b_prefix = 0;
        S.b_shift = 64;
        S.b_rem = k;
        S.b_done = 0;
    }
    __syncthreads();
    while (!S.b_done) {
        const int pshift = S.b_shift, shift = pshift - 8;
        const unsigned long long prefix = S.b_prefix;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) S.hist[i] = 0;
        __syncthreads();
        for (uint32_t p = threadIdx.x; p < n; p += blockDim.x) {
            const unsigned long long key = key_of(p);
            if (pshift < 64 && (key >> pshift) != prefix) continue;
            atomicAdd(&S.hist[(key >> shift) & 0xff], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t c = 0;
            int dsel;
            for (dsel = 255; dsel > 0; --dsel) {
                if (c + S.hist[dsel] >= S.b_rem) break;
                c += S.hist[dsel];
            }
            const uint32_t bucket = S.hist[dsel];
            S.b_rem -= c;
            S.b_prefix = (pshift == 64 ? 0ull : (prefix << 8)) | static_cast<unsigned>(dsel);
            S.b_shift = shift;
            if (bucket == S.b_rem || shift == 0) S.b_done = 1;
        }
        __syncthreads();
    }
    return S.b_prefix << S.b_shift;
}

}  // namespace csa
