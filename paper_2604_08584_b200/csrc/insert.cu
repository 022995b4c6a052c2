// insert.cu — KvStore::append (core.cpp:71-79) + streaming_insert
// (retrieval.cpp:272-301, TopList::try_insert index.cpp:22-44) on sm_100a.
//
// One CTA per session. The new key's index N is larger than every stored key,
// so in the index-sorted layout an admitted entry is a plain append at
// n_used[t]. Eviction removes the TopList back = the live entry first in
// eviction order (score asc, key desc), found in O(1) at the tail of the
// per-table low buffer (kept in DESCENDING eviction order: the next victim is
// low[cnt-1]) and tombstoned in place.
//   A. one thread per (subspace b, centroid j) table: fp64 score of the new key
//      slice, strict-win admission against the victim, tombstone + append;
//   B. one warp per table whose new entry belongs in its low buffer: the
//      buffer is loaded into registers, ranked by ballot and written back
//      shifted by one (two memory round trips, no serial shifting);
//   C. the whole CTA compacts any table whose buffer ran dry or whose slack is
//      used up, rebuilds its key-block offsets and refills the buffer (radix
//      select of the LOW_Q lowest eviction keys).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "tables.cuh"

namespace csa {

constexpr int INS_THREADS = 512;
constexpr int INS_WARPS = INS_THREADS / 32;
constexpr int LQ_PER_LANE = LOW_Q / 32;

struct BufEnt {
    float score;
    uint32_t pos;
    uint32_t cnt;
};

struct InsSmem {
    float ks[DMAX];
    uint32_t zero_mask;
    uint32_t nref, nbuf;
    uint32_t applied;
    uint32_t reflist[MAX_TABLES];  // tables needing compaction + refill
    uint32_t buflist[MAX_TABLES];  // tables whose new entry enters the low buffer
    BufEnt bufent[MAX_TABLES];     // that entry (key = N) + the buffer count
    RefillSmem r;
};

// score of an eviction key (inverse of evkey's order-preserving map)
__device__ __forceinline__ float ev_score(unsigned long long k) {
    const uint32_t o = static_cast<uint32_t>(k >> 32);
    return __uint_as_float((o >> 31) ? (o & 0x7fffffffu) : ~o);
}

// Sharded sessions: the first entry of each table in eviction order on this
// shard (low[cnt-1]); the caller all-reduces (min) over the shards to get the
// global TopList back (score asc, key desc).
__global__ void shard_victim_kernel(const InsertProblem* __restrict__ probs,
                                    unsigned long long* __restrict__ vk) {
    const InsertProblem& P = probs[blockIdx.x];
    const SessionDev& sd = *P.s;
    const uint32_t T = sd.m * sd.C;
    for (uint32_t t = threadIdx.x; t < T; t += blockDim.x) {
        const uint32_t cnt = sd.low_cnt[t];
        unsigned long long k = ~0ull;
        if (cnt) {
            const LowEnt v = sd.low[static_cast<size_t>(t) * LOW_Q + cnt - 1];
            k = evkey(v.score, v.key);
        }
        vk[static_cast<size_t>(blockIdx.x) * T + t] = k;
    }
}

__global__ void __launch_bounds__(INS_THREADS)
insert_kernel(const InsertProblem* __restrict__ probs, const unsigned long long* __restrict__ gvk) {
    __shared__ InsSmem S;
    const InsertProblem& P = probs[blockIdx.x];
    const SessionDev& sd = *P.s;
    const uint32_t d = sd.d, m = sd.m, C = sd.C, T = m * C, N = P.N;
    // KvStore::append rejects a non-finite row before touching the store
    // (core.cpp:71-79): the whole append + insert is skipped and flagged (the
    // host raises DataError), so the KV rows and tables stay as they were
    int kbad = 0, vbad = 0;
    for (uint32_t x = threadIdx.x; x < d; x += blockDim.x) {
        const float kx = P.key[x], vx = P.value[x];
        kbad |= !isfinite(kx);
        vbad |= !isfinite(vx);
        S.ks[x] = kx;
    }
    kbad = __syncthreads_or(kbad);
    vbad = __syncthreads_or(vbad);
    if (kbad | vbad) {  // 1: the key (checked first, as require_finite), 2: the value
        if (threadIdx.x == 0) {
            if (P.bad) *P.bad = kbad ? 1u : 2u;
            P.rep[0] = 0u;
        }
        return;
    }
    // row N lands at tail row N - P (on the owner shard)
    if (sd.owner)
        for (uint32_t x = threadIdx.x; x < d; x += blockDim.x) {
            sd.ktail[static_cast<size_t>(N - sd.P) * d + x] = S.ks[x];
            sd.vtail[static_cast<size_t>(N - sd.P) * d + x] = P.value[x];
        }
    if (threadIdx.x == 0) {
        S.zero_mask = 0;
        S.nref = 0;
        S.nbuf = 0;
        S.applied = 0;
    }
    // this thread's first table's state does not depend on the key: load it
    // now, overlapped with the key load and normalization (non-sharded path;
    // a table is touched by exactly one thread in phase A)
    const bool pf = threadIdx.x < T && sd.L != 0 && !sd.sharded;
    uint32_t pf_nu = 0, pf_live = 0, pf_cnt = 0;
    LowEnt pf_victim{}, pf_lo0{};
    float2 pf_mm{};
    if (pf) {
        const uint32_t t = threadIdx.x;
        pf_nu = sd.n_used[t];
        pf_live = sd.live[t];
        pf_cnt = sd.low_cnt[t];
        pf_mm = sd.tmm[t];
        if (pf_cnt) {
            const LowEnt* lo = sd.low + static_cast<size_t>(t) * LOW_Q;
            pf_lo0 = lo[0];
            if (pf_live >= sd.L) pf_victim = lo[pf_cnt - 1];
        }
    }
    __syncthreads();
    if (sd.normalize_keys && threadIdx.x < m) {
        // normalize_keys: score against the normalized slice (l2_normalize)
        const uint32_t off = sd.offs[threadIdx.x], w = sd.widths[threadIdx.x];
        double n2 = 0.0;
        for (uint32_t t = 0; t < w; ++t) n2 = __fma_rn((double)S.ks[off + t], (double)S.ks[off + t], n2);
        if (n2 == 0.0) {
            atomicOr(&S.zero_mask, 1u << threadIdx.x);
        } else {
            const double inv = 1.0 / sqrt(n2);
            for (uint32_t t = 0; t < w; ++t)
                S.ks[off + t] = __double2float_rn(__dmul_rn((double)S.ks[off + t], inv));
        }
    }
    __syncthreads();
    // ---- A: admission, tombstone, append ----
    uint8_t* mask = reinterpret_cast<uint8_t*>(P.rep + 1);
    const uint32_t new_blk = (N & (KEY_BLOCK - 1)) == 0;
    for (uint32_t t = threadIdx.x; t < T; t += blockDim.x) {
        const uint32_t b = t / C, j = t - b * C;
        const uint32_t off = sd.offs[b], w = sd.widths[b];
        double s = 0.0;
        if (!(S.zero_mask & (1u << b))) {
            const float* c = sd.cent + static_cast<size_t>(C) * off + static_cast<size_t>(j) * w;
            if ((w & 3u) == 0u && ((C * off + j * w) & 3u) == 0u) {  // 16-byte rows: vector loads
                const float4* c4 = reinterpret_cast<const float4*>(c);
#pragma unroll 4
                for (uint32_t x4 = 0; x4 < w / 4; ++x4) {
                    const float4 v = __ldg(c4 + x4);
                    const float* ks = S.ks + off + 4 * x4;
                    s = __fma_rn((double)v.x, (double)ks[0], s);
                    s = __fma_rn((double)v.y, (double)ks[1], s);
                    s = __fma_rn((double)v.z, (double)ks[2], s);
                    s = __fma_rn((double)v.w, (double)ks[3], s);
                }
            } else {
                for (uint32_t x = 0; x < w; ++x) s = __fma_rn((double)__ldg(c + x), (double)S.ks[off + x], s);
            }
        }
        const float sc = __double2float_rn(s);
        // programmatic dependent launch (fused step -> insert): everything
        // above reads only the key, the centroids and table state that the
        // previous kernel does not write; the table writes below wait for it
        // (it gathers these tables). Without the launch attribute: a no-op.
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const bool mine = pf && t == threadIdx.x;  // prefetched above
        uint32_t nu = mine ? pf_nu : sd.n_used[t];
        if (new_blk) sd.blk_off[static_cast<size_t>(t) * sd.nb_stride + (N >> KEY_BLOCK_SHIFT)] = nu;
        uint32_t applied = 0;
        if (sd.L != 0 && sd.sharded) {
            // global TopList semantics over the shards: the list is full when the
            // GLOBAL live count reaches L; a full list admits only a strict win
            // over the global back (gvk, all-reduced); the shard holding it
            // tombstones it, the owner shard appends the new entry
            const uint32_t live_g = sd.live_g[t];
            uint32_t live = sd.live[t];
            uint32_t cnt = sd.low_cnt[t];
            LowEnt* lo = sd.low + static_cast<size_t>(t) * LOW_Q;
            uint2* e = sd.ent + static_cast<size_t>(t) * sd.cap2;
            const bool full = live_g >= sd.L;
            const bool complete = cnt == live;
            bool ok = true, evicted = false;
            if (full) {
                const unsigned long long gv = gvk[static_cast<size_t>(blockIdx.x) * T + t];
                if (!(sc > ev_score(gv))) {
                    ok = false;
                } else if (cnt && evkey(lo[cnt - 1].score, lo[cnt - 1].key) == gv) {
                    e[lo[cnt - 1].pos].x = lo[cnt - 1].key | TOMB;
                    cnt -= 1;
                    live -= 1;
                    evicted = true;
                }
            }
            if (ok) {
                applied = 1;
                float2 mm = sd.tmm[t];  // global bounds, replicated on every shard
                mm = live_g == 0 ? make_float2(sc, sc) : make_float2(fminf(mm.x, sc), fmaxf(mm.y, sc));
                sd.tmm[t] = mm;
                if (!full) sd.live_g[t] = live_g + 1;
                if (sd.owner) {
                    e[nu] = make_uint2(N, __float_as_uint(sc));
                    const uint32_t pos = nu;
                    nu += 1;
                    live += 1;
                    sd.n_used[t] = nu;
                    bool ins;
                    if (cnt == 0)
                        ins = complete;
                    else if (complete && cnt < static_cast<uint32_t>(LOW_Q))
                        ins = true;
                    else
                        ins = ev_before(sc, N, lo[0].score, lo[0].key);
                    if (ins) {
                        const uint32_t k = atomicAdd(&S.nbuf, 1u);
                        S.buflist[k] = t;
                        S.bufent[k] = BufEnt{sc, pos, cnt};
                    } else {
                        sd.low_cnt[t] = cnt;
                        if (cnt == 0 || nu == sd.cap2) S.reflist[atomicAdd(&S.nref, 1u)] = t;
                    }
                } else if (evicted) {
                    sd.low_cnt[t] = cnt;
                    if (cnt == 0 && live > 0) S.reflist[atomicAdd(&S.nref, 1u)] = t;
                }
                sd.live[t] = live;
            }
        } else if (sd.L != 0) {
            const uint32_t live = mine ? pf_live : sd.live[t];
            uint32_t cnt = mine ? pf_cnt : sd.low_cnt[t];
            LowEnt* lo = sd.low + static_cast<size_t>(t) * LOW_Q;
            uint2* e = sd.ent + static_cast<size_t>(t) * sd.cap2;
            const bool full = live >= sd.L;
            const bool complete = cnt == live;  // buffer holds every live entry
            bool ok = true;
            if (full) {
                const LowEnt victim = mine ? pf_victim : lo[cnt - 1];
                if (!(sc > victim.score)) {
                    ok = false;  // strict win required (index.cpp:25)
                } else {
                    e[victim.pos].x = victim.key | TOMB;
                    cnt -= 1;
                }
            }
            if (ok) {
                applied = 1;
                e[nu] = make_uint2(N, __float_as_uint(sc));
                {  // live score bounds (evictions only raise the min: kept as a bound)
                    float2 mm = mine ? pf_mm : sd.tmm[t];
                    mm = live == 0 ? make_float2(sc, sc)
                                   : make_float2(fminf(mm.x, sc), fmaxf(mm.y, sc));
                    sd.tmm[t] = mm;
                }
                const uint32_t pos = nu;
                nu += 1;
                if (!full) sd.live[t] = live + 1;
                sd.n_used[t] = nu;
                // does the new entry belong among the cnt lowest live entries?
                bool ins;
                if (cnt == 0)
                    ins = complete;  // an empty, incomplete buffer is refilled instead
                else if (complete && cnt < static_cast<uint32_t>(LOW_Q))
                    ins = true;
                else {  // lo[0] is the same entry after an eviction (cnt >= 1 left)
                    const LowEnt l0 = mine ? pf_lo0 : lo[0];
                    ins = ev_before(sc, N, l0.score, l0.key);
                }
                if (ins) {
                    const uint32_t k = atomicAdd(&S.nbuf, 1u);
                    S.buflist[k] = t;
                    S.bufent[k] = BufEnt{sc, pos, cnt};
                } else {
                    sd.low_cnt[t] = cnt;
                    if (cnt == 0 || nu == sd.cap2) S.reflist[atomicAdd(&S.nref, 1u)] = t;
                }
            }
        }
        mask[t] = static_cast<uint8_t>(applied);
        if (applied) atomicAdd(&S.applied, 1u);
    }
    __syncthreads();
    // ---- B: warp-cooperative low-buffer insertion ----
    const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
    for (uint32_t k = wid; k < S.nbuf; k += INS_WARPS) {
        const uint32_t t = S.buflist[k];
        const BufEnt be = S.bufent[k];
        const LowEnt ne{be.score, N, be.pos, 0};
        const uint32_t cnt = be.cnt;
        LowEnt* lo = sd.low + static_cast<size_t>(t) * LOW_Q;
        LowEnt v[LQ_PER_LANE];
        uint32_t after = 0;  // entries evicted after the new one precede it
#pragma unroll
        for (int i = 0; i < LQ_PER_LANE; ++i) {
            const uint32_t e = i * 32 + ln;
            if (e < cnt) {
                v[i] = lo[e];
                after += ev_before(v[i].score, v[i].key, ne.score, ne.key) ? 0u : 1u;
            }
        }
        for (int o = 16; o; o >>= 1) after += __shfl_xor_sync(0xffffffffu, after, o);
        const uint32_t p = after;  // sorted buffer: entries [0, p) go before new
        const bool drop_first = cnt == static_cast<uint32_t>(LOW_Q);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < LQ_PER_LANE; ++i) {
            const uint32_t e = i * 32 + ln;
            if (e >= cnt) continue;
            if (drop_first) {
                if (e >= 1 && e < p) lo[e - 1] = v[i];  // drop lo[0], shift down
            } else {
                if (e >= p) lo[e + 1] = v[i];  // shift up
            }
        }
        if (ln == 0) {
            lo[drop_first ? p - 1 : p] = ne;
            const uint32_t nc = drop_first ? cnt : cnt + 1;
            sd.low_cnt[t] = nc;
            if (sd.n_used[t] == sd.cap2) S.reflist[atomicAdd(&S.nref, 1u)] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) P.rep[0] = S.applied;
    // ---- C: compaction + refill ----
    const uint32_t last_blk = N >> KEY_BLOCK_SHIFT;  // block of the newest key
    for (uint32_t r = 0; r < S.nref; ++r) refill_table(S.r, sd, S.reflist[r], last_blk);
}

cudaError_t launch_shard_victim(const InsertProblem* probs, uint32_t nprob,
                                unsigned long long* vk, cudaStream_t st) {
    shard_victim_kernel<<<nprob, 256, 0, st>>>(probs, vk);
    return cudaGetLastError();
}

cudaError_t launch_insert(const InsertProblem* probs, uint32_t nprob, cudaStream_t st,
                          const unsigned long long* gvk, bool pdl) {
    if (pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nprob);
        cfg.blockDim = dim3(INS_THREADS);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, insert_kernel, probs, gvk);
    }
    insert_kernel<<<nprob, INS_THREADS, 0, st>>>(probs, gvk);
    return cudaGetLastError();
}

}  // namespace csa
