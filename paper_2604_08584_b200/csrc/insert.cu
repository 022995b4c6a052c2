// insert.cu — KvStore::append (core.cpp:71-79) + streaming_insert
// (retrieval.cpp:272-301, TopList::try_insert index.cpp:22-44) on sm_100a.
//
// One CTA per session, one thread per (subspace b, centroid j) table.
// The new key's index N is larger than every stored key, so in the
// index-sorted layout an admitted entry is a plain append at n_used[t].
// Eviction removes the TopList back = the live entry that is first in
// eviction order (score asc, key desc); it is found in O(1) at the tail of
// the per-table low buffer (stored in DESCENDING eviction order, so the next
// victim is low[cnt-1]) and tombstoned in place. When a buffer runs dry the
// CTA compacts that table (dropping its <= LOW_Q tombstones, rebuilding the
// key-block offsets) and refills the buffer with the LOW_Q lowest live entries
// via a radix select over the 64-bit eviction key.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "tables.cuh"

namespace csa {

constexpr int INS_THREADS = 512;

struct InsSmem {
    float ks[DMAX];
    uint32_t zero_mask;
    uint32_t nref;
    uint32_t applied;
    uint32_t reflist[MAX_TABLES];  // tables needing compaction + refill
    RefillSmem r;
};

__global__ void __launch_bounds__(INS_THREADS)
insert_kernel(const InsertProblem* __restrict__ probs) {
    __shared__ InsSmem S;
    const InsertProblem& P = probs[blockIdx.x];
    const SessionDev& sd = *P.s;
    const uint32_t d = sd.d, m = sd.m, C = sd.C, T = m * C, N = P.N;
    // KvStore::append: row N lands at tail row N - P
    for (uint32_t x = threadIdx.x; x < d; x += blockDim.x) {
        sd.ktail[static_cast<size_t>(N - sd.P) * d + x] = P.key[x];
        sd.vtail[static_cast<size_t>(N - sd.P) * d + x] = P.value[x];
        S.ks[x] = P.key[x];
    }
    if (threadIdx.x == 0) {
        S.zero_mask = 0;
        S.nref = 0;
        S.applied = 0;
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
    uint8_t* mask = reinterpret_cast<uint8_t*>(P.rep + 1);
    const uint32_t new_blk = (N & (KEY_BLOCK - 1)) == 0;
    for (uint32_t t = threadIdx.x; t < T; t += blockDim.x) {
        const uint32_t b = t / C, j = t - b * C;
        const uint32_t off = sd.offs[b], w = sd.widths[b];
        double s = 0.0;
        if (!(S.zero_mask & (1u << b))) {
            const float* c = sd.cent + static_cast<size_t>(C) * off + static_cast<size_t>(j) * w;
            for (uint32_t x = 0; x < w; ++x) s = __fma_rn((double)__ldg(c + x), (double)S.ks[off + x], s);
        }
        const float sc = __double2float_rn(s);
        uint32_t nu = sd.n_used[t];
        if (new_blk) sd.blk_off[static_cast<size_t>(t) * sd.nb_stride + (N >> KEY_BLOCK_SHIFT)] = nu;
        uint32_t applied = 0;
        const uint32_t live = sd.live[t];
        uint32_t cnt = sd.low_cnt[t];
        LowEnt* lo = sd.low + static_cast<size_t>(t) * LOW_Q;
        uint2* e = sd.ent + static_cast<size_t>(t) * sd.cap2;
        if (sd.L != 0) {
            const bool full = live >= sd.L;
            bool ok = true;
            bool complete = (cnt == live);
            if (full) {
                const LowEnt victim = lo[cnt - 1];
                if (!(sc > victim.score)) {
                    ok = false;
                } else {
                    e[victim.pos].x = victim.key | TOMB;
                    cnt -= 1;
                }
            }
            if (ok) {
                applied = 1;
                e[nu] = make_uint2(N, __float_as_uint(sc));
                const uint32_t pos = nu;
                nu += 1;
                if (!full) sd.live[t] = live + 1;
                // keep low buffer = the cnt lowest live entries
                bool ins;
                if (cnt == 0)
                    ins = complete;  // empty: only a complete buffer may take it
                else if (complete && cnt < static_cast<uint32_t>(LOW_Q))
                    ins = true;
                else
                    ins = ev_before(sc, N, lo[0].score, lo[0].key);
                if (ins) {
                    // descending eviction order: skip entries evicted after new
                    uint32_t p = 0;
                    while (p < cnt && !ev_before(lo[p].score, lo[p].key, sc, N)) ++p;
                    const bool drop_first = cnt == static_cast<uint32_t>(LOW_Q);
                    if (drop_first) {
                        // drop lo[0] (the largest), insert at p-1
                        for (uint32_t x = 0; x + 1 < p; ++x) lo[x] = lo[x + 1];
                        LowEnt le{sc, N, pos, 0};
                        lo[p - 1] = le;
                    } else {
                        for (uint32_t x = cnt; x > p; --x) lo[x] = lo[x - 1];
                        LowEnt le{sc, N, pos, 0};
                        lo[p] = le;
                        cnt += 1;
                    }
                }
                sd.n_used[t] = nu;
                sd.low_cnt[t] = cnt;
                if (cnt == 0 || nu == sd.cap2) S.reflist[atomicAdd(&S.nref, 1u)] = t;
            }
        }
        mask[t] = static_cast<uint8_t>(applied);
        if (applied) atomicAdd(&S.applied, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) P.rep[0] = S.applied;
    const uint32_t last_blk = N >> KEY_BLOCK_SHIFT;  // block of the newest key
    for (uint32_t r = 0; r < S.nref; ++r) refill_table(S.r, sd, S.reflist[r], last_blk);
}

cudaError_t launch_insert(const InsertProblem* probs, uint32_t nprob, cudaStream_t st) {
    insert_kernel<<<nprob, INS_THREADS, 0, st>>>(probs);
    return cudaGetLastError();
}

}  // namespace csa
