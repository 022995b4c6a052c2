// select.cu — CSAttention decode, part 1: gather + accumulate + top-K on sm_100a.
//
// Persistent kernel, two 288-thread CTAs per SM; CTA b takes problems
// b, b + grid, ... (a problem = one (session, query head) decode search).
//
//   producer warp   streams the gathered lists (route.cu's plan) tile by tile:
//                   for each 4096-key tile and each list, the list's entries
//                   with keys in the tile ([blk_off(tile), blk_off(tile+1)),
//                   the tables are index-sorted) are copied by TMA bulk copies
//                   (cp.async.bulk, L2 evict_first, mbarrier complete_tx) into
//                   a 6-slot ring. It runs ahead across tile and problem
//                   boundaries, so the next problem's lists are in flight while
//                   the current one is being selected.
//   8 consumer      accumulate list by list in gathered-list order (the
//   warps           reference's per-key order [gather_lists :95-109,
//                   reduce_by_key :111-148]): warp w owns keys [512w, 512w+512)
//                   of every tile and takes, from each list's segment, exactly
//                   the entries in its range (bounds from blk_off, passed by the
//                   producer in the slot metadata), so no two warps touch a key
//                   and no CTA barrier separates lists:
//                   score(i) = sum_l w_b(l) * double(score_l(i)).
//                   At the end of a tile each warp turns its 512 keys into pool
//                   candidates [select_topk :150-228 pool rules]: a cheap
//                   compare against the current cut compacts the survivors in
//                   place, then only those are binned into a 2048-bin linear
//                   histogram fixed up front by route.cu's score bounds (a
//                   monotone map, so bins never split equal scores) and
//                   appended to the warp's candidate log. The cut is the highest
//                   bin whose suffix count already reaches `need`; it only
//                   rises, so every candidate that can still be selected is
//                   logged.
//   final phase     the exact bin of the need-th best candidate comes from the
//                   histogram; candidates above it are selected, the bin's
//                   members are ranked by (score desc, index asc) in shared
//                   memory (64-bit radix passes for large bins), then window
//                   passthrough and newest-first padding are applied on a key
//                   bitmap that is emitted in ascending order.
// The per-key scores never leave the SM except as logged candidates.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace csa {

constexpr int SEL_CW = 8;                    // consumer warps (2 CTAs per SM)
constexpr int SEL_CT = SEL_CW * 32;          // consumer threads
constexpr int SEL_THREADS = SEL_CT + 32;     // + producer warp
constexpr uint32_t TILE = 4096;              // keys per tile (fp64 accumulator: 32 KB)
constexpr uint32_t TILE_BLKS = TILE / KEY_BLOCK;
constexpr uint32_t WKEYS = TILE / SEL_CW;    // keys per warp in the tile-end filter
constexpr int NSLOT = 3;                     // ring slots
constexpr uint32_t SLOT_E = 2048;            // entries per slot (16 KB)
constexpr uint32_t MAXSUB = 4;               // list segments packed into one slot
constexpr int NB = 2048;                     // histogram bins
constexpr int NCB = NB / 32;                 // coarse bins (32 fine bins each)
constexpr int BKT = 512;                     // threshold-bin members ranked in smem
constexpr int RANK_DIRECT = 384;             // O(n^2) ranking up to this size
constexpr uint32_t F_TILE_END = 1, F_PROB_END = 2, F_CACHE = 4;
constexpr int MAXPART = 16;                  // key-range parts of a split problem
constexpr uint32_t MAXSEG = MAXPART * 8;     // log segments (parts x warps)
static_assert(SELECT_MAX_PART == MAXPART && SELECT_CONSUMER_WARPS == SEL_CW, "kernels.h mirrors");
constexpr uint32_t UNIT_META = 2048 + 64 + 8;  // per part unit: hist, coarse, per-warp log lengths
constexpr unsigned long long ABSENT = 0x7ff4deadbeef0000ull;  // NaN box: key not gathered
static_assert(TILE * 64 == SELECT_MAX_CONTEXT, "bitmap capacity = accumulator bits");
static_assert(SELECT_MAX_CONTEXT / TILE <= 128 && MAXL < 127, "chunk info fields");
static_assert(UNIT_META == NB + NCB + SEL_CW && SEL_CW == 8, "unit metadata layout");

// One ring chunk = one slot: up to MAXSUB list segments of one tile, packed
// at even (16-byte aligned) slot positions, in gathered-list order.
// info = nsub | flags << 3 | tile << 8; sub s is list `lists[s]` and consumer
// warp w's entries of it are the slot positions wr[s][w] = [x, y) (its own key
// range of the tile intersected with the segment; y <= x when none).
struct SlotMeta {
    uint32_t info;
    uint8_t lists[MAXSUB];
    uint2 wr[MAXSUB][SEL_CW];
};
static_assert(WKEYS % KEY_BLOCK == 0, "warp key ranges are whole key blocks");
constexpr uint32_t WBLKS = WKEYS / KEY_BLOCK;  // key blocks per warp range

struct SelHdr {
    unsigned long long full[NSLOT], empty[NSLOT];
    SlotMeta meta[NSLOT];
    uint32_t plist[MAXL];  // producer: table ids of its current problem
    uint32_t wbs[2][MAXL][SEL_CW + 1];  // producer: per-warp bounds of tiles t, t+1 per list
    double cw[MAXL];       // consumers: weight of each gathered list
    uint32_t cut, nbkt;
    // candidate-log segments of the problem being finalised
    uint32_t seg_len[MAXSEG], seg_off[MAXSEG], seg_pre[MAXSEG + 1];
    uint32_t wsum[SEL_CW];
    // final-phase broadcasts
    uint32_t f_bin, f_above, f_count, f_take_all, f_fail, f_last;
    unsigned long long tk;
    uint32_t tx;
};

__device__ __forceinline__ unsigned long long ordkey(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 == +0.0 (retrieval.cpp:168-171)
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ bool is_absent(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == ABSENT;
}
__device__ __forceinline__ double absent_d() {
    return __longlong_as_double(static_cast<long long>(ABSENT));
}
// The tile accumulator marks "not gathered" with -0.0: a gathered key's sum
// starts as 0.0 + w*s (reduce_by_key). Table scores CAN be -0.0f (float() of a
// negative dot below 2^-150, index.cpp:81 / retrieval.cpp:293-294), so every
// term is canonicalised to +0.0 when zero (canon0 below): then no term and no
// sum is -0.0, and -0.0 + x == 0.0 + x for every canonical term x.
constexpr unsigned long long NEG0 = 0x8000000000000000ull;
__device__ __forceinline__ double neg0_d() { return __longlong_as_double(static_cast<long long>(NEG0)); }
__device__ __forceinline__ uint32_t canon0(uint32_t f32_bits) {  // -0.0f -> +0.0f
    return f32_bits == 0x80000000u ? 0u : f32_bits;
}
__device__ __forceinline__ bool is_neg0(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == NEG0;
}
// monotone non-decreasing score -> bin map (IEEE sub/mul preserve <=)
__device__ __forceinline__ uint32_t bin_of(double s, double lo, double scale) {
    const double f = __dmul_rn(__dsub_rn(s, lo), scale);
    return f >= static_cast<double>(NB - 1) ? static_cast<uint32_t>(NB - 1)
                                            : (f > 0.0 ? static_cast<uint32_t>(f) : 0u);
}

__device__ __forceinline__ void cbar() {  // consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(SEL_CT) : "memory");
}

// exclusive scan over the consumer threads in thread order; total = sum
__device__ uint32_t cscan(SelHdr& S, uint32_t v, uint32_t& total) {
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (ln >= o) inc += x;
    }
    if (ln == 31) S.wsum[w] = inc;
    cbar();
    uint32_t pre = 0;
    total = 0;
#pragma unroll
    for (int i = 0; i < SEL_CW; ++i) {
        const uint32_t x = S.wsum[i];
        pre += i < w ? x : 0u;
        total += x;
    }
    cbar();
    return pre + inc - v;
}

// Top-down crossing over a warp-held group of 32 counts: lane l holds count of
// bin (base + l); `above` = count above the group. Returns the highest lane
// whose suffix (bins >= it, plus above) reaches `need`, or -1; sets the count
// strictly above that lane.
__device__ __forceinline__ int warp_cross(uint32_t v, uint32_t above, uint32_t need,
                                          uint32_t& above_out) {
    const int ln = threadIdx.x & 31;
    uint32_t suf = v;  // inclusive suffix over lanes >= ln
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o);
        if (ln + o < 32) suf += x;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, above + suf >= need);
    if (!hit) return -1;
    const int l = 31 - __clz(hit);
    above_out = above + __shfl_sync(0xffffffffu, suf - v, l);
    return l;
}

// Highest fine bin whose suffix count reaches `need`, from the two-level
// histogram, by one warp (counts at and above the answer must be exact).
// Returns -1 if the total is below need; `above` = count strictly above.
__device__ int warp_find_bin(const uint32_t* hist, const uint32_t* coarse, uint32_t need,
                             uint32_t& above) {
    const int ln = threadIdx.x & 31;
    uint32_t run = 0;
    for (int g = NCB / 32 - 1; g >= 0; --g) {
        const uint32_t v = coarse[g * 32 + ln];
        uint32_t ab;
        const int l = warp_cross(v, run, need, ab);
        if (l >= 0) {
            const int cb = g * 32 + l;
            uint32_t ab2;
            const int f = warp_cross(hist[cb * 32 + ln], ab, need, ab2);
            above = ab2;
            // f < 0 only while other warps are mid-update (coarse counted
            // before fine): report no crossing, the caller keeps its cut
            return f < 0 ? -1 : cb * 32 + f;
        }
        uint32_t s = v;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        run += s;
    }
    above = run;
    return -1;
}

// Exact rem-th best member (key desc, index asc) by radix passes; members are
// get(e, key, idx) == true for e < n. Leaves S.tk / S.tx such that a member is
// selected iff key > tk || (key == tk && idx < tx). Uses hist as scratch.
template <class Get>
__device__ void radix_kth(SelHdr& S, uint32_t* hist, uint32_t n, uint32_t rem, Get get) {
    const uint32_t tid = threadIdx.x;
    unsigned long long prefix = 0;
    int pshift = 64;
    bool ties = false;
    for (;;) {  // stage 1: the score key
        const int shift = pshift > 11 ? pshift - 11 : 0;
        const uint32_t nbins = 1u << (pshift - shift);
        for (uint32_t i = tid; i < nbins; i += SEL_CT) hist[i] = 0;
        cbar();
        for (uint32_t e = tid; e < n; e += SEL_CT) {
            unsigned long long k;
            uint32_t ix;
            if (!get(e, k, ix)) continue;
            if (pshift < 64 && (k >> pshift) != prefix) continue;
            atomicAdd(&hist[(k >> shift) & (nbins - 1)], 1u);
        }
        cbar();
        if (tid < 32) {
            uint32_t run = 0;
            for (int g = static_cast<int>(nbins / 32) - 1; g >= 0; --g) {
                const uint32_t v = hist[g * 32 + tid];
                uint32_t ab;
                const int l = warp_cross(v, run, rem, ab);
                if (l >= 0) {
                    if (tid == 0) {
                        S.f_bin = g * 32 + l;
                        S.f_above = ab;
                        S.f_count = hist[g * 32 + l];
                    }
                    break;
                }
                uint32_t s = v;
                for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                run += s;
            }
        }
        cbar();
        rem -= S.f_above;
        prefix = (pshift == 64 ? 0ull : (prefix << (pshift - shift))) | S.f_bin;
        pshift = shift;
        if (S.f_count == rem) {  // the whole digit bucket is taken
            const unsigned long long T = prefix << pshift;
            if (tid == 0) {
                S.tk = T ? T - 1 : 0ull;
                S.tx = 0;
            }
            cbar();
            return;
        }
        if (pshift == 0) {
            ties = true;
            break;
        }
    }
    // stage 2: rem lowest indices among the members tied at key == prefix
    const unsigned long long tk = prefix;
    uint32_t ipre = 0;
    int ishift = 32;
    if (ties) {
        for (;;) {
            const int shift = ishift > 11 ? ishift - 11 : 0;
            const uint32_t nbins = 1u << (ishift - shift);
            for (uint32_t i = tid; i < nbins; i += SEL_CT) hist[i] = 0;
            cbar();
            for (uint32_t e = tid; e < n; e += SEL_CT) {
                unsigned long long k;
                uint32_t ix;
                if (!get(e, k, ix) || k != tk) continue;
                const uint32_t r = ~ix;  // largest r = smallest index
                if (ishift < 32 && (r >> ishift) != ipre) continue;
                atomicAdd(&hist[(r >> shift) & (nbins - 1)], 1u);
            }
            cbar();
            if (tid < 32) {
                uint32_t run = 0;
                for (int g = static_cast<int>(nbins / 32) - 1; g >= 0; --g) {
                    const uint32_t v = hist[g * 32 + tid];
                    uint32_t ab;
                    const int l = warp_cross(v, run, rem, ab);
                    if (l >= 0) {
                        if (tid == 0) {
                            S.f_bin = g * 32 + l;
                            S.f_above = ab;
                            S.f_count = hist[g * 32 + l];
                        }
                        break;
                    }
                    uint32_t s = v;
                    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    run += s;
                }
            }
            cbar();
            rem -= S.f_above;
            ipre = (ishift == 32 ? 0u : (ipre << (ishift - shift))) | S.f_bin;
            ishift = shift;
            if (S.f_count == rem || ishift == 0) break;  // indices are unique
        }
    }
    // selected ties: ~idx >= (ipre << ishift)  <=>  idx <= ~(ipre << ishift)
    if (tid == 0) {
        S.tk = tk;
        S.tx = ~(ipre << ishift) + 1u;  // idx < tx
    }
    cbar();
}

__device__ __forceinline__ void set_bit(uint32_t* bm, uint32_t i) {
    atomicOr(bm + (i >> 5), 1u << (i & 31));
}


// Per-problem state of the consumer warps (registers).
struct ProbState {
    uint32_t N, K, need, f_lo, wlo;
    uint32_t n_cache;
    uint32_t cut_init;  // speculative cut from the previous step's threshold (0 = none)
    double* hint;       // [threshold score, valid] of this (session, head)
    bool pt, store_cache;
    double lo, scale;
    double* cache;
    uint32_t* sel;
    uint32_t* rep;
    unsigned long long* prof;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// consumer warps: load problem p's descriptor, list weights, score bounds
// Speculation: the previous search's threshold score t of this (session, head)
// seeds the cut at lo + spec_keep * (t - lo) (spec_keep = 0.9 by default,
// 0 disables). The final phase verifies that the threshold bin is at or above
// it; otherwise the problem is redone without speculation by the retry pass,
// so the result never depends on the guess.

__device__ void setup_problem(SelHdr& S, const DecodeProblem* probs, const RoutePlan* plans,
                              uint32_t p, ProbState& st, bool speculate, double spec_keep) {
    const uint32_t tid = threadIdx.x;
    const DecodeProblem* Pp = probs + p;
    const SessionDev* sdp = Pp->s;
    st.N = Pp->N;
    st.K = Pp->K;
    const uint32_t mode = Pp->mode;
    st.n_cache = Pp->n_cache;
    st.cache = Pp->cache;
    double* const cbounds = Pp->cbounds;
    st.sel = Pp->sel;
    st.rep = Pp->rep;
    st.prof = Pp->prof;
    const uint32_t window = sdp->window;
    st.pt = sdp->passthrough != 0;
    const bool search = mode & MODE_SEARCH;
    st.store_cache = (mode & MODE_STORE_CACHE) && st.cache;
    if (search) {
        const uint32_t nl = __ldcg(&plans[p].nl);
        for (uint32_t l = tid; l < nl; l += SEL_CT) S.cw[l] = sdp->weights[__ldcg(plans[p].lsub + l)];
    }
    double lo, hi;
    if (search) {
        lo = __ldcg(&plans[p].lo);
        hi = __ldcg(&plans[p].hi);
        if (st.store_cache && tid == 0) {
            cbounds[0] = lo;
            cbounds[1] = hi;
        }
    } else {
        lo = __ldcg(cbounds);
        hi = __ldcg(cbounds + 1);
    }
    st.lo = lo;
    st.scale = hi > lo ? static_cast<double>(NB) / (hi - lo) : 0.0;
    st.hint = cbounds + 2;
    st.cut_init = 0;
    if (speculate && spec_keep > 0.0 && search && !st.store_cache && __ldcg(cbounds + 3) != 0.0 &&
        st.scale > 0.0) {
        const double t = __ldcg(cbounds + 2);
        const double g = lo + spec_keep * (t - lo);
        st.cut_init = bin_of(g, lo, st.scale);
    }
    const uint32_t N = st.N, K = st.K;
    const uint32_t r_eff = window < N ? window : N;
    st.wlo = N - r_eff;
    if (st.pt) {
        st.need = K > r_eff ? K - r_eff : 0;
        st.f_lo = K > r_eff ? st.wlo : N - K;
    } else {
        st.need = K;
        st.f_lo = N;
    }
    if (tid == 0) S.cut = st.cut_init;
    cbar();  // weights + cut visible
    if (st.prof && tid == 0) st.prof[0] = gtimer();
}


// The final selection of one problem from its histogram (hist/coarse, complete
// at and above every cut used) and its candidate log, given as nseg segments
// (S.seg_off[k], S.seg_len[k]) of log_idx/log_sc. Consumer threads only (named
// barrier 1). Leaves the bitmap region dirty; the caller resets its scratch.
__device__ unsigned long long g_fin_dbg[8];
constexpr uint32_t SEL_TS_MAX = 1024;            // CSATTN_PHASE_PROF: per-CTA start / end
__device__ unsigned long long g_cta_ts[2 * SEL_TS_MAX];
__device__ unsigned long long g_cta_ev[8 * SEL_TS_MAX];  // (globaltimer << 2) | item type  // CSATTN_PHASE_PROF: final-phase stage ns, summed
__device__ void final_select(SelHdr& S, const ProbState& st, uint32_t p, uint32_t* hist,
                             uint32_t* coarse, uint32_t* bm, unsigned long long* bkey,
                             uint32_t* bidx, const uint32_t* log_idx, const double* log_sc,
                             uint32_t nseg, uint32_t* retry_out, uint32_t* retry_out_count) {
    const uint32_t tid = threadIdx.x;
    const uint32_t N = st.N, K = st.K, need = st.need, f_lo = st.f_lo;
    const double lo = st.lo, scale = st.scale;
    unsigned long long* const prof = st.prof;
    uint32_t* const sel = st.sel;
    uint32_t* const rep = st.rep;
    if (tid == 0) {  // exclusive prefix of the segment lengths
        uint32_t run = 0;
        for (uint32_t k = 0; k <= nseg; ++k) {
            const uint32_t x = k < nseg ? S.seg_len[k] : 0u;
            S.seg_pre[k] = run;
            run += x;
        }
    }
    if (prof && tid == 0) prof[1] = gtimer();
    unsigned long long tdbg = (prof && tid == 0) ? gtimer() : 0ull;
    const uint32_t nw = div_up(N, 32);
    if (tid < 32) {
        uint32_t ab = 0;
        int b = -1;
        if (need) b = warp_find_bin(hist, coarse, need, ab);
        if (tid == 0) {
            // the speculative cut must not exceed the threshold bin: every
            // key at or above the threshold bin was then counted and logged
            const bool fail = need && st.cut_init &&
                              (b < 0 || static_cast<uint32_t>(b) < st.cut_init);
            S.f_fail = fail ? 1u : 0u;
            if (fail) retry_out[atomicAdd(retry_out_count, 1u)] = p;
            // b < 0: fewer than `need` pool keys (then the cut never rose
            // and the log holds the whole pool): take them all
            S.f_take_all = (need && b < 0) ? 1u : 0u;
            S.f_bin = b < 0 ? 0u : static_cast<uint32_t>(b);
            S.f_above = ab;
            S.f_count = b < 0 ? 0u : hist[b];
        }
    }
    for (uint32_t x = tid; x < nw; x += SEL_CT) bm[x] = 0;
    cbar();
    if (prof && tid == 0) { const unsigned long long t_ = gtimer(); atomicAdd(&g_fin_dbg[0], t_ - tdbg); tdbg = t_; }
    const bool failed = S.f_fail != 0;
    const uint32_t take_all = S.f_take_all, dsel = S.f_bin;
    const uint32_t rem = need - (take_all ? 0u : min(need, S.f_above));
    const uint32_t nlog = S.seg_pre[nseg];
    // flat log index -> log position through the segment table (search from
    // `w`: the indices one thread visits only grow)
    auto lpos = [&](uint32_t e, uint32_t& w) {
        while (S.seg_pre[w + 1] <= e) ++w;
        return S.seg_off[w] + (e - S.seg_pre[w]);
    };
    if (!failed) {  // (a failed speculation is redone by the retry pass)
        if (need) {
            constexpr int LOGU = 8;  // entries per thread in flight (the log lives in L2)
            uint32_t w = 0;
            for (uint32_t e0 = tid; e0 < nlog; e0 += SEL_CT * LOGU) {
                uint32_t ii[LOGU];
                double sv[LOGU];
#pragma unroll
                for (int u = 0; u < LOGU; ++u) {
                    const uint32_t e = e0 + u * SEL_CT;
                    const uint32_t x = e < nlog ? lpos(e, w) : 0u;
                    ii[u] = e < nlog ? __ldcg(log_idx + x) : 0u;
                    sv[u] = e < nlog ? __ldcg(log_sc + x) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < LOGU; ++u) {
                    if (e0 + u * SEL_CT >= nlog) break;
                    const uint32_t b = bin_of(sv[u], lo, scale);
                    if (take_all || b > dsel) {
                        set_bit(bm, ii[u]);
                    } else if (b == dsel) {
                        const uint32_t k = atomicAdd(&S.nbkt, 1u);
                        if (k < static_cast<uint32_t>(BKT)) {
                            bkey[k] = ordkey(sv[u]);
                            bidx[k] = ii[u];
                        }
                    }
                }
            }
        }
        cbar();
        if (prof && tid == 0) { const unsigned long long t_ = gtimer(); atomicAdd(&g_fin_dbg[1], t_ - tdbg); tdbg = t_; }
        const uint32_t nb = S.nbkt;
        if (need && !take_all && rem) {
            if (nb <= static_cast<uint32_t>(RANK_DIRECT)) {
                // direct ranking: member e is selected iff fewer than rem beat it
                for (uint32_t e = tid; e < nb; e += SEL_CT) {
                    const unsigned long long ke = bkey[e];
                    const uint32_t ie = bidx[e];
                    uint32_t r = 0;
                    for (uint32_t f = 0; f < nb; ++f) {
                        const unsigned long long kf = bkey[f];
                        r += (kf > ke) || (kf == ke && bidx[f] < ie);
                    }
                    if (r < rem) set_bit(bm, ie);
                }
            } else if (nb <= static_cast<uint32_t>(BKT)) {
                radix_kth(S, hist, nb, rem, [&](uint32_t e, unsigned long long& k, uint32_t& ix) {
                    k = bkey[e];
                    ix = bidx[e];
                    return true;
                });
                const unsigned long long tk = S.tk;
                const uint32_t tx = S.tx;
                for (uint32_t e = tid; e < nb; e += SEL_CT) {
                    const unsigned long long k = bkey[e];
                    if (k > tk || (k == tk && bidx[e] < tx)) set_bit(bm, bidx[e]);
                }
            } else {  // huge threshold bin: rank straight from the log
                auto member = [&](uint32_t e, unsigned long long& k, uint32_t& ix) {
                    uint32_t w = 0;
                    const uint32_t x = lpos(e, w);
                    const double s = __ldcg(log_sc + x);
                    if (bin_of(s, lo, scale) != dsel) return false;
                    k = ordkey(s);
                    ix = __ldcg(log_idx + x);
                    return true;
                };
                radix_kth(S, hist, nlog, rem, member);
                const unsigned long long tk = S.tk;
                const uint32_t tx = S.tx;
                for (uint32_t e = tid; e < nlog; e += SEL_CT) {
                    unsigned long long k;
                    uint32_t ix;
                    if (member(e, k, ix) && (k > tk || (k == tk && ix < tx))) set_bit(bm, ix);
                }
            }
        }
        // window passthrough (or the newest K when K <= R)
        for (uint32_t i = f_lo + tid; i < N; i += SEL_CT) set_bit(bm, i);
        cbar();
        if (prof && tid == 0) { const unsigned long long t_ = gtimer(); atomicAdd(&g_fin_dbg[2], t_ - tdbg); tdbg = t_; }
        // ---- count, newest-first padding, ascending emit ----
        const uint32_t wpt = div_up(nw, SEL_CT);
        const uint32_t w0 = min(nw, tid * wpt), w1 = min(nw, w0 + wpt);
        auto valid = [&](uint32_t x) {
            return x + 1 < nw || (N & 31) == 0 ? 0xffffffffu : ((1u << (N & 31)) - 1u);
        };
        uint32_t cnt = 0, zeros = 0;
        for (uint32_t x = w0; x < w1; ++x) {
            const uint32_t b = bm[x];
            cnt += __popc(b);
            zeros += __popc(~b & valid(x));
        }
        uint32_t total;
        cscan(S, cnt, total);
        if (prof && tid == 0) { const unsigned long long t_ = gtimer(); atomicAdd(&g_fin_dbg[3], t_ - tdbg); tdbg = t_; }
        if (total < K) {  // pad with the newest untaken keys (retrieval.cpp:218-225)
            const uint32_t pad = K - total;
            uint32_t zt;
            const uint32_t zbelow = cscan(S, zeros, zt);
            const uint32_t zabove = zt - zbelow - zeros;  // zeros in higher threads
            uint32_t take = pad > zabove ? min(pad - zabove, zeros) : 0u;
            for (uint32_t x = w1; x > w0 && take;) {
                --x;
                uint32_t z = ~bm[x] & valid(x);
                while (z && take) {
                    const int hb = 31 - __clz(z);
                    bm[x] |= 1u << hb;
                    z &= ~(1u << hb);
                    --take;
                    ++cnt;
                }
            }
        }
        const uint32_t at = cscan(S, cnt, total);
        if (prof && tid == 0) { const unsigned long long t_ = gtimer(); atomicAdd(&g_fin_dbg[4], t_ - tdbg); tdbg = t_; }
        {
            uint32_t pos = at;
            for (uint32_t x = w0; x < w1; ++x) {
                uint32_t b = bm[x];
                while (b) {
                    const int lb = __ffs(b) - 1;
                    sel[pos++] = x * 32 + lb;
                    b &= b - 1;
                }
            }
        }
        if (tid == 0) {
            reinterpret_cast<DecodeReport*>(rep)->k = K;
            if (prof) {
                prof[2] = gtimer();
                atomicAdd(&g_fin_dbg[5], gtimer() - tdbg); atomicAdd(&g_fin_dbg[6], 1ull);
                prof[3] = nlog;
                prof[4] = nb;
                prof[5] = static_cast<unsigned long long>(__double_as_longlong(lo));
                prof[6] = static_cast<unsigned long long>(
                    __double_as_longlong(scale > 0.0 ? lo + NB / scale : lo));
                prof[7] = S.f_take_all | (dsel << 1);
            }
        }
        if (tid == 0) {  // next step's speculative cut: this threshold bin's lower edge
            st.hint[0] = scale > 0.0 ? lo + static_cast<double>(dsel) / scale : lo;
            st.hint[1] = (need && !take_all) ? 1.0 : 0.0;
        }
    }
}

__global__ void __launch_bounds__(SEL_THREADS, 2)
select_kernel(const DecodeProblem* __restrict__ probs, const RoutePlan* __restrict__ plans,
              uint32_t nprob, uint32_t* __restrict__ log_idx_all, double* __restrict__ log_sc_all,
              uint32_t log_cap, const uint32_t* __restrict__ retry_in,
              const uint32_t* __restrict__ retry_in_count, uint32_t* __restrict__ retry_out,
              uint32_t* __restrict__ retry_out_count, double spec_keep, uint32_t split,
              uint32_t* __restrict__ unit_meta, const SelMixed mx) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // The work sequence of this CTA: units b, b + grid, ... A unit is problem
    // u / split, tiles [part u % split] of its key range; split == 1 (one unit
    // per problem, finalised here) or split > 1 (part units dump histogram and
    // log lengths to unit_meta; select_merge_kernel finalises). The retry pass
    // walks the retry list (split == 1 only).
    // Mixed mode (mx.items): this CTA walks its own item list, whole problems
    // (finalised here) then tail pieces (part units: histogram + log to
    // mx.umeta / the part logs; the CTA finishing a problem's LAST piece
    // merges them and finalises it), so 512 problems over 296 slots cost
    // 1.73 problems per CTA instead of two rounds.
    const bool mixed = mx.items != nullptr;
    // the retry pass (a programmatic dependent of the first pass) reads the
    // retry list the first pass wrote
    if (retry_in) asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t it0 = mixed ? __ldg(mx.cta_items + blockIdx.x) : 0u;
    const uint32_t it1 = mixed ? __ldg(mx.cta_items + blockIdx.x + 1) : 0u;
    const uint32_t nwork = mixed ? it1 : (retry_in ? __ldcg(retry_in_count) : nprob * split);
    const uint32_t kfirst = mixed ? it0 : blockIdx.x, kstep = mixed ? 1u : gridDim.x;
    if (kfirst >= nwork) return;
    auto prob_of = [&](uint32_t k) {
        return mixed ? __ldg(&mx.items[k].x) : (retry_in ? __ldcg(retry_in + k) : k / split);
    };
    // unit k's tiles: part k % split of the problem's tile range (a shard's
    // range [tile_lo, tile_hi), else all tiles of its N keys); mixed: the item's
    auto tiles_of = [&](uint32_t k, const DecodeProblem& P, uint32_t& tl, uint32_t& th) {
        if (mixed) {
            tl = __ldg(&mx.items[k].y);
            th = __ldg(&mx.items[k].z);
            return;
        }
        const uint32_t t0 = P.tile_hi ? P.tile_lo : 0u;
        const uint32_t t1 = P.tile_hi ? P.tile_hi : div_up(P.N, TILE);
        const uint32_t nt = t1 - t0, j = retry_in ? 0u : k % split;
        tl = t0 + (nt * j) / split;
        th = t0 + (nt * (j + 1)) / split;
    };
    auto slot_of = [&](uint32_t k) { return mixed ? __ldg(&mx.items[k].w) : NO_SLOT; };
    const bool speculate = (retry_out != nullptr || unit_meta != nullptr) && !retry_in;
    SelHdr& S = *reinterpret_cast<SelHdr*>(smem_raw);
    unsigned char* p0 = smem_raw + ((sizeof(SelHdr) + 127) & ~size_t(127));
    double* acc = reinterpret_cast<double*>(p0);                    // TILE fp64
    uint32_t* bm = reinterpret_cast<uint32_t*>(p0);                 // bitmap (aliases acc)
    uint32_t* hist = reinterpret_cast<uint32_t*>(p0 + TILE * 8);    // NB
    uint32_t* coarse = hist + NB;                                   // NCB
    unsigned long long* bkey = reinterpret_cast<unsigned long long*>(coarse + NCB);  // BKT
    uint32_t* bidx = reinterpret_cast<uint32_t*>(bkey + BKT);       // BKT
    uint16_t* cidx = reinterpret_cast<uint16_t*>(bidx + BKT);       // SEL_CW * WKEYS
    uint2* ring = reinterpret_cast<uint2*>(cidx + SEL_CW * WKEYS);  // NSLOT * SLOT_E
    const uint32_t tid = threadIdx.x;
    const int wid = tid >> 5, ln = tid & 31;
    uint32_t* log_idx = log_idx_all + static_cast<size_t>(blockIdx.x) * log_cap;
    double* log_sc = log_sc_all + static_cast<size_t>(blockIdx.x) * log_cap;

    if (tid == 0) {
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], SEL_CW);
        }
        fence_mbar_init();
        S.cut = 0;
        S.nbkt = 0;
    }
    for (uint32_t i = tid; i < TILE; i += SEL_THREADS) acc[i] = neg0_d();
    for (uint32_t i = tid; i < NB + NCB; i += SEL_THREADS) hist[i] = 0;
    __syncthreads();
    // programmatic launch: the route plans are visible after this (a no-op
    // for a normal launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const bool cta_prof = probs[0].prof != nullptr && blockIdx.x < SEL_TS_MAX;
    if (cta_prof && tid == 0) g_cta_ts[2 * blockIdx.x] = gtimer();
    uint32_t nev = 0;  // CSATTN_PHASE_PROF: item-end events of this CTA (thread 0)
    auto stamp = [&](uint32_t type) {
        if (cta_prof && tid == 0 && nev < 8) g_cta_ev[blockIdx.x * 8 + nev++] = (gtimer() << 2) | type;
    };

    // ======================= producer warp =======================
    if (wid == SEL_CW) {
        const unsigned long long pol = l2_evict_first_policy();
        uint32_t c = 0;         // slots opened so far
        uint32_t nsub = 0, fill = 0, open_slot = 0;  // the slot being packed
        auto open = [&]() {      // wait for the next slot to be free
            open_slot = c % NSLOT;
            if (c >= static_cast<uint32_t>(NSLOT))
                mbar_wait_sleep(&S.empty[open_slot], ((c / NSLOT) - 1) & 1u);
            ++c;
            nsub = 0;
            fill = 0;
        };
        // stage positions [lo, hi) of list l (table row tbl) into the open slot
        auto add = [&](uint32_t l, const uint2* tbl, uint32_t lo, uint32_t hi, const uint32_t* wb) {
            const uint32_t ab = lo & ~1u, ae = (hi + 1) & ~1u;  // <= cap2 (even)
            const uint32_t at = fill;                          // slot position of ab
            if (ln < SEL_CW) {  // consumer warp ln's slot-relative entry range
                const uint32_t x = max(lo, wb[ln]), y = min(hi, wb[ln + 1]);
                S.meta[open_slot].wr[nsub][ln] = y > x ? make_uint2(x - ab + at, y - ab + at) : make_uint2(0u, 0u);
            }
            if (ln == 0) {
                S.meta[open_slot].lists[nsub] = static_cast<uint8_t>(l);
                const uint32_t bytes = (ae - ab) * 8u;
                mbar_expect_tx_only(&S.full[open_slot], bytes);
                bulk_g2s_hint(ring + static_cast<size_t>(open_slot) * SLOT_E + at, tbl + ab, bytes,
                              &S.full[open_slot], pol);
            }
            ++nsub;
            fill += ae - ab;
        };
        auto close = [&](uint32_t flags, uint32_t tile) {  // publish the open slot
            __syncwarp();  // lane 0's arrive below releases the other lanes' meta writes
            if (ln == 0) {
                S.meta[open_slot].info = nsub | (flags << 3) | (tile << 8);
                mbar_arrive(&S.full[open_slot]);
            }
            __syncwarp();
        };
        for (uint32_t k = kfirst; k < nwork; k += kstep) {
            const uint32_t p = prob_of(k);
            const DecodeProblem& P = probs[p];
            const SessionDev& sd = *P.s;
            const uint32_t N = P.N;
            uint32_t tl, ntile;
            tiles_of(k, P, tl, ntile);  // this unit's tiles [tl, ntile)
            uint32_t nl = 0;
            if (P.mode & MODE_SEARCH) {
                nl = __ldcg(&plans[p].nl);
                for (uint32_t l = ln; l < nl; l += 32) S.plist[l] = __ldcg(plans[p].lists + l);
                __syncwarp();
            }
            const uint32_t last_blk = (N - 1) >> KEY_BLOCK_SHIFT;
            const uint32_t* const blk_off = sd.blk_off;
            const uint32_t* const n_used = sd.n_used;
            const uint2* const ent = sd.ent;
            const uint32_t nb_stride = sd.nb_stride, cap2 = sd.cap2;
            // first table position of tile `tile` in list l (lanes l and l+32);
            // tile t+2's bounds are loaded while tile t is published
            auto bound = [&](uint32_t tile, uint32_t l) -> uint32_t {
                if (l >= nl) return 0u;
                const uint32_t t = S.plist[l];
                const uint32_t kb = tile * TILE_BLKS;
                return kb <= last_blk ? __ldcg(blk_off + static_cast<size_t>(t) * nb_stride + kb)
                                      : __ldcg(n_used + t);
            };
            // per-warp key-range bounds of every list in tile `tile` (the
            // consumer warps own fixed 512-key ranges: no per-list barrier):
            // nl x (SEL_CW + 1) table positions, three per lane. Loaded one
            // tile ahead into registers (issued before the current tile's
            // chunks are published, stored after), so the blk_off misses
            // overlap the ring waits instead of stalling the stream.
            const uint32_t nwb = nl * (SEL_CW + 1);
            auto wb_load = [&](uint32_t tile, uint32_t (&v)[3]) {
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const uint32_t idx = u * 32 + ln;
                    v[u] = 0;
                    if (idx < nwb && tile < ntile) {
                        const uint32_t l = idx / (SEL_CW + 1), j = idx - l * (SEL_CW + 1);
                        const uint32_t t = S.plist[l];
                        const uint32_t kb = tile * TILE_BLKS + j * WBLKS;
                        v[u] = kb <= last_blk ? __ldcg(blk_off + static_cast<size_t>(t) * nb_stride + kb)
                                              : __ldcg(n_used + t);
                    }
                }
            };
            auto wb_store = [&](uint32_t tile, const uint32_t (&v)[3]) {
                uint32_t* const dst = &S.wbs[tile & 1][0][0];
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const uint32_t idx = u * 32 + ln;
                    if (idx < nwb) dst[idx] = v[u];
                }
                // more than 10 lists (tau > 1 backoff): the rest synchronously
                for (uint32_t idx = 96 + ln; idx < nwb; idx += 32) {
                    const uint32_t l = idx / (SEL_CW + 1), j = idx - l * (SEL_CW + 1);
                    const uint32_t t = S.plist[l];
                    const uint32_t kb = tile * TILE_BLKS + j * WBLKS;
                    dst[idx] = kb <= last_blk ? __ldcg(blk_off + static_cast<size_t>(t) * nb_stride + kb)
                                              : __ldcg(n_used + t);
                }
                __syncwarp();
            };
            uint32_t wv[3];
            if (nl) {
                wb_load(tl, wv);
                wb_store(tl, wv);
            }
            uint32_t a0 = bound(tl, ln), a1 = bound(tl, ln + 32);
            uint32_t b0 = bound(tl + 1, ln), b1 = bound(tl + 1, ln + 32);
            for (uint32_t tile = tl; tile < ntile; ++tile) {
                const uint32_t tflag = F_TILE_END | (tile + 1 == ntile ? F_PROB_END : 0u);
                if (nl == 0) {  // cached scores: one data-less chunk per tile
                    open();
                    close(tflag | F_CACHE, tile);
                    continue;
                }
                const uint32_t c0 = bound(tile + 2, ln), c1 = bound(tile + 2, ln + 32);
                wb_load(tile + 1, wv);  // stored after this tile's chunks are out
                open();
                for (uint32_t l = 0; l < nl; ++l) {
                    const uint32_t e0 = __shfl_sync(0xffffffffu, l < 32 ? a0 : a1, l & 31);
                    const uint32_t e1 = __shfl_sync(0xffffffffu, l < 32 ? b0 : b1, l & 31);
                    if (e0 == e1) continue;  // nothing of this list in this tile
                    const uint2* tbl = ent + static_cast<size_t>(S.plist[l]) * cap2;
                    const uint32_t* wb = &S.wbs[tile & 1][l][0];
                    uint32_t pos = e0;
                    while (pos < e1) {
                        const uint32_t room = SLOT_E - fill;  // even
                        const uint32_t need = ((e1 + 1) & ~1u) - (pos & ~1u);
                        if (nsub == MAXSUB || room < 2 || (need > room && nsub > 0)) {
                            close(0u, tile);  // full: publish, continue in a fresh slot
                            open();
                            continue;
                        }
                        // the segment, or as much of it as fits an empty slot
                        const uint32_t pe = need <= room ? e1 : (pos & ~1u) + room;
                        add(l, tbl, pos, pe, wb);
                        pos = pe;
                    }
                }
                close(tflag, tile);
                if (tile + 1 < ntile) wb_store(tile + 1, wv);
                a0 = b0;
                a1 = b1;
                b0 = c0;
                b1 = c1;
            }
        }
        return;
    }

    // ======================= consumer warps =======================
    uint32_t kk = kfirst;
    uint32_t p = prob_of(kk);
    ProbState st;
    setup_problem(S, probs, plans, p, st, speculate, spec_keep);
    // warp w logs into its own region (it owns 1/8 of every tile's keys): the
    // CTA's log (split == 1, mixed whole items), the unit's (split > 1,
    // log_cap per unit) or the piece's (mixed part items: mx.slotinfo)
    uint32_t wlog_n = 0;
    auto log_base = [&](uint32_t k) -> size_t {
        return (split == 1 ? static_cast<size_t>(0) : static_cast<size_t>(k) * log_cap -
                                                          static_cast<size_t>(blockIdx.x) * log_cap) +
               static_cast<size_t>(wid) * (log_cap / SEL_CW);
    };
    auto set_log = [&](uint32_t k, uint32_t*& li, double*& ls) {
        const uint32_t sl = slot_of(k);
        if (sl != NO_SLOT) {
            const uint2 si = __ldg(mx.slotinfo + sl);
            const size_t b = static_cast<size_t>(si.x) + static_cast<size_t>(wid) * si.y;
            li = mx.plog_idx + b;
            ls = mx.plog_sc + b;
        } else {
            li = log_idx + log_base(k);
            ls = log_sc + log_base(k);
        }
    };
    uint32_t* wlog_idx;
    double* wlog_sc;
    set_log(kk, wlog_idx, wlog_sc);
    uint16_t* const wcidx = cidx + wid * WKEYS;
    double* const wacc = acc + wid * WKEYS;
    uint32_t slot = 0, phase = 0;  // ring position of the next chunk
    const uint32_t full0 = smem_u32(&S.full[0]), empty0 = smem_u32(&S.empty[0]);
    const uint32_t ring_s = smem_u32(ring), acc_s = smem_u32(acc);
    auto rmw = [&](const uint2 (&e)[4], uint32_t accb, double w, auto unit_weight) {
        double o[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (!(e[u].x & TOMB)) o[u] = lds_f64(accb + e[u].x * 8u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            // a -0.0f table score (float(dot) of a tiny negative dot,
            // index.cpp:81) is a present key at 0.0 + (-0.0) = +0.0 in
            // reduce_by_key: s + 0.0f canonicalises it, so no term (and no
            // sum) equals the -0.0 "not gathered" marker
            double x = static_cast<double>(__fadd_rn(__uint_as_float(e[u].y), 0.0f));
            if constexpr (!decltype(unit_weight)::value)  // 0.0 + w * double(s)
                x = __dadd_rn(__dmul_rn(w, x), 0.0);
            if (!(e[u].x & TOMB)) sts_f64(accb + e[u].x * 8u, __dadd_rn(o[u], x));
        }
    };
    // this warp's entries of slot positions [x, y): lane-consecutive, four in
    // flight per lane (keys are unique within a list: independent RMWs)
    auto load4 = [&](uint32_t eb, uint32_t x, uint32_t y, uint2 (&e)[4]) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t q = x + ln + 32u * u;
            e[u] = lds_u2(eb + q * 8u);  // the ring has a 128-entry tail pad
            if (q >= y) e[u].x = TOMB;
        }
    };
    while (kk < nwork) {
        mbar_wait_sleep_u32(full0 + 8 * slot, phase);
        const uint32_t info = S.meta[slot].info;
        const uint32_t nsub = info & 7u, flags = (info >> 3) & 7u, tile = info >> 8;
        const uint32_t kbase = tile * TILE;
        const uint32_t eb = ring_s + slot * (SLOT_E * 8u);
        if (!(flags & F_CACHE)) {
            const uint32_t accb = acc_s - kbase * 8u;  // shared address of key k: accb + 8k
            // the slot's list segments in gathered order; the next one's first
            // entries are loaded before the current one is accumulated
            uint2 wr = S.meta[slot].wr[0][wid];
            uint2 e[4];
            if (nsub) load4(eb, wr.x, wr.y, e);
            for (uint32_t sb = 0; sb < nsub; ++sb) {
                const uint32_t list = S.meta[slot].lists[sb];
                uint2 wrn = make_uint2(0u, 0u);
                uint2 en[4];
                if (sb + 1 < nsub) {
                    wrn = S.meta[slot].wr[sb + 1][wid];
                    load4(eb, wrn.x, wrn.y, en);
                }
                if (wr.y > wr.x) {
                    const double w = S.cw[list];
                    auto run = [&](auto unit_weight) {
                        rmw(e, accb, w, unit_weight);
                        for (uint32_t p0 = wr.x + 128; p0 < wr.y; p0 += 128) {  // long ranges
                            uint2 t[4];
                            load4(eb, p0, wr.y, t);
                            rmw(t, accb, w, unit_weight);
                        }
                    };
                    if (w == 1.0) run(std::true_type{});  // w * double(s) == double(s)
                    else run(std::false_type{});
                }
                if (sb + 1 < nsub) {
                    wr = wrn;
#pragma unroll
                    for (int u = 0; u < 4; ++u) e[u] = en[u];
                    // a key of this list and of the next may sit in different
                    // lanes: order the RMWs (memory model, not just issue order)
                    __syncwarp();
                }
            }
        } else {  // cached candidate scores (search_period > 1): this warp's keys
            for (uint32_t u = 0; u < WKEYS / 32; ++u) {
                const uint32_t li = wid * WKEYS + u * 32 + ln, i = kbase + li;
                if (i >= st.N) continue;
                double v = neg0_d();
                if (st.cache && i < st.n_cache) {
                    v = __ldcg(st.cache + i);
                    if (is_absent(v)) v = neg0_d();
                }
                acc[li] = v;
            }
        }
        __syncwarp();
        if (ln == 0) mbar_arrive_u32(empty0 + 8 * slot);
        if (++slot == NSLOT) {
            slot = 0;
            phase ^= 1u;
        }
        // each warp owns its keys in every tile: lists accumulate in order per
        // key without a CTA barrier, and the filter reads only the warp's keys
        if (!(flags & F_TILE_END)) continue;

        // ---- tile end: this warp's 512 keys -> pool candidates ----
        {
            const uint32_t N = st.N, need = st.need, wlo = st.wlo;
            const double lo = st.lo, scale = st.scale;
            const uint32_t cut = *reinterpret_cast<volatile uint32_t*>(&S.cut);
            const double cut_lo = (cut > 1 && scale > 0.0)
                                      ? lo + static_cast<double>(cut - 1) / scale
                                      : -DBL_MAX;  // s < cut_lo  =>  bin(s) < cut
            const uint32_t kw = kbase + wid * WKEYS;  // this warp's first key
            const bool tile_win = kbase + TILE > wlo;  // holds window keys
            double2* const a2 = reinterpret_cast<double2*>(wacc);
            if (!tile_win && !st.store_cache) {
                // common case (every key below the window, nothing cached): one
                // pass per lane over its 16 keys (8 pairs, all loads in flight)
                // builds a survivor mask; the survivors are binned and logged
                // in rounds (about 8% of keys), then the slice is reset
                double2 v[WKEYS / 64];
#pragma unroll
                for (uint32_t u = 0; u < WKEYS / 64; ++u) v[u] = a2[u * 32 + ln];
                if (need) {
                    uint32_t sm = 0;  // bit 2u + c: key 64u + 2ln + c survives the cheap compare
                    if (cut_lo > 0.0) {  // the -0.0 marker fails `>= cut_lo` by itself
#pragma unroll
                        for (uint32_t u = 0; u < WKEYS / 64; ++u)
                            sm |= (v[u].x >= cut_lo ? 1u : 0u) << (2 * u) | (v[u].y >= cut_lo ? 2u : 0u) << (2 * u);
                    } else {
#pragma unroll
                        for (uint32_t u = 0; u < WKEYS / 64; ++u)
                            sm |= ((!is_neg0(v[u].x) && v[u].x >= cut_lo) ? 1u : 0u) << (2 * u) |
                                  ((!is_neg0(v[u].y) && v[u].y >= cut_lo) ? 2u : 0u) << (2 * u);
                    }
                    while (__any_sync(0xffffffffu, sm != 0)) {
                        bool a = false;
                        uint32_t b = 0, koff = 0;
                        double sc = 0.0;
                        if (sm) {
                            const uint32_t bit = __ffs(sm) - 1;
                            sm &= sm - 1;
                            koff = 64 * (bit >> 1) + 2 * ln + (bit & 1);
                            sc = wacc[koff];  // not reset yet
                            b = bin_of(sc, lo, scale);
                            a = b >= cut;
                        }
                        const unsigned m = __ballot_sync(0xffffffffu, a);
                        if (a) {
                            const uint32_t pos = wlog_n + __popc(m & ((1u << ln) - 1u));
                            wlog_idx[pos] = kw + koff;
                            wlog_sc[pos] = sc;
                            atomicAdd(&hist[b], 1u);
                            atomicAdd(&coarse[b >> 5], 1u);
                        }
                        wlog_n += __popc(m);
                    }
                }
                __syncwarp();  // survivors read before the reset
                const double2 nz = make_double2(neg0_d(), neg0_d());
#pragma unroll
                for (uint32_t u = 0; u < WKEYS / 64; ++u) a2[u * 32 + ln] = nz;
            } else {
            // pass 1: cheap compare, survivors compacted to the front of the
            // warp's accumulator slice (positions never pass the read front)
            uint32_t nadm = 0;
            {
#pragma unroll 2
                for (uint32_t u = 0; u < WKEYS / 64; ++u) {
                    const uint32_t lp = u * 32 + ln;
                    const uint32_t i0 = kw + 2 * lp;
                    const double2 v = a2[lp];
                    double s0 = v.x, s1 = v.y;
                    const bool p0 = !is_neg0(s0), p1 = !is_neg0(s1);  // gathered
                    if (st.store_cache) {
                        if (i0 < N) st.cache[i0] = p0 ? s0 : absent_d();
                        if (i0 + 1 < N) st.cache[i0 + 1] = p1 ? s1 : absent_d();
                    }
                    bool in0 = p0, in1 = p1;
                    if (tile_win) {  // window: passthrough keeps them out of the pool;
                                     // otherwise they compete, at 0 when absent
                        if (i0 >= wlo) {
                            in0 = !st.pt && i0 < N;
                            s0 = p0 ? s0 : 0.0;
                        }
                        if (i0 + 1 >= wlo) {
                            in1 = !st.pt && i0 + 1 < N;
                            s1 = p1 ? s1 : 0.0;
                        }
                    }
                    const bool k0 = need && in0 && s0 >= cut_lo, k1 = need && in1 && s1 >= cut_lo;
                    const unsigned m0 = __ballot_sync(0xffffffffu, k0);
                    const unsigned m1 = __ballot_sync(0xffffffffu, k1);
                    if (m0 | m1) {
                        const unsigned lt = (1u << ln) - 1u;
                        const uint32_t n0 = __popc(m0);
                        __syncwarp();  // every lane has read its pair
                        if (k0) {
                            const uint32_t pos = nadm + __popc(m0 & lt);
                            wacc[pos] = s0;
                            wcidx[pos] = static_cast<uint16_t>(2 * lp);
                        }
                        if (k1) {
                            const uint32_t pos = nadm + n0 + __popc(m1 & lt);
                            wacc[pos] = s1;
                            wcidx[pos] = static_cast<uint16_t>(2 * lp + 1);
                        }
                        nadm += n0 + __popc(m1);
                    }
                }
            }
            __syncwarp();
            // pass 2: bin the survivors, count and log those at or above the cut
            for (uint32_t j0 = 0; j0 < nadm; j0 += 32) {
                const uint32_t j = j0 + ln;
                bool a = false;
                uint32_t b = 0;
                double sc = 0.0;
                uint32_t off = 0;
                if (j < nadm) {
                    sc = wacc[j];
                    off = wcidx[j];
                    b = bin_of(sc, lo, scale);
                    a = b >= cut;
                }
                const unsigned m = __ballot_sync(0xffffffffu, a);
                if (a) {
                    const uint32_t pos = wlog_n + __popc(m & ((1u << ln) - 1u));
                    wlog_idx[pos] = kw + off;
                    wlog_sc[pos] = sc;
                    atomicAdd(&hist[b], 1u);
                    atomicAdd(&coarse[b >> 5], 1u);
                }
                wlog_n += __popc(m);
            }
            __syncwarp();
#pragma unroll
            for (uint32_t u = 0; u < WKEYS / 64; ++u)
                a2[u * 32 + ln] = make_double2(neg0_d(), neg0_d());
            }  // generic path
            // raise the cut (stale counts only under-estimate: still safe)
            if (need && (tile % SEL_CW) == static_cast<uint32_t>(wid)) {
                uint32_t ab;
                const int b = warp_find_bin(hist, coarse, need, ab);
                if (ln == 0 && b > static_cast<int>(*reinterpret_cast<volatile uint32_t*>(&S.cut)))
                    atomicMax(&S.cut, static_cast<uint32_t>(b));
            }
        }
        if (!(flags & F_PROB_END)) continue;
        cbar();  // every warp's log and histogram counts are in

        if (unit_meta) {  // part unit / shard: hand histogram + log lengths on
            uint32_t* const um = unit_meta + static_cast<size_t>(kk) * UNIT_META;
            if (ln == 0) um[NB + NCB + wid] = wlog_n;
            cbar();
            for (uint32_t x = tid; x < NB + NCB; x += SEL_CT) {
                um[x] = hist[x];
                hist[x] = 0;
            }
            if (tid == 0) {
                S.cut = 0;
                S.nbkt = 0;
            }
            wlog_n = 0;
            kk += gridDim.x;
            if (kk < nwork) {
                p = prob_of(kk);
                set_log(kk, wlog_idx, wlog_sc);
                setup_problem(S, probs, plans, p, st, speculate, spec_keep);  // ends with a barrier
            } else {
                cbar();
            }
            continue;
        }
        const uint32_t slot = slot_of(kk);
        if (slot != NO_SLOT) {  // mixed-mode piece: dump, and the last piece merges
            uint32_t* const um = mx.umeta + static_cast<size_t>(slot) * UNIT_META;
            if (ln == 0) um[NB + NCB + wid] = wlog_n;
            for (uint32_t x = tid; x < NB + NCB; x += SEL_CT) {
                um[x] = hist[x];
                hist[x] = 0;
            }
            __threadfence();  // this piece's log, histogram and lengths before the count
            cbar();
            const uint2 pi = __ldg(mx.pinfo + p);  // (first slot, pieces) of the problem
            if (tid == 0) S.f_last = atomicAdd(mx.pdone + p, 1u) + 1u == pi.y ? 1u : 0u;
            cbar();
            if (S.f_last) {
                __threadfence();  // the other pieces' data (they fenced before counting)
                {  // the pieces' histograms, every piece's words in flight at once
                    constexpr uint32_t HX = (NB + NCB + SEL_CT - 1) / SEL_CT;  // words per thread
                    uint32_t hv[HX];
#pragma unroll
                    for (uint32_t i = 0; i < HX; ++i) hv[i] = 0;
#pragma unroll 4
                    for (uint32_t j = 0; j < pi.y; ++j) {
                        const uint32_t* u = mx.umeta + static_cast<size_t>(pi.x + j) * UNIT_META;
#pragma unroll
                        for (uint32_t i = 0; i < HX; ++i) {
                            const uint32_t x = tid + i * SEL_CT;
                            if (x < NB + NCB) hv[i] += __ldcg(u + x);
                        }
                    }
#pragma unroll
                    for (uint32_t i = 0; i < HX; ++i) {
                        const uint32_t x = tid + i * SEL_CT;
                        if (x < NB + NCB) hist[x] = hv[i];
                    }
                }
                if (tid < pi.y * SEL_CW) {
                    const uint32_t j = tid / SEL_CW, w = tid % SEL_CW;
                    const uint2 si = __ldg(mx.slotinfo + pi.x + j);
                    S.seg_len[tid] = __ldcg(mx.umeta + static_cast<size_t>(pi.x + j) * UNIT_META + NB + NCB + w);
                    S.seg_off[tid] = si.x + w * si.y;
                }
                cbar();
                final_select(S, st, p, hist, coarse, bm, bkey, bidx, mx.plog_idx, mx.plog_sc, pi.y * SEL_CW,
                             retry_out, retry_out_count);
                const uint32_t nw = div_up(st.N, 32);
                cbar();  // bitmap emitted, scratch free
                for (uint32_t x = tid; x < div_up(nw, 2); x += SEL_CT) acc[x] = neg0_d();
                for (uint32_t x = tid; x < NB + NCB; x += SEL_CT) hist[x] = 0;
                if (tid == 0) mx.pdone[p] = 0;  // ready for the next step
                stamp(2);
            } else {
                stamp(1);
            }
            if (tid == 0) {
                S.cut = 0;
                S.nbkt = 0;
            }
            wlog_n = 0;
            kk += kstep;
            if (kk < nwork) {
                p = prob_of(kk);
                set_log(kk, wlog_idx, wlog_sc);
                setup_problem(S, probs, plans, p, st, speculate, spec_keep);  // ends with a barrier
            } else {
                cbar();
            }
            continue;
        }
        // ======================= final selection =======================
        {
            if (ln == 0) {  // this CTA's log: one segment per warp
                S.seg_len[wid] = wlog_n;
                S.seg_off[wid] = wid * (log_cap / SEL_CW);
            }
            cbar();  // every warp has logged its keys
            final_select(S, st, p, hist, coarse, bm, bkey, bidx, log_idx, log_sc, SEL_CW, retry_out,
                         retry_out_count);
            const uint32_t nw = div_up(st.N, 32);
            cbar();  // bitmap emitted, scratch free
            stamp(3);
            // ---- reset for the next problem ----
            for (uint32_t x = tid; x < div_up(nw, 2); x += SEL_CT) acc[x] = neg0_d();
            for (uint32_t x = tid; x < NB + NCB; x += SEL_CT) hist[x] = 0;
            if (tid == 0) {
                S.cut = 0;
                S.nbkt = 0;
            }
            wlog_n = 0;
            kk += kstep;
            if (kk < nwork) {
                p = prob_of(kk);
                set_log(kk, wlog_idx, wlog_sc);
                setup_problem(S, probs, plans, p, st, speculate, spec_keep);  // ends with a barrier
            } else {
                cbar();
            }
        }
    }
    if (cta_prof && tid == 0) g_cta_ts[2 * blockIdx.x + 1] = gtimer();
}

// Finalise split problems (split > 1): sum the parts' histograms (each part's
// cut is a lower bound of the global threshold bin, so the sum is complete at
// and above it), take the parts' warp logs as segments, run the final
// selection. One 256-thread CTA per problem.
__global__ void __launch_bounds__(SEL_CT)
select_merge_kernel(const DecodeProblem* __restrict__ probs, const RoutePlan* __restrict__ plans,
                    uint32_t split, const uint32_t* __restrict__ unit_meta,
                    const uint32_t* __restrict__ log_idx, const double* __restrict__ log_sc,
                    uint32_t log_cap, double spec_keep, uint32_t* __restrict__ retry_out,
                    uint32_t* __restrict__ retry_out_count) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SelHdr& S = *reinterpret_cast<SelHdr*>(smem_raw);
    unsigned char* p0 = smem_raw + ((sizeof(SelHdr) + 127) & ~size_t(127));
    uint32_t* bm = reinterpret_cast<uint32_t*>(p0);                 // SELECT_MAX_CONTEXT bits
    uint32_t* hist = bm + SELECT_MAX_CONTEXT / 32;                  // NB
    uint32_t* coarse = hist + NB;                                   // NCB
    unsigned long long* bkey = reinterpret_cast<unsigned long long*>(coarse + NCB);  // BKT
    uint32_t* bidx = reinterpret_cast<uint32_t*>(bkey + BKT);       // BKT
    const uint32_t tid = threadIdx.x, p = blockIdx.x;
    if (tid == 0) S.nbkt = 0;
    const uint32_t* um = unit_meta + static_cast<size_t>(p) * split * UNIT_META;
    // the parts' histograms summed with every part's load in flight at once
    // (issued before setup_problem's dependent descriptor loads)
    constexpr uint32_t HX = (NB + NCB + SEL_CT - 1) / SEL_CT;  // words per thread
    uint32_t hv[HX];
#pragma unroll
    for (uint32_t i = 0; i < HX; ++i) hv[i] = 0;
#pragma unroll
    for (uint32_t j = 0; j < static_cast<uint32_t>(MAXPART); ++j) {
        const uint32_t* u = um + static_cast<size_t>(j < split ? j : 0u) * UNIT_META;
#pragma unroll
        for (uint32_t i = 0; i < HX; ++i) {
            const uint32_t x = tid + i * SEL_CT;
            const uint32_t v = (j < split && x < NB + NCB) ? __ldcg(u + x) : 0u;
            hv[i] += v;
        }
    }
    ProbState st;
    // the parts' speculative cut (same hint, read before any part finished)
    setup_problem(S, probs, plans, p, st, true, spec_keep);  // ends with a barrier
#pragma unroll
    for (uint32_t i = 0; i < HX; ++i) {
        const uint32_t x = tid + i * SEL_CT;
        if (x < NB + NCB) hist[x] = hv[i];
    }
    if (tid < split * SEL_CW) {
        const uint32_t j = tid / SEL_CW, w = tid % SEL_CW;
        S.seg_len[tid] = __ldcg(um + static_cast<size_t>(j) * UNIT_META + NB + NCB + w);
        S.seg_off[tid] = (p * split + j) * log_cap + w * (log_cap / SEL_CW);
    }
    cbar();
    final_select(S, st, p, hist, coarse, bm, bkey, bidx, log_idx, log_sc, split * SEL_CW, retry_out,
                 retry_out_count);
}

// ===========================================================================
// Sequence-sharded decode. Shard s holds keys
// [key_lo, key_hi) of every global list (+ appended keys on the owner shard).
// After the per-shard scan (select_kernel in dump mode over the shard's tiles)
// the caller all-reduces the histograms; then:
//   shard_bucket_kernel  threshold bin from the global histogram; this shard's
//                        members of that bin -> bucket (caller all-gathers)
//   shard_mark_kernel    rank the gathered bucket globally (score desc, index
//                        asc) -> local selection bitmap; per-shard (selected,
//                        untaken) counts (caller all-gathers)
//   shard_emit_kernel    newest-first padding across shards (higher shards hold
//                        newer keys) and the ascending local selection + its
//                        size for attend
// Every shard computes the same global threshold, so the union of the local
// selections is exactly the unsharded selection.
// ===========================================================================
struct ShardPState {
    uint32_t dsel, above, take_all, nbkt;
};
constexpr uint32_t SHARD_BCAP = 2048;  // bucket members per problem per shard

// flat log index -> (segment) for a problem's dump-mode log (one unit per problem)
struct LogView {
    const uint32_t* idx;
    const double* sc;
    const uint32_t* wl;  // per-warp lengths (unit_meta tail)
    size_t base;         // p * log_cap
    uint32_t stride;     // log_cap / SEL_CW
};

__global__ void __launch_bounds__(SEL_CT)
shard_bucket_kernel(const DecodeProblem* __restrict__ probs, const RoutePlan* __restrict__ plans,
                    const uint32_t* __restrict__ ghist, const uint32_t* __restrict__ unit_meta,
                    const uint32_t* __restrict__ log_idx, const double* __restrict__ log_sc,
                    uint32_t log_cap, uint32_t split, uint4* __restrict__ bucket,
                    ShardPState* __restrict__ pstate, double spec_keep,
                    uint32_t* __restrict__ spec_fail) {
    __shared__ SelHdr S;
    const uint32_t tid = threadIdx.x, p = blockIdx.x;
    ProbState st;
    // the scan's speculative cut (same hint, same margin) for the verification
    setup_problem(S, probs, plans, p, st, spec_keep > 0.0, spec_keep);
    const uint32_t* gh = ghist + static_cast<size_t>(p) * (NB + NCB);
    if (tid < 32) {
        uint32_t ab = 0;
        int b = -1;
        if (st.need) b = warp_find_bin(gh, gh + NB, st.need, ab);
        if (tid == 0) {
            S.f_take_all = (st.need && b < 0) ? 1u : 0u;
            S.f_bin = b < 0 ? 0u : static_cast<uint32_t>(b);
            S.f_above = ab;
            S.nbkt = 0;
            // a speculative cut above the global threshold bin lost candidates:
            // the caller rescans without speculation (every shard sees the same
            // global histogram, so they agree)
            if (st.need && st.cut_init && (b < 0 || static_cast<uint32_t>(b) < st.cut_init))
                atomicOr(spec_fail, 1u);
        }
    }
    cbar();
    const uint32_t dsel = S.f_bin;
    const bool collect = st.need && !S.f_take_all;
    uint4* bk = bucket + static_cast<size_t>(p) * (SHARD_BCAP + 1);
    if (collect) {
        for (uint32_t sg = 0; sg < split * SEL_CW; ++sg) {  // (part unit, warp) log segments
            const uint32_t u = p * split + sg / SEL_CW, w = sg % SEL_CW;
            const size_t base = static_cast<size_t>(u) * log_cap + w * (log_cap / SEL_CW);
            const uint32_t n = __ldcg(unit_meta + static_cast<size_t>(u) * UNIT_META + NB + NCB + w);
            for (uint32_t e = tid; e < n; e += SEL_CT) {
                const double sv = __ldcg(log_sc + base + e);
                if (bin_of(sv, st.lo, st.scale) != dsel) continue;
                const uint32_t k = atomicAdd(&S.nbkt, 1u);
                if (k < SHARD_BCAP) {
                    const unsigned long long key = ordkey(sv);
                    bk[1 + k] = make_uint4(static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32),
                                           __ldcg(log_idx + base + e), 0u);
                }
            }
        }
    }
    cbar();
    if (tid == 0) {
        bk[0] = make_uint4(min(S.nbkt, SHARD_BCAP), S.nbkt > SHARD_BCAP ? 1u : 0u, 0u, 0u);
        pstate[p] = ShardPState{dsel, S.f_above, S.f_take_all, S.nbkt};
    }
}

__global__ void __launch_bounds__(SEL_CT)
shard_mark_kernel(const DecodeProblem* __restrict__ probs, const RoutePlan* __restrict__ plans,
                  const ShardPState* __restrict__ pstate, const uint4* __restrict__ bucket_all,
                  uint32_t nshard, uint32_t nprob, const uint32_t* __restrict__ unit_meta,
                  const uint32_t* __restrict__ log_idx, const double* __restrict__ log_sc,
                  uint32_t log_cap, uint32_t split, uint32_t* __restrict__ bitmap,
                  uint32_t bm_words, uint32_t* __restrict__ counts) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SelHdr& S = *reinterpret_cast<SelHdr*>(smem_raw);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw + ((sizeof(SelHdr) + 127) & ~size_t(127)));
    const uint32_t tid = threadIdx.x, p = blockIdx.x;
    ProbState st;
    setup_problem(S, probs, plans, p, st, false, 0.0);
    const SessionDev& sd = *probs[p].s;
    const ShardPState ps = pstate[p];
    const uint32_t need = st.need, N = st.N;
    const uint32_t rem = need - (ps.take_all ? 0u : min(need, ps.above));
    // gathered bucket: shard j's members at bucket_all[(j*nprob + p)*(BCAP+1) + 1 ..]
    if (tid == 0) {
        uint32_t run = 0;
        for (uint32_t j = 0; j <= nshard; ++j) {
            S.seg_pre[j] = run;
            if (j < nshard)
                run += __ldcg(&bucket_all[(static_cast<size_t>(j) * nprob + p) * (SHARD_BCAP + 1)].x);
        }
    }
    cbar();
    const uint32_t nb = S.seg_pre[nshard];
    auto member = [&](uint32_t e, unsigned long long& k, uint32_t& ix) {
        uint32_t j = 0;
        while (S.seg_pre[j + 1] <= e) ++j;
        const uint4 v = __ldcg(&bucket_all[(static_cast<size_t>(j) * nprob + p) * (SHARD_BCAP + 1) + 1 +
                                           (e - S.seg_pre[j])]);
        k = (static_cast<unsigned long long>(v.y) << 32) | v.x;
        ix = v.z;
        return true;
    };
    unsigned long long tk = ~0ull;
    uint32_t tx = 0;
    if (need && !ps.take_all && rem) {
        radix_kth(S, hist, nb, rem, member);
        tk = S.tk;
        tx = S.tx;
    }
    // local selection bitmap over this shard's key range
    const uint32_t klo = sd.key_lo;
    const uint32_t khi = sd.owner ? N : min(sd.key_hi, N);
    const uint32_t nwb = khi > klo ? div_up(khi - klo, 32) : 0u;
    uint32_t* bm = bitmap + static_cast<size_t>(p) * bm_words;
    for (uint32_t x = tid; x < nwb; x += SEL_CT) bm[x] = 0;
    cbar();
    if (need) {
        for (uint32_t sg = 0; sg < split * SEL_CW; ++sg) {  // (part unit, warp) log segments
            const uint32_t u = p * split + sg / SEL_CW, w = sg % SEL_CW;
            const size_t base = static_cast<size_t>(u) * log_cap + w * (log_cap / SEL_CW);
            const uint32_t n = __ldcg(unit_meta + static_cast<size_t>(u) * UNIT_META + NB + NCB + w);
            for (uint32_t e = tid; e < n; e += SEL_CT) {
                const double sv = __ldcg(log_sc + base + e);
                const uint32_t b = bin_of(sv, st.lo, st.scale);
                bool on = ps.take_all || b > ps.dsel;
                if (!on && b == ps.dsel) {
                    const unsigned long long k = ordkey(sv);
                    on = k > tk || (k == tk && __ldcg(log_idx + base + e) < tx);
                }
                if (on) {
                    const uint32_t i = __ldcg(log_idx + base + e);
                    atomicOr(bm + ((i - klo) >> 5), 1u << ((i - klo) & 31));
                }
            }
        }
    }
    // window passthrough (or the newest K when K <= R) within this shard
    for (uint32_t i = max(st.f_lo, klo) + tid; i < khi; i += SEL_CT)
        atomicOr(bm + ((i - klo) >> 5), 1u << ((i - klo) & 31));
    cbar();
    uint32_t cnt = 0;
    for (uint32_t x = tid; x < nwb; x += SEL_CT) cnt += __popc(bm[x]);
    uint32_t total;
    cscan(S, cnt, total);
    if (tid == 0) {
        // next step's speculative cut: the global threshold bin's lower edge
        st.hint[0] = st.scale > 0.0 ? st.lo + static_cast<double>(ps.dsel) / st.scale : st.lo;
        st.hint[1] = (need && !ps.take_all) ? 1.0 : 0.0;
        counts[2 * p] = total;
        counts[2 * p + 1] = (khi > klo ? khi - klo : 0u) - total;  // untaken keys of the range
    }
}

__global__ void __launch_bounds__(SEL_CT)
shard_emit_kernel(const DecodeProblem* __restrict__ probs, const RoutePlan* __restrict__ plans,
                  const uint32_t* __restrict__ counts_all, uint32_t nshard, uint32_t shard,
                  uint32_t nprob, uint32_t* __restrict__ bitmap, uint32_t bm_words,
                  uint32_t* __restrict__ kdev) {
    __shared__ SelHdr S;
    const uint32_t tid = threadIdx.x, p = blockIdx.x;
    ProbState st;
    setup_problem(S, probs, plans, p, st, false, 0.0);
    const SessionDev& sd = *probs[p].s;
    const uint32_t N = st.N, K = st.K;
    uint32_t total = 0, above = 0;
    for (uint32_t j = 0; j < nshard; ++j) {
        total += __ldcg(counts_all + (static_cast<size_t>(j) * nprob + p) * 2);
        if (j > shard) above += __ldcg(counts_all + (static_cast<size_t>(j) * nprob + p) * 2 + 1);
    }
    const uint32_t klo = sd.key_lo;
    const uint32_t khi = sd.owner ? N : min(sd.key_hi, N);
    const uint32_t nwb = khi > klo ? div_up(khi - klo, 32) : 0u;
    uint32_t* bm = bitmap + static_cast<size_t>(p) * bm_words;
    const uint32_t wpt = div_up(nwb, SEL_CT);
    const uint32_t w0 = min(nwb, tid * wpt), w1 = min(nwb, w0 + wpt);
    auto valid = [&](uint32_t x) {
        const uint32_t r = khi - klo;
        return x + 1 < nwb || (r & 31) == 0 ? 0xffffffffu : ((1u << (r & 31)) - 1u);
    };
    uint32_t cnt = 0, zeros = 0;
    for (uint32_t x = w0; x < w1; ++x) {
        cnt += __popc(bm[x]);
        zeros += __popc(~bm[x] & valid(x));
    }
    if (total < K) {  // newest untaken keys first: higher shards, then this one's top
        const uint32_t pad = K - total;
        uint32_t zt;
        const uint32_t zbelow = cscan(S, zeros, zt);
        const uint32_t mine = pad > above ? min(pad - above, zt) : 0u;  // this shard's share
        const uint32_t zabove = zt - zbelow - zeros;
        uint32_t take = mine > zabove ? min(mine - zabove, zeros) : 0u;
        for (uint32_t x = w1; x > w0 && take;) {
            --x;
            uint32_t z = ~bm[x] & valid(x);
            while (z && take) {
                const int hb = 31 - __clz(z);
                bm[x] |= 1u << hb;
                z &= ~(1u << hb);
                --take;
                ++cnt;
            }
        }
    }
    uint32_t n_local;
    const uint32_t at = cscan(S, cnt, n_local);
    uint32_t pos = at;
    for (uint32_t x = w0; x < w1; ++x) {
        uint32_t b = bm[x];
        while (b) {
            const int lb = __ffs(b) - 1;
            st.sel[pos++] = klo + x * 32 + lb;
            b &= b - 1;
        }
    }
    if (tid == 0) {
        kdev[p] = n_local;
        // attend reads K from the (device) descriptor: this shard's share
        const_cast<DecodeProblem*>(probs)[p].K = n_local;
        reinterpret_cast<DecodeReport*>(st.rep)->k = K;
    }
}

uint32_t shard_bucket_words() { return (SHARD_BCAP + 1) * 4; }
uint32_t shard_hist_words() { return NB + NCB; }

// per problem: sum of its `split` part units' histograms -> ghist (the shard's
// histogram, all-reduced over the shards by the caller)
__global__ void shard_hist_sum_kernel(const uint32_t* __restrict__ unit_meta, uint32_t split,
                                      uint32_t* __restrict__ ghist) {
    const uint32_t p = blockIdx.x;
    for (uint32_t x = threadIdx.x; x < NB + NCB; x += blockDim.x) {
        uint32_t v = 0;
        for (uint32_t j = 0; j < split; ++j)
            v += __ldcg(unit_meta + (static_cast<size_t>(p) * split + j) * UNIT_META + x);
        ghist[static_cast<size_t>(p) * (NB + NCB) + x] = v;
    }
}

cudaError_t launch_shard_hist_sum(const uint32_t* unit_meta, uint32_t nprob, uint32_t split,
                                  uint32_t* ghist, cudaStream_t st) {
    shard_hist_sum_kernel<<<nprob, 256, 0, st>>>(unit_meta, split, ghist);
    return cudaGetLastError();
}

cudaError_t launch_shard_bucket(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                                const uint32_t* ghist, const uint32_t* unit_meta,
                                const uint32_t* log_idx, const double* log_sc, uint32_t log_cap,
                                uint32_t split, void* bucket, void* pstate, double spec_keep,
                                uint32_t* spec_fail, cudaStream_t st) {
    shard_bucket_kernel<<<nprob, SEL_CT, 0, st>>>(probs, plans, ghist, unit_meta, log_idx, log_sc,
                                                   log_cap, split, static_cast<uint4*>(bucket),
                                                   static_cast<ShardPState*>(pstate), spec_keep,
                                                   spec_fail);
    return cudaGetLastError();
}

cudaError_t launch_shard_mark(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                              const void* pstate, const void* bucket_all, uint32_t nshard,
                              const uint32_t* unit_meta, const uint32_t* log_idx,
                              const double* log_sc, uint32_t log_cap, uint32_t split,
                              uint32_t* bitmap, uint32_t bm_words, uint32_t* counts,
                              cudaStream_t st) {
    const size_t smem = ((sizeof(SelHdr) + 127) & ~size_t(127)) + NB * 4;
    shard_mark_kernel<<<nprob, SEL_CT, smem, st>>>(
        probs, plans, static_cast<const ShardPState*>(pstate), static_cast<const uint4*>(bucket_all),
        nshard, nprob, unit_meta, log_idx, log_sc, log_cap, split, bitmap, bm_words, counts);
    return cudaGetLastError();
}

cudaError_t launch_shard_emit(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                              const uint32_t* counts_all, uint32_t nshard, uint32_t shard,
                              uint32_t* bitmap, uint32_t bm_words, uint32_t* kdev, cudaStream_t st) {
    shard_emit_kernel<<<nprob, SEL_CT, 0, st>>>(probs, plans, counts_all, nshard, shard, nprob,
                                                bitmap, bm_words, kdev);
    return cudaGetLastError();
}

uint32_t shard_pstate_bytes() { return sizeof(ShardPState); }

static size_t select_smem() {
    return ((sizeof(SelHdr) + 127) & ~size_t(127)) + TILE * 8 + (NB + NCB) * 4 + BKT * 12 +
           SEL_CW * WKEYS * 2 + (static_cast<size_t>(NSLOT) * SLOT_E + 128) * 8;
}

uint32_t select_grid(uint32_t nprob, int num_sms) {
    const uint32_t g = 2u * static_cast<uint32_t>(num_sms > 0 ? num_sms : 1);  // 2 CTAs per SM
    return nprob < g ? nprob : g;
}

uint32_t select_unit_meta_words() { return UNIT_META; }
uint32_t select_ctas_per_sm() { return 2; }
cudaError_t select_fin_debug(unsigned long long* out8, cudaStream_t st) {
    cudaError_t e = cudaMemcpyFromSymbolAsync(out8, g_fin_dbg, 64, 0, cudaMemcpyDeviceToHost, st);
    static const unsigned long long z[8] = {};
    if (e == cudaSuccess) e = cudaMemcpyToSymbolAsync(g_fin_dbg, z, 64, 0, cudaMemcpyHostToDevice, st);
    return e;
}
cudaError_t select_cta_times(unsigned long long* out, uint32_t n, cudaStream_t st) {
    n = n < SEL_TS_MAX ? n : SEL_TS_MAX;
    cudaError_t e = cudaMemcpyFromSymbolAsync(out, g_cta_ts, 16 * n, 0, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
        e = cudaMemcpyFromSymbolAsync(out + 2 * n, g_cta_ev, 64 * n, 0, cudaMemcpyDeviceToHost, st);
    return e;
}
uint32_t select_tile_keys() { return TILE; }

cudaError_t launch_select_merge(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                                uint32_t split, const uint32_t* unit_meta, const uint32_t* log_idx,
                                const double* log_sc, uint32_t log_cap, double spec_keep,
                                uint32_t* retry_out, uint32_t* retry_out_count, cudaStream_t st) {
    const size_t smem = ((sizeof(SelHdr) + 127) & ~size_t(127)) + SELECT_MAX_CONTEXT / 8 +
                        (NB + NCB) * 4 + BKT * 12;
    cudaError_t e = cudaFuncSetAttribute(select_merge_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    select_merge_kernel<<<nprob, SEL_CT, smem, st>>>(probs, plans, split, unit_meta, log_idx, log_sc,
                                                     log_cap, spec_keep, retry_out, retry_out_count);
    return cudaGetLastError();
}

cudaError_t launch_select(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                          uint32_t grid, uint32_t* log_idx, double* log_sc, uint32_t log_cap,
                          const uint32_t* retry_in, const uint32_t* retry_in_count,
                          uint32_t* retry_out, uint32_t* retry_out_count, double spec_keep,
                          uint32_t split, uint32_t* unit_meta, cudaStream_t st, const SelMixed* mixed,
                          bool pdl) {
    const size_t smem = select_smem();
    {  // once per device (a host call per launch otherwise)
        static bool set[64] = {};
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev < 0 || dev >= 64 || !set[dev]) {
            e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem));
            if (e != cudaSuccess) return e;
            if (dev >= 0 && dev < 64) set[dev] = true;
        }
    }
    const SelMixed mx = mixed ? *mixed : SelMixed{};
    if (pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(SEL_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, select_kernel, probs, plans, nprob, log_idx, log_sc, log_cap,
                                  retry_in, retry_in_count, retry_out, retry_out_count, spec_keep,
                                  split, unit_meta, mx);
    }
    select_kernel<<<grid, SEL_THREADS, smem, st>>>(probs, plans, nprob, log_idx, log_sc, log_cap,
                                                   retry_in, retry_in_count, retry_out,
                                                   retry_out_count, spec_keep, split, unit_meta, mx);
    return cudaGetLastError();
}

}  // namespace csa
