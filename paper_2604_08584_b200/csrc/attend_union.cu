// attend_union.cu — sparse attention for problems that share one prefill
// (masked dense_attention, core.cpp:118-169), on sm_100a tensor cores.
//
// The batch-decode case (config c3: 16 sequences forked from one prefill, GQA
// groups of 4 -> 64 (sequence, head) problems per KV head) selects each prefill
// row ~6x on average. The per-problem path (attend.cu) handles every
// (problem, selected row) pair on CUDA cores. Here a group of <= 64 problems
// ("members") on one prefill is processed by prefill ROW RANGE as a small dense
// attention over the UNION of their selected rows, masked per member:
//   union_build_kernel  per (group, range of UN_RANGE prefill rows): each
//                       member's selected rows in the range (binary search in
//                       its ascending list) are marked in a shared-memory
//                       bitmask (bit b = member b) and compacted -> global
//                       union list (row offsets, member masks, count)
//   attend_tc_kernel    persistent, one CTA per SM over the (group, range)
//                       items: tiles of 64 union rows, S = Q K^T and O += P V
//                       on tcgen05 (operands in swizzled smem, accumulators in
//                       TMEM), masked online softmax in between
//                       -> partial (max, sum, acc[128]) per (member, range)
//   attend_tail_kernel  per member: its appended rows (index >= P, private to
//                       its session), one warp -> a partial
//   union_merge_kernel  per member: log-sum-exp of its range partials in range
//                       order, then the tail -> output
// Every problem attends exactly its own selected rows (its mask bit) in a fixed
// order, so results are deterministic and independent of how problems are
// grouped.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace csa {

constexpr uint32_t UN_PART = UN_PART_WORDS;  // max, sum, 2 pad, acc[128]
constexpr uint32_t UN_NONE = 0xffffffffu;
// attend_tc_kernel shared-memory operand offsets (see TcSmem)
constexpr uint32_t TcSmem_K0 = 0, TcSmem_KSZ = 32768, TcSmem_V0 = 65536, TcSmem_VSZ = 32768;
constexpr uint32_t TcSmem_QHI = 131072, TcSmem_QLO = 147456, TcSmem_P0 = 163840, TcSmem_PSZ = 16384;

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t key) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// ---- union lists: one CTA per (group, range) ----
constexpr int UB_THREADS = 256;
__global__ void __launch_bounds__(UB_THREADS)
union_build_kernel(const DecodeProblem* __restrict__ probs, const uint32_t* __restrict__ members,
                   const uint32_t* __restrict__ gmember, const uint32_t* __restrict__ gP,
                   uint32_t nrange, uint16_t* __restrict__ urow, unsigned long long* __restrict__ umask,
                   uint32_t* __restrict__ ucount) {
    __shared__ unsigned long long mask[UN_RANGE];
    __shared__ uint32_t lo_s[64], hi_s[64], wcount[UB_THREADS / 32];
    __shared__ const uint32_t* sel_s[64];
    const uint32_t item = blockIdx.x, g = item / nrange, r = item % nrange;
    const uint32_t tid = threadIdx.x;
    const int w = tid >> 5, ln = tid & 31;
    const uint32_t P0 = gP[g], r0 = r * UN_RANGE;
    if (r0 >= P0) return;
    const uint32_t r1 = min(P0, r0 + UN_RANGE);
    for (uint32_t i = tid; i < UN_RANGE; i += UB_THREADS) mask[i] = 0ull;
    if (tid < 128) {  // member tid >> 1: bound tid & 1
        const uint32_t b = tid >> 1, kk = gmember[g * UN_GROUP + b];
        uint32_t v = 0;
        const uint32_t* sel = nullptr;
        if (kk != UN_NONE) {
            const DecodeProblem& Pb = probs[members[kk]];
            sel = Pb.sel;
            v = lower_bound_u32(sel, Pb.K, (tid & 1) ? r1 : r0);
        }
        if (tid & 1)
            hi_s[b] = v;
        else {
            lo_s[b] = v;
            sel_s[b] = sel;
        }
    }
    __syncthreads();
    // warp w marks members 8w..8w+7 (32-bit halves: native shared atomics)
    uint32_t* m32 = reinterpret_cast<uint32_t*>(mask) + (w >= 4 ? 1 : 0);
    for (int j = 0; j < 8; ++j) {
        const uint32_t b = 8 * w + j;
        const uint32_t* sel = sel_s[b];
        if (!sel) continue;
        const uint32_t bit = 1u << (b & 31);
        for (uint32_t e = lo_s[b] + ln; e < hi_s[b]; e += 32) atomicOr(m32 + 2 * (__ldg(sel + e) - r0), bit);
    }
    __syncthreads();
    // compaction (thread order = row order)
    constexpr int PER = UN_RANGE / UB_THREADS;
    unsigned long long v[PER];
    uint32_t n = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        v[i] = mask[tid * PER + i];
        n += v[i] != 0ull;
    }
    uint32_t inc = n;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (ln >= o) inc += y;
    }
    if (ln == 31) wcount[w] = inc;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < UB_THREADS / 32; ++i) {
        pre += i < w ? wcount[i] : 0u;
        tot += wcount[i];
    }
    uint32_t pos = pre + inc - n;
    uint16_t* ur = urow + static_cast<size_t>(item) * UN_RANGE;
    unsigned long long* um = umask + static_cast<size_t>(item) * UN_RANGE;
#pragma unroll
    for (int i = 0; i < PER; ++i)
        if (v[i]) {
            ur[pos] = static_cast<uint16_t>(tid * PER + i);
            um[pos] = v[i];
            ++pos;
        }
    if (tid == 0) ucount[item] = tot;
}

__device__ __forceinline__ float4 ld4(const float* p, int ln) {
    return reinterpret_cast<const float4*>(p)[ln];
}
__device__ __forceinline__ float dot4(float4 a, float4 b) {
    return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x)));
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// One member over up to four rows (kr[u], vr[u], u < n) with online softmax in
// base 2 (q is pre-scaled by log2(e)/sqrt(d), so exp(x) = 2^(x log2 e)).
// Transposed butterfly: after the xor-16 and xor-8 exchanges lane l holds the
// partial dot of row (l >> 3) & 3, then a 3-step reduction completes it. The
// accumulator is rescaled only when the running max grows.
__device__ __forceinline__ void group4(const float* const kr[4], const float* const vr[4], int n,
                                       float4 q, float& m, float& s, float4& acc, int ln) {
    const float4 k0 = ld4(kr[0], ln), k1 = ld4(kr[1], ln), k2 = ld4(kr[2], ln), k3 = ld4(kr[3], ln);
    const float4 v0 = ld4(vr[0], ln), v1 = ld4(vr[1], ln), v2 = ld4(vr[2], ln), v3 = ld4(vr[3], ln);
    const float d0 = dot4(q, k0), d1 = dot4(q, k1), d2 = dot4(q, k2), d3 = dot4(q, k3);
    const bool h16 = ln & 16, h8 = ln & 8;
    float a0 = h16 ? d2 : d0, a1 = h16 ? d3 : d1;
    const float b0 = h16 ? d0 : d2, b1 = h16 ? d1 : d3;
    a0 += __shfl_xor_sync(0xffffffffu, b0, 16);
    a1 += __shfl_xor_sync(0xffffffffu, b1, 16);
    float c = h8 ? a1 : a0;
    c += __shfl_xor_sync(0xffffffffu, h8 ? a0 : a1, 8);
    c += __shfl_xor_sync(0xffffffffu, c, 4);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    const bool ok = ((ln >> 3) & 3) < n;
    const float lg = ok ? c : -FLT_MAX;
    float mg = fmaxf(lg, __shfl_xor_sync(0xffffffffu, lg, 8));
    mg = fmaxf(mg, __shfl_xor_sync(0xffffffffu, mg, 16));
    if (mg > m) {  // warp-uniform
        const float f = ex2(m - mg);
        s *= f;
        acc.x *= f;
        acc.y *= f;
        acc.z *= f;
        acc.w *= f;
        m = mg;
    }
    const float pr = ok ? ex2(lg - m) : 0.0f;
    float ps = pr + __shfl_xor_sync(0xffffffffu, pr, 8);
    ps += __shfl_xor_sync(0xffffffffu, ps, 16);
    s += ps;
    const float p0 = __shfl_sync(0xffffffffu, pr, 0), p1 = __shfl_sync(0xffffffffu, pr, 8);
    const float p2 = __shfl_sync(0xffffffffu, pr, 16), p3 = __shfl_sync(0xffffffffu, pr, 24);
    acc.x = fmaf(p3, v3.x, fmaf(p2, v2.x, fmaf(p1, v1.x, fmaf(p0, v0.x, acc.x))));
    acc.y = fmaf(p3, v3.y, fmaf(p2, v2.y, fmaf(p1, v1.y, fmaf(p0, v0.y, acc.y))));
    acc.z = fmaf(p3, v3.z, fmaf(p2, v2.z, fmaf(p1, v1.z, fmaf(p0, v0.z, acc.z))));
    acc.w = fmaf(p3, v3.w, fmaf(p2, v2.w, fmaf(p1, v1.w, fmaf(p0, v0.w, acc.w))));
}

// q row pre-scaled for base-2 logits
__device__ __forceinline__ float4 load_q2(const float* q, int ln) {
    const float c = static_cast<float>(1.4426950408889634 / sqrt(128.0));
    float4 x = __ldg(reinterpret_cast<const float4*>(q) + ln);
    x.x *= c;
    x.y *= c;
    x.z *= c;
    x.w *= c;
    return x;
}

// ---- tensor-core union attention: one persistent CTA per SM ----
// Item = (group g, range r); its union rows in tiles of 64, FlashAttention-4
// orientation (member = TMEM lane):
//   S[member][row] = Q . K_tile^T   (tcgen05 M = 128: 64 members + padding, N = 64)
//   P[member][row] = mask ? 2^(S - m_member) : 0
//   O[member][dim] += P . V_tile    (tcgen05 M = 128, N = 128)
// fp32 operands are split into bf16 hi + lo; each product is three MMAs
// (hi.hi + lo.hi + hi.lo, ~2^-16 relative: fp32-grade). Consecutive MMAs into
// one accumulator serialise (~128 cycles each on B200 whatever N is), so S and
// O each use two accumulators that the MMAs alternate between (summed when
// read). Q is pre-scaled by log2(e)/sqrt(d): base-2 logits. A member's
// running max is raised only when a tile exceeds it by more than UN_TAU (lazy
// rescale of its O row), so P <= 2^UN_TAU. MMA lanes 64-127 read padding.
// Roles (warps 0-17; warp w runs on SM sub-partition w % 4, which also fixes
// its TMEM lane quadrant): w % 4 in {0, 1}, w < 16 (8 warps): softmax, member
// (w & 1) * 32 + lane over tile rows 16 (w >> 2) .. +15; warp 2: QK issuer,
// warp 6: PV issuer (one thread each: issuing a tcgen05.mma costs ~70 cycles
// on B200, so at N = 64 / 128 the issue streams, not the tensor core, pace a
// tile and two streams overlap); warps 3, 7, 11, 15: K loaders; 10, 14, 16,
// 17: V loaders (global -> regs -> bf16 hi/lo -> swizzled smem).
// K, V, P and S are double-buffered; mbarrier rings connect the roles.
constexpr int TC_LOAD = 128;
constexpr int TC_THREADS = 18 * 32;  // 576
__device__ __forceinline__ int loader_slot(int w) {  // 0-3 K, 4-7 V, -1 other
    switch (w) {  // K and V loaders alternate over sub-partitions 2 and 3
        case 3: return 0;
        case 10: return 1;
        case 7: return 2;
        case 14: return 3;
        case 11: return 4;
        case 15: return 5;
        case 16: return 6;
        case 17: return 7;
        default: return -1;
    }
}
// MMA issue with every descriptor a compile-time offset from uniform bases
template <int B>
__device__ __forceinline__ void issue_qk(uint32_t sbase, uint32_t tS, uint32_t id_qk) {
    const uint32_t kb = sbase + TcSmem_K0 + B * TcSmem_KSZ;
    const uint32_t d0 = tS + B * 128, d1 = d0 + 64;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const uint32_t o = (s >> 2) * 64 * 128 + (s & 3) * 32;
        const uint64_t qhi = tc::desc_sw128(sbase + TcSmem_QHI + o, 16, 1024);
        const uint64_t qlo = tc::desc_sw128(sbase + TcSmem_QLO + o, 16, 1024);
        const uint64_t khi = tc::desc_sw128(kb + o, 16, 1024);
        const uint64_t klo = tc::desc_sw128(kb + 16384 + o, 16, 1024);
        // MMA i = 3s + term -> accumulator i & 1 (independent chains)
        tc::mma_bf16((3 * s) & 1 ? d1 : d0, qhi, khi, id_qk, s > 0);
        tc::mma_bf16((3 * s + 1) & 1 ? d1 : d0, qlo, khi, id_qk, s > 0 || (3 * s + 1) > 1);
        tc::mma_bf16((3 * s + 2) & 1 ? d1 : d0, qhi, klo, id_qk, 1);
    }
}
template <int B>
__device__ __forceinline__ void issue_pv(uint32_t sbase, uint32_t tO, uint32_t id_pv, bool first) {
    const uint32_t vb = sbase + TcSmem_V0 + B * TcSmem_VSZ;
    const uint32_t pb = sbase + TcSmem_P0 + B * TcSmem_PSZ;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const uint64_t phi = tc::desc_sw128(pb + s * 32, 16, 1024);
        const uint64_t plo = tc::desc_sw128(pb + 8192 + s * 32, 16, 1024);
        const uint64_t vhi = tc::desc_sw128(vb + s * 2048, 8192, 1024);
        const uint64_t vlo = tc::desc_sw128(vb + 16384 + s * 2048, 8192, 1024);
        const int i0 = 3 * s;
        tc::mma_bf16(tO + 128 * (i0 & 1), phi, vhi, id_pv, (!first || i0 > 1) ? 1u : 0u);
        tc::mma_bf16(tO + 128 * ((i0 + 1) & 1), plo, vhi, id_pv, (!first || i0 + 1 > 1) ? 1u : 0u);
        tc::mma_bf16(tO + 128 * ((i0 + 2) & 1), phi, vlo, id_pv, 1);
    }
}
constexpr uint32_t TC_TILE = 64;
constexpr float UN_TAU = 8.0f;
struct TcSmem {  // 1024-byte aligned operand buffers
    static constexpr uint32_t K0 = 0, KSZ = 32768;        // K tile (B of QK, K-major): hi | lo; x2
    static constexpr uint32_t V0 = 65536, VSZ = 32768;    // V tile (B of PV, MN-major): hi | lo; x2
    static constexpr uint32_t QHI = 131072, QLO = 147456; // Q (A of QK, K-major, 64 rows)
    static constexpr uint32_t P0 = 163840, PSZ = 16384;   // P (A of PV, K-major, 64 rows): hi | lo; x2
    static constexpr uint32_t MISC = 196608;
    // MMA lanes 64-127 of the last P slot read up to 8 KB past it: keep it in bounds
    static constexpr uint32_t CROW = MISC + 8192;       // u16[UN_RANGE]: the item's union rows
    static constexpr uint32_t BYTES = CROW + UN_RANGE * 2;
};
static_assert(TcSmem::BYTES + 1024 <= 232448, "shared memory budget");
struct TcMisc {
    uint64_t kfull[2], vfull[2], kempty[2], vempty[2], sfull[2], pfull[2], odone;
    const float* kv[2];
    uint32_t nu, tbase;
    uint32_t kidx[64];
    float hmax[4][64];  // [row quarter][member]
    float hsum[4][64];
};
static_assert(sizeof(TcMisc) <= 4096, "misc");

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tc::smem_u32(b)) : "memory");
}
__device__ __forceinline__ void math_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }
// x = hi + lo with hi = bf16(x), lo = bf16(x - hi): 16 significant bits
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    const float2 hf = __bfloat1622float2(h);
    const __nv_bfloat162 l = __floats2bfloat162_rn(x - hf.x, y - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};\n" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void store4_split(uint32_t hi_addr, uint32_t lo_addr, float4 v) {
    uint32_t h0, l0, h1, l1;
    split2(v.x, v.y, h0, l0);
    split2(v.z, v.w, h1, l1);
    sts64(hi_addr, h0, h1);
    sts64(lo_addr, l0, l1);
}

// K (PASS 0) or V (PASS 1) loader warps: tile t of the item into slot T & 1
template <int PASS>
__device__ __forceinline__ void tc_loader(TcMisc& X, uint32_t sbase, const float* src, const uint16_t* urow,
                                          uint32_t nu, uint32_t ntile, uint32_t lt, uint32_t& T,
                                          unsigned long long* ts) {
    constexpr int NV = TC_TILE * 32 / TC_LOAD;  // float4 per thread per tile (8)
    constexpr uint32_t PF = 4;                  // L2 prefetch distance (tiles)
    auto prefetch_tile = [&](uint32_t tt) {
        if (lt < TC_TILE && tt < ntile) {
            const uint32_t u = tt * TC_TILE + lt;
            if (u < nu) prefetch_l2(src + static_cast<size_t>(urow[u]) * 128, 512);
        }
    };
    // software pipeline over half tiles: the loads of item j + 1 are in
    // flight while item j waits for its slot, converts and stores
    constexpr int NH = NV / 2;
    auto load_half = [&](uint32_t item, float4 (&v)[NH]) {
        const uint32_t tt = item >> 1, hh = item & 1u;
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            const uint32_t x = lt + TC_LOAD * (i + NH * hh);
            const uint32_t row = x >> 5, e = x & 31, u = tt * TC_TILE + row;
            v[i] = (tt < ntile && u < nu)
                       ? __ldg(reinterpret_cast<const float4*>(src + static_cast<size_t>(urow[u]) * 128) + e)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    for (uint32_t tt = 0; tt < PF; ++tt) prefetch_tile(tt);
    float4 cur[NH], nxt[NH];
    load_half(0, cur);
    for (uint32_t item = 0; item < 2 * ntile; ++item) {
        const uint32_t t = item >> 1, hh = item & 1u;
        if (hh == 0) prefetch_tile(t + PF);
        load_half(item + 1, nxt);
        const uint32_t b = T & 1u;
        if (hh == 0 && T >= 2) tc::mbar_wait(PASS ? &X.vempty[b] : &X.kempty[b], ((T >> 1) - 1) & 1u);
        const uint32_t base = sbase + (PASS ? TcSmem::V0 + b * TcSmem::VSZ : TcSmem::K0 + b * TcSmem::KSZ);
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            const uint32_t x = lt + TC_LOAD * (i + NH * hh);
            const uint32_t row = x >> 5, e = x & 31;
            const uint32_t off = PASS ? tc::mnmaj_off(4 * e, row, TC_TILE) : tc::kmaj_off(row, 4 * e, TC_TILE);
            store4_split(base + off, base + 16384 + off, cur[i]);
        }
        if (hh == 1) {
            tc::fence_smem_async();
            mbar_arrive(PASS ? &X.vfull[b] : &X.kfull[b]);
            if (ts && lt == 0 && t < 10) ts[t * 8 + 4 + PASS] = gtime();
            ++T;
        }
#pragma unroll
        for (int i = 0; i < NH; ++i) cur[i] = nxt[i];
    }
}

__global__ void __launch_bounds__(TC_THREADS, 1)
attend_tc_kernel(const DecodeProblem* __restrict__ probs, const uint32_t* __restrict__ members,
                 const uint32_t* __restrict__ gmember, const uint32_t* __restrict__ gP,
                 const uint16_t* __restrict__ urow_all, const unsigned long long* __restrict__ umask_all,
                 const uint32_t* __restrict__ ucount, uint32_t ngroups, uint32_t nrange,
                 float* __restrict__ parts, unsigned long long* __restrict__ tprof) {
    // tprof (diagnostics, CSATTN_UNION_PROF): per CTA [16 items][4] globaltimer
    // stamps (item start, prologue done, tiles done, item done), [16] tile counts
    extern __shared__ unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays shared
    TcMisc& X = *reinterpret_cast<TcMisc*>(sm + TcSmem::MISC);
    const uint32_t tid = threadIdx.x;
    const int w = tid >> 5, ln = tid & 31;
    const uint32_t sbase = tc::smem_u32(sm);
    const bool math = (w & 3) < 2 && w < 16;
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&X.kfull[b], TC_LOAD);
            tc::mbar_init(&X.vfull[b], TC_LOAD);
            tc::mbar_init(&X.kempty[b], 1);
            tc::mbar_init(&X.vempty[b], 1);
            tc::mbar_init(&X.sfull[b], 1);
            tc::mbar_init(&X.pfull[b], 256);
        }
        tc::mbar_init(&X.odone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (w == 0) tc::tmem_alloc<512>(&X.tbase);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    // TMEM: S[slot][acc] at 64 (2 slot + acc) | O[acc] at 256 + 128 acc
    const uint32_t tS = X.tbase, tO = X.tbase + 256;
    const uint32_t id_qk = tc::idesc_bf16(128, TC_TILE, false, false);
    const uint32_t id_pv = tc::idesc_bf16(128, 128, false, true);
    uint32_t T = 0;      // tiles processed by this CTA (ring positions)
    uint32_t items = 0;  // items with tiles (odone phases)
    uint32_t it_no = 0;
    unsigned long long* tp = tprof ? tprof + static_cast<size_t>(blockIdx.x) * 160 : nullptr;
    const uint32_t nitems = ngroups * nrange;
    for (uint32_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const uint32_t g = item / nrange, r = item % nrange;
        if (r * UN_RANGE >= gP[g]) continue;  // uniform across the CTA
        const uint32_t nu = __ldg(ucount + item);
        const uint32_t ntile = div_up(nu, TC_TILE);
        const bool rec = tp && tid == 0 && it_no < 16;
        if (rec) tp[it_no * 4] = gtime();
        const uint16_t* urow = urow_all + static_cast<size_t>(item) * UN_RANGE;
        const unsigned long long* umask = umask_all + static_cast<size_t>(item) * UN_RANGE;
        // ---- prologue (all threads): members, Q (pre-scaled, split) -> A operand ----
        if (tid < 64) X.kidx[tid] = gmember[g * UN_GROUP + tid];
        if (tid == 0) {
            const DecodeProblem& Pf = probs[members[gmember[g * UN_GROUP]]];  // member 0 exists
            X.kv[0] = Pf.s->kpre + static_cast<size_t>(r) * UN_RANGE * 128;
            X.kv[1] = Pf.s->vpre + static_cast<size_t>(r) * UN_RANGE * 128;
        }
        {
            const float c = static_cast<float>(1.4426950408889634 / sqrt(128.0));
            for (uint32_t x = tid; x < 64 * 32; x += TC_THREADS) {
                const uint32_t j = x >> 5, e = x & 31;
                const uint32_t kk = gmember[g * UN_GROUP + j];
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (kk != UN_NONE && ntile) {
                    v = __ldg(reinterpret_cast<const float4*>(probs[members[kk]].q) + e);
                    v.x *= c;
                    v.y *= c;
                    v.z *= c;
                    v.w *= c;
                }
                const uint32_t off = tc::kmaj_off(j, 4 * e, 64);
                store4_split(sbase + TcSmem::QHI + off, sbase + TcSmem::QLO + off, v);
            }
        }
        {   // the item's union rows -> shared memory (the loaders' index lookups)
            uint16_t* crow = reinterpret_cast<uint16_t*>(sm + TcSmem::CROW);
            for (uint32_t u = tid; u < nu; u += TC_THREADS) crow[u] = __ldg(urow + u);
        }
        tc::fence_smem_async();
        __syncthreads();
        if (rec) {
            tp[it_no * 4 + 1] = gtime();
            tp[64 + it_no] = ntile;
        }
        if (ntile == 0) {  // no member selected a row here: empty partials
            if (tid < 64 && X.kidx[tid] != UN_NONE) {
                float* pp = parts + (static_cast<size_t>(X.kidx[tid]) * nrange + r) * UN_PART;
                pp[0] = -FLT_MAX;
                pp[1] = 0.0f;
                for (int d = 0; d < 128; ++d) pp[4 + d] = 0.0f;
            }
            __syncthreads();
            ++it_no;
            continue;
        }
        if (loader_slot(w) >= 0) {
            // ================= loaders =================
            const int sl = loader_slot(w);
            const uint32_t lw = static_cast<uint32_t>(sl & 3) * 32 + ln;
            if (sl < 4)
                tc_loader<0>(X, sbase, X.kv[0], reinterpret_cast<const uint16_t*>(sm + TcSmem::CROW), nu, ntile,
                             lw, T, (tp && it_no == 0) ? tp + 80 : nullptr);
            else
                tc_loader<1>(X, sbase, X.kv[1], reinterpret_cast<const uint16_t*>(sm + TcSmem::CROW), nu, ntile,
                             lw, T, (tp && it_no == 0) ? tp + 80 : nullptr);
        } else if (w == 2) {
            // ================= QK issuer: S[slot] = Q . K^T =================
            for (uint32_t t = 0; t < ntile; ++t, ++T) {
                const uint32_t b = T & 1u;
                if (T >= 2) tc::mbar_wait(&X.pfull[b], ((T >> 1) - 1) & 1u);  // S slot read (tile T-2)
                tc::mbar_wait(&X.kfull[b], (T >> 1) & 1u);
                tc::fence_after();
                if (tp && it_no == 0 && t < 10 && ln == 0) tp[80 + t * 8 + 7] = gtime();
                if (ln == 0) {
                    if (b)
                        issue_qk<1>(sbase, tS, id_qk);
                    else
                        issue_qk<0>(sbase, tS, id_qk);
                    tc::commit(&X.sfull[b]);
                    tc::commit(&X.kempty[b]);
                    if (tp && it_no == 0 && t < 10) tp[80 + t * 8 + 0] = gtime();
                }
                __syncwarp();
            }
        } else if (w == 6) {
            // ================= PV issuer: O += P . V =================
            for (uint32_t t = 0; t < ntile; ++t, ++T) {
                const uint32_t b = T & 1u;
                tc::mbar_wait(&X.pfull[b], (T >> 1) & 1u);
                tc::mbar_wait(&X.vfull[b], (T >> 1) & 1u);
                tc::fence_after();
                if (tp && it_no == 0 && t < 10 && ln == 0) tp[80 + t * 8 + 6] = gtime();
                if (ln == 0) {
                    if (b)
                        issue_pv<1>(sbase, tO, id_pv, t == 0);
                    else
                        issue_pv<0>(sbase, tO, id_pv, t == 0);
                    tc::commit(&X.vempty[b]);  // V and P slots free; O stable up to tile t
                    if (t + 1 == ntile) tc::commit(&X.odone);
                    if (tp && it_no == 0 && t < 10) tp[80 + t * 8 + 3] = gtime();
                }
                __syncwarp();
            }
        } else if (math) {
            // ================= softmax (math) =================
            const uint32_t j = (w & 1) * 32 + ln;  // member = TMEM lane
            const uint32_t qt = w >> 2;            // tile rows 16 qt .. 16 qt + 15
            const uint32_t lane_off = (static_cast<uint32_t>(w & 3) * 32u) << 16;
            float m = -FLT_MAX, s = 0.0f;
            for (uint32_t t = 0; t < ntile; ++t, ++T) {
                const uint32_t b = T & 1u;
                // this member's selection bits over its 16 rows (loads issued before the wait)
                uint32_t bits = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const uint32_t u = t * TC_TILE + 16 * qt + i;
                    const unsigned long long mk = u < nu ? __ldg(umask + u) : 0ull;
                    bits |= static_cast<uint32_t>((mk >> j) & 1ull) << i;
                }
                tc::mbar_wait(&X.sfull[b], (T >> 1) & 1u);
                tc::fence_after();
                if (tp && it_no == 0 && t < 10 && tid == 0) tp[80 + t * 8 + 1] = gtime();
                float a[16], a2[16];
                tc::tmem_ld16(tS + b * 128 + 16 * qt + lane_off, a);
                tc::tmem_ld16(tS + b * 128 + 64 + 16 * qt + lane_off, a2);
                float mx = -FLT_MAX;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    a[i] += a2[i];
                    if ((bits >> i) & 1u) mx = fmaxf(mx, a[i]);
                }
                X.hmax[qt][j] = mx;
                math_sync();
                mx = fmaxf(fmaxf(X.hmax[0][j], X.hmax[1][j]), fmaxf(X.hmax[2][j], X.hmax[3][j]));
                // lazy rescale; TMEM accesses are warp-collective (f = 1 elsewhere)
                const bool up = mx > m + UN_TAU;
                float f = 1.0f;
                if (up) {
                    f = ex2(m - mx);  // 0 on the first update (m = -FLT_MAX)
                    s *= f;
                    m = mx;
                }
                if (t > 0 && __any_sync(0xffffffffu, up)) {
                    tc::mbar_wait(&X.vempty[(T - 1) & 1u], ((T - 1) >> 1) & 1u);  // PV(t-1) done
                    tc::fence_after();
                    float o[32];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {  // O accumulators 0,1 x columns 32 qt .. +31
                        const uint32_t col = tO + 128 * q + 32 * qt + lane_off;
                        tc::tmem_ld32(col, o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= f;
                        tc::tmem_st32(col, o);
                    }
                }
                if (T >= 2) tc::mbar_wait(&X.vempty[b], ((T >> 1) - 1) & 1u);  // PV(T-2) read this P slot
                const uint32_t pb = sbase + TcSmem::P0 + b * TcSmem::PSZ;
#pragma unroll
                for (int c = 0; c < 16; c += 8) {
                    float p[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        p[u] = ((bits >> (c + u)) & 1u) ? ex2(a[c + u] - m) : 0.0f;
                        s += p[u];
                    }
                    uint4 hh, ll;
                    split2(p[0], p[1], hh.x, ll.x);
                    split2(p[2], p[3], hh.y, ll.y);
                    split2(p[4], p[5], hh.z, ll.z);
                    split2(p[6], p[7], hh.w, ll.w);
                    const uint32_t off = tc::kmaj_off(j, 16 * qt + c, 64);
                    sts128(pb + off, hh);
                    sts128(pb + 8192 + off, ll);
                }
                tc::fence_smem_async();
                tc::fence_before();
                mbar_arrive(&X.pfull[b]);
                if (tp && it_no == 0 && t < 10 && tid == 0) tp[80 + t * 8 + 2] = gtime();
            }
            // ---- item epilogue: O row of this member (columns 32 qt ..) -> partial ----
            tc::mbar_wait(&X.odone, items & 1u);
            tc::fence_after();
            if (rec) tp[it_no * 4 + 2] = gtime();
            const uint32_t kk = X.kidx[j];
            float* pp = kk != UN_NONE ? parts + (static_cast<size_t>(kk) * nrange + r) * UN_PART : nullptr;
            {
                float o[32], o2[32];
                tc::tmem_ld32(tO + 32 * qt + lane_off, o);
                tc::tmem_ld32(tO + 128 + 32 * qt + lane_off, o2);
                if (pp)
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        *reinterpret_cast<float4*>(pp + 4 + 32 * qt + i) =
                            make_float4(o[i] + o2[i], o[i + 1] + o2[i + 1], o[i + 2] + o2[i + 2], o[i + 3] + o2[i + 3]);
            }
            X.hsum[qt][j] = s;
            math_sync();
            if (pp && qt == 0) {
                const float st = (s + X.hsum[1][j]) + (X.hsum[2][j] + X.hsum[3][j]);
                pp[0] = st > 0.0f ? m : -FLT_MAX;
                pp[1] = st;
            }
        }
        ++items;
        tc::fence_before();
        __syncthreads();  // item done: Q, rows and O may be rewritten
        tc::fence_after();
        if (rec) tp[it_no * 4 + 3] = gtime();
        ++it_no;
    }
    tc::fence_before();
    __syncthreads();
    if (w == 0) tc::tmem_free<512>(X.tbase);
}

// ---- appended rows (>= P) of every member: one warp each ----
__global__ void attend_tail_kernel(const DecodeProblem* __restrict__ probs,
                                   const uint32_t* __restrict__ members, uint32_t n,
                                   float* __restrict__ tails) {
    const uint32_t k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int ln = threadIdx.x & 31;
    if (k >= n) return;
    const DecodeProblem& Pb = probs[members[k]];
    const SessionDev& sd = *Pb.s;
    const uint32_t K = Pb.K, P0 = sd.P;
    const uint32_t first = lower_bound_u32(Pb.sel, K, P0);
    const float4 q = load_q2(Pb.q, ln);
    float m = -FLT_MAX, s = 0.0f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t e = first; e < K; e += 4) {
        const float* kr[4];
        const float* vr[4];
        const int nn = static_cast<int>(min(4u, K - e));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t i = Pb.sel[e + (u < nn ? u : 0)] - P0;
            kr[u] = sd.ktail + static_cast<size_t>(i) * 128;
            vr[u] = sd.vtail + static_cast<size_t>(i) * 128;
        }
        group4(kr, vr, nn, q, m, s, acc, ln);
    }
    float* pp = tails + static_cast<size_t>(k) * UN_PART;
    if (ln == 0) {
        pp[0] = m;
        pp[1] = s;
    }
    reinterpret_cast<float4*>(pp + 4)[ln] = acc;
}

// ---- per member (one CTA of 4 warps): range partials in range order, then the tail ----
__global__ void __launch_bounds__(128)
union_merge_kernel(const DecodeProblem* __restrict__ probs, const uint32_t* __restrict__ members,
                   const uint32_t* __restrict__ mgroup, const uint32_t* __restrict__ gP, uint32_t nrange,
                   const float* __restrict__ parts, const float* __restrict__ tails) {
    __shared__ float wsh[UN_MAX_RANGES + 1];
    __shared__ float red[4];
    __shared__ float4 acc_s[4][32];
    const uint32_t k = blockIdx.x;
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    const DecodeProblem& Pb = probs[members[k]];
    const uint32_t nr = div_up(gP[mgroup[k]], UN_RANGE);
    auto part = [&](uint32_t r) {
        return r < nr ? parts + (static_cast<size_t>(k) * nrange + r) * UN_PART
                      : tails + static_cast<size_t>(k) * UN_PART;
    };
    // global max over non-empty partials
    float gm = -FLT_MAX;
    for (uint32_t r = threadIdx.x; r <= nr; r += 128) {
        const float* pp = part(r);
        if (pp[1] > 0.0f) gm = fmaxf(gm, pp[0]);
    }
    for (int o = 16; o; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if (ln == 0) red[w] = gm;
    __syncthreads();
    gm = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    __syncthreads();
    float gs = 0.0f;
    for (uint32_t r = threadIdx.x; r <= nr; r += 128) {
        const float* pp = part(r);
        const float f = pp[1] > 0.0f ? ex2(pp[0] - gm) : 0.0f;
        wsh[r] = f;
        gs = fmaf(pp[1], f, gs);
    }
    for (int o = 16; o; o >>= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
    if (ln == 0) red[w] = gs;
    __syncthreads();
    gs = (red[0] + red[1]) + (red[2] + red[3]);
    // warp w accumulates partials r = w, w + 4, ... (fixed order), lanes own 4 dims
    float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t r = w; r <= nr; r += 4) {
        const float f = wsh[r];  // 0 for empty partials (their acc is 0)
        const float4 a = reinterpret_cast<const float4*>(part(r) + 4)[ln];
        o4.x = fmaf(f, a.x, o4.x);
        o4.y = fmaf(f, a.y, o4.y);
        o4.z = fmaf(f, a.z, o4.z);
        o4.w = fmaf(f, a.w, o4.w);
    }
    acc_s[w][ln] = o4;
    __syncthreads();
    if (w == 0 && Pb.out) {
        const float4 x0 = acc_s[0][ln], x1 = acc_s[1][ln], x2 = acc_s[2][ln], x3 = acc_s[3][ln];
        const float inv = 1.0f / gs;
        reinterpret_cast<float4*>(Pb.out)[ln] =
            make_float4(((x0.x + x1.x) + (x2.x + x3.x)) * inv, ((x0.y + x1.y) + (x2.y + x3.y)) * inv,
                        ((x0.z + x1.z) + (x2.z + x3.z)) * inv, ((x0.w + x1.w) + (x2.w + x3.w)) * inv);
    }
}

cudaError_t launch_attend_union(const DecodeProblem* probs, uint32_t ngroups, const uint32_t* gP,
                                const uint32_t* gmember, const uint32_t* members,
                                const uint32_t* mgroup, uint32_t nmembers, uint32_t nrange,
                                uint16_t* urow, unsigned long long* umask, uint32_t* ucount,
                                float* parts, float* tails, int num_sms, unsigned long long* tprof,
                                cudaStream_t st) {
    if (nrange > UN_MAX_RANGES) return cudaErrorInvalidValue;
    static bool attr = false;
    const int smem = static_cast<int>(TcSmem::BYTES + 1024);
    if (!attr) {
        const cudaError_t e =
            cudaFuncSetAttribute(attend_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const uint32_t items = ngroups * nrange;
    union_build_kernel<<<items, UB_THREADS, 0, st>>>(probs, members, gmember, gP, nrange, urow, umask, ucount);
    // CSATTN_UNION_CTAS caps the persistent grid (tests: many items per CTA)
    const char* cenv = std::getenv("CSATTN_UNION_CTAS");
    const uint32_t cap = cenv ? static_cast<uint32_t>(std::atoi(cenv)) : 0u;
    uint32_t grid = items < static_cast<uint32_t>(num_sms) ? items : static_cast<uint32_t>(num_sms);
    if (cap && cap < grid) grid = cap;
    attend_tc_kernel<<<grid, TC_THREADS, smem, st>>>(probs, members, gmember, gP, urow, umask, ucount, ngroups,
                                                     nrange, parts, tprof);
    attend_tail_kernel<<<div_up(nmembers, 8), 256, 0, st>>>(probs, members, nmembers, tails);
    union_merge_kernel<<<nmembers, 128, 0, st>>>(probs, members, mgroup, gP, nrange, parts, tails);
    return cudaGetLastError();
}

}  // namespace csa
