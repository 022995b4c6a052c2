// attend_union.cu — sparse attention for problems that share one prefill
// (masked dense_attention, core.cpp:118-169), on sm_100a.
//
// The batch-decode case (config c3: 16 sequences forked from one prefill, GQA
// groups of 4 -> 64 (sequence, head) problems per KV head) selects each prefill
// row ~6x on average. The per-problem path (attend.cu) gathers a row once per
// problem that selected it; here a group of <= 64 problems ("members") on one
// prefill is processed by prefill ROW RANGE, so a row crosses HBM/L2 once per
// group:
//   union_bounds_kernel  per member: where each row range starts in its
//                        (ascending) selected list, and where its appended
//                        rows (index >= P) start
//   attend_range_kernel  per (group, range of UN_RANGE prefill rows): the
//                        members' selected rows in the range are marked in a
//                        shared-memory bitmask (bit b = member b), the union is
//                        compacted and streamed through a cp.async double
//                        buffer; warp w owns members 8w..8w+7 (q and the
//                        online-softmax state in registers) and runs each
//                        member over ITS rows of the batch in groups of four
//                        -> partial (max, sum, acc[128]) per (member, range)
//   attend_tail_kernel   per member: its appended rows (private to its
//                        session), one warp -> a partial
//   union_merge_kernel   per member: log-sum-exp of its range partials in
//                        range order, then the tail -> output
// Every problem attends exactly its own selected rows in a fixed order, so the
// result is deterministic and independent of how problems are grouped.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include <cuda_bf16.h>

#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace csa {

constexpr uint32_t UN_PART = UN_PART_WORDS;  // max, sum, 2 pad, acc[128]
constexpr uint32_t UN_NONE = 0xffffffffu;

// ---- per member: range starts in its selected list ----
// bnd[k][r] = lower_bound(sel, r * UN_RANGE) for r < nr = ceil(P / UN_RANGE),
// bnd[k][nr] = lower_bound(sel, P): the first appended row.
__global__ void __launch_bounds__(256)
union_bounds_kernel(const DecodeProblem* __restrict__ probs, const uint32_t* __restrict__ members,
                    const uint32_t* __restrict__ mgroup, const uint32_t* __restrict__ gP,
                    uint32_t nrange, uint32_t* __restrict__ bnd) {
    const uint32_t k = blockIdx.x;
    const DecodeProblem& Pb = probs[members[k]];
    const uint32_t* sel = Pb.sel;
    const uint32_t K = Pb.K, P0 = gP[mgroup[k]];
    const uint32_t nr = div_up(P0, UN_RANGE);
    uint32_t* b = bnd + static_cast<size_t>(k) * (nrange + 1);
    // entry i (i == K: +infinity) starts every boundary e with sel[i-1] < e <= sel[i]
    for (uint32_t i = threadIdx.x; i <= K; i += blockDim.x) {
        const long long prev = i ? static_cast<long long>(sel[i - 1]) : -1ll;
        const long long x = i < K ? static_cast<long long>(sel[i]) : (1ll << 40);
        for (uint32_t r = prev < 0 ? 0u : min(nr, static_cast<uint32_t>(prev / UN_RANGE) + 1u); r <= nr;
             ++r) {
            const long long e = r < nr ? static_cast<long long>(r) * UN_RANGE : P0;
            if (e > x) break;
            if (e > prev) b[r] = i;
        }
    }
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
// Work item = (group g, prefill range r of UN_RANGE rows); its union rows are
// processed in tiles of 64 (FlashAttention-4 orientation, member = TMEM lane):
//   S[member][row] = Q . K_tile^T   (tcgen05 M = 128: 64 members + padding, N = 64)
//   P[member][row] = mask ? 2^(S - m_member) : 0     (thread = member)
//   O[member][dim] += P . V_tile    (tcgen05 M = 128, N = 128)
// fp32 operands are split into bf16 hi + lo, each product takes three terms
// (hi.hi + lo.hi + hi.lo): ~2^-16 relative, fp32-grade. Q is pre-scaled by
// log2(e)/sqrt(d) (base-2 logits). A member's running max is raised only when
// a tile exceeds it by more than UN_TAU (lazy rescale of its O row), so
// P <= 2^UN_TAU. Lanes 64-127 of every MMA read padding (their rows are never
// used). K, V, P and S are double-buffered; mbarrier rings connect the roles:
//   warps 0-1   math: softmax of member lane (tid), epilogue
//   warp 2      MMA issuer (one thread)
//   warps 3-10  K loaders, warps 11-18 V loaders (global -> regs -> bf16 hi/lo
//               -> swizzled smem), one tile ahead in registers + L2 prefetch
constexpr int TC_MATH = 64, TC_LOAD = 256;
constexpr int TC_THREADS = TC_MATH + 32 + 2 * TC_LOAD;  // 608
constexpr int TC_KW0 = (TC_MATH + 32) / 32;             // first K-loader warp
constexpr uint32_t TC_TILE = 64;
constexpr float UN_TAU = 8.0f;
struct TcSmem {  // 1024-byte aligned operand buffers
    // K tile (B of QK, K-major, 64 rows x 128 dims): hi | lo, 16 KB each; x2
    static constexpr uint32_t K0 = 0, KSZ = 32768;
    // V tile (B of PV, MN-major, 64 rows x 128 dims): hi | lo; x2
    static constexpr uint32_t V0 = 65536, VSZ = 32768;
    // Q (A of QK, K-major, 64 member rows x 128 dims): hi | lo
    static constexpr uint32_t QHI = 131072, QLO = 147456;
    // P (A of PV, K-major, 64 member rows x 64 tile rows): hi | lo, 8 KB each; x2
    static constexpr uint32_t P0 = 163840, PSZ = 16384;
    static constexpr uint32_t MASK = 196608;               // u64[UN_RANGE]: marks, then compacted
    static constexpr uint32_t CROW = MASK + UN_RANGE * 8;  // u16[UN_RANGE]
    static constexpr uint32_t MISC = CROW + UN_RANGE * 2;
    static constexpr uint32_t BYTES = MISC + 1024;
};
static_assert(TcSmem::BYTES + 1024 <= 232448, "shared memory budget");
struct TcMisc {
    uint64_t kfull[2], vfull[2], kempty[2], vempty[2], sfull[2], pfull[2], odone;
    const float* kv[2];
    uint32_t wcount[TC_THREADS / 32];
    uint32_t nu, tbase;
    uint32_t kidx[64];
};
static_assert(sizeof(TcMisc) <= 1024, "misc");

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
__device__ __forceinline__ void tc_loader(TcMisc& X, uint32_t sbase, const float* src,
                                          const uint16_t* crow, uint32_t nu, uint32_t ntile,
                                          uint32_t lt, uint32_t& T, unsigned long long* tstamp) {
    constexpr int NV = TC_TILE * 32 / TC_LOAD;  // float4 per thread per tile (8)
    constexpr uint32_t PF = 4;                  // L2 prefetch distance (tiles)
    auto prefetch_tile = [&](uint32_t tt) {
        if (lt < TC_TILE && tt < ntile) {
            const uint32_t u = tt * TC_TILE + lt;
            if (u < nu) prefetch_l2(src + static_cast<size_t>(crow[u]) * 128, 512);
        }
    };
    auto load = [&](uint32_t tt, float4 (&v)[NV]) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const uint32_t x = lt + TC_LOAD * i;
            const uint32_t row = x >> 5, e = x & 31, u = tt * TC_TILE + row;
            v[i] = (tt < ntile && u < nu)
                       ? __ldg(reinterpret_cast<const float4*>(src + static_cast<size_t>(crow[u]) * 128) + e)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    for (uint32_t tt = 0; tt < PF; ++tt) prefetch_tile(tt);
    for (uint32_t t = 0; t < ntile; ++t, ++T) {
        prefetch_tile(t + PF);
        float4 cur[NV];
        load(t, cur);
        const uint32_t b = T & 1u;
        if (T >= 2) tc::mbar_wait(PASS ? &X.vempty[b] : &X.kempty[b], ((T >> 1) - 1) & 1u);
        const uint32_t base = sbase + (PASS ? TcSmem::V0 + b * TcSmem::VSZ : TcSmem::K0 + b * TcSmem::KSZ);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const uint32_t x = lt + TC_LOAD * i;
            const uint32_t row = x >> 5, e = x & 31;
            const uint32_t off = PASS ? tc::mnmaj_off(4 * e, row, TC_TILE) : tc::kmaj_off(row, 4 * e, TC_TILE);
            store4_split(base + off, base + 16384 + off, cur[i]);
        }
        tc::fence_smem_async();
        mbar_arrive(PASS ? &X.vfull[b] : &X.kfull[b]);
        if (tstamp && lt == 0 && t < 10) tstamp[t * 8 + 4 + PASS] = gtime();
    }
}

__global__ void __launch_bounds__(TC_THREADS, 1)
attend_tc_kernel(const DecodeProblem* __restrict__ probs, const uint32_t* __restrict__ members,
                 const uint32_t* __restrict__ gmember, const uint32_t* __restrict__ gP,
                 const uint32_t* __restrict__ bnd, uint32_t ngroups, uint32_t nrange,
                 float* __restrict__ parts, unsigned long long* __restrict__ tprof) {
    // tprof (diagnostics, CSATTN_UNION_PROF): per CTA [16 items][4] globaltimer
    // stamps (item start, prologue done, tiles done, item done), [16] tile counts
    extern __shared__ unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays shared
    TcMisc& X = *reinterpret_cast<TcMisc*>(sm + TcSmem::MISC);
    unsigned long long* mask = reinterpret_cast<unsigned long long*>(sm + TcSmem::MASK);
    uint16_t* crow = reinterpret_cast<uint16_t*>(sm + TcSmem::CROW);
    const uint32_t tid = threadIdx.x;
    const int w = tid >> 5, ln = tid & 31;
    const uint32_t sbase = tc::smem_u32(sm);
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&X.kfull[b], TC_LOAD);
            tc::mbar_init(&X.vfull[b], TC_LOAD);
            tc::mbar_init(&X.kempty[b], 1);
            tc::mbar_init(&X.vempty[b], 1);
            tc::mbar_init(&X.sfull[b], 1);
            tc::mbar_init(&X.pfull[b], TC_MATH);
        }
        tc::mbar_init(&X.odone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (w == 0) tc::tmem_alloc<256>(&X.tbase);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tS = X.tbase, tO = X.tbase + 128;  // S[2] (64 cols each) | O (128 cols)
    const uint32_t id_qk = tc::idesc_bf16(128, TC_TILE, false, false);
    const uint32_t id_pv = tc::idesc_bf16(128, 128, false, true);
    uint32_t T = 0;      // tiles processed by this CTA (ring positions)
    uint32_t items = 0;  // items with tiles (odone phases)
    uint32_t it_no = 0;
    unsigned long long* tp = tprof ? tprof + static_cast<size_t>(blockIdx.x) * 160 : nullptr;
    const uint32_t nitems = ngroups * nrange;
    for (uint32_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const uint32_t g = item / nrange, r = item % nrange;
        const uint32_t P0 = gP[g];
        const uint32_t r0 = r * UN_RANGE;
        if (r0 >= P0) continue;  // uniform across the CTA
        const bool rec = tp && tid == 0 && it_no < 16;
        if (rec) tp[it_no * 4] = gtime();
        // ---- item prologue (all threads): members, marks, compaction, Q ----
        for (uint32_t i = tid; i < UN_RANGE; i += TC_THREADS) mask[i] = 0ull;
        if (tid < 64) X.kidx[tid] = gmember[g * UN_GROUP + tid];
        if (tid == 0) {
            const DecodeProblem& Pf = probs[members[gmember[g * UN_GROUP]]];  // member 0 exists
            X.kv[0] = Pf.s->kpre;
            X.kv[1] = Pf.s->vpre;
        }
        __syncthreads();
        if (w < 8) {  // warp w marks members 8w..8w+7 (32-bit halves: native shared atomics)
            const uint32_t* selp = nullptr;
            uint32_t lo = 0, hi = 0;
            if (ln < 8) {
                const uint32_t kk = X.kidx[8 * w + ln];
                if (kk != UN_NONE) {
                    const uint32_t* b = bnd + static_cast<size_t>(kk) * (nrange + 1);
                    lo = b[r];
                    hi = b[r + 1];
                    selp = probs[members[kk]].sel;
                }
            }
            uint32_t* m32 = reinterpret_cast<uint32_t*>(mask) + (w >= 4 ? 1 : 0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t* sp = reinterpret_cast<const uint32_t*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(selp), j));
                const uint32_t elo = __shfl_sync(0xffffffffu, lo, j), ehi = __shfl_sync(0xffffffffu, hi, j);
                const uint32_t bit = 1u << ((8 * w + j) & 31);
                for (uint32_t e = elo + ln; e < ehi; e += 32) atomicOr(m32 + 2 * (__ldg(sp + e) - r0), bit);
            }
        }
        {   // Q (pre-scaled by log2(e)/sqrt(d), split) -> A operand, K-major, 64 rows
            const float c = static_cast<float>(1.4426950408889634 / sqrt(128.0));
            for (uint32_t x = tid; x < 64 * 32; x += TC_THREADS) {
                const uint32_t j = x >> 5, e = x & 31;
                const uint32_t kk = X.kidx[j];
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (kk != UN_NONE) {
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
        __syncthreads();
        {   // in-place compaction (thread order = row order)
            constexpr int PER = (UN_RANGE + TC_THREADS - 1) / TC_THREADS;
            unsigned long long v[PER];
            uint32_t n = 0;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                v[i] = tid * PER + i < UN_RANGE ? mask[tid * PER + i] : 0ull;
                n += v[i] != 0ull;
            }
            uint32_t inc = n;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (ln >= o) inc += y;
            }
            if (ln == 31) X.wcount[w] = inc;
            __syncthreads();
            uint32_t pre = 0, tot = 0;
#pragma unroll
            for (int i = 0; i < TC_THREADS / 32; ++i) {
                pre += i < w ? X.wcount[i] : 0u;
                tot += X.wcount[i];
            }
            uint32_t pos = pre + inc - n;
#pragma unroll
            for (int i = 0; i < PER; ++i)
                if (v[i]) {
                    crow[pos] = static_cast<uint16_t>(tid * PER + i);
                    mask[pos] = v[i];
                    ++pos;
                }
            if (tid == 0) X.nu = tot;
            tc::fence_smem_async();  // Q operand
            __syncthreads();
        }
        const uint32_t nu = X.nu;
        const uint32_t ntile = div_up(nu, TC_TILE);
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
        const float* kpre = X.kv[0] + static_cast<size_t>(r0) * 128;
        const float* vpre = X.kv[1] + static_cast<size_t>(r0) * 128;
        if (w >= TC_KW0) {
            // ================= loaders =================
            const uint32_t lw = tid - (TC_MATH + 32);
            if (lw < TC_LOAD)
                tc_loader<0>(X, sbase, kpre, crow, nu, ntile, lw, T, (tp && it_no == 0) ? tp + 80 : nullptr);
            else
                tc_loader<1>(X, sbase, vpre, crow, nu, ntile, lw - TC_LOAD, T, (tp && it_no == 0) ? tp + 80 : nullptr);
        } else if (w == 2) {
            // ================= MMA issuer =================
            const uint32_t T0 = T;
            auto qk = [&](uint32_t t) {  // S[slot] = Q . K^T
                const uint32_t TT = T0 + t, b = TT & 1u;
                tc::mbar_wait(&X.kfull[b], (TT >> 1) & 1u);
                tc::fence_after();
                if (ln == 0) {
                    const uint32_t kb = sbase + TcSmem::K0 + b * TcSmem::KSZ;
#pragma unroll
                    for (int s = 0; s < 8; ++s) {
                        const uint32_t o = (s >> 2) * 64 * 128 + (s & 3) * 32;
                        const uint64_t qhi = tc::desc_sw128(sbase + TcSmem::QHI + o, 16, 1024);
                        const uint64_t qlo = tc::desc_sw128(sbase + TcSmem::QLO + o, 16, 1024);
                        const uint64_t khi = tc::desc_sw128(kb + o, 16, 1024);
                        const uint64_t klo = tc::desc_sw128(kb + 16384 + o, 16, 1024);
                        tc::mma_bf16(tS + b * 64, qhi, khi, id_qk, s > 0);
                        tc::mma_bf16(tS + b * 64, qlo, khi, id_qk, 1);
                        tc::mma_bf16(tS + b * 64, qhi, klo, id_qk, 1);
                    }
                    tc::commit(&X.sfull[b]);
                    tc::commit(&X.kempty[b]);
                    if (tp && it_no == 0 && t < 10) tp[80 + t * 8 + 0] = gtime();
                }
                __syncwarp();
            };
            qk(0);
            if (ntile > 1) qk(1);
            for (uint32_t t = 0; t < ntile; ++t) {
                const uint32_t TT = T0 + t, b = TT & 1u;
                tc::mbar_wait(&X.pfull[b], (TT >> 1) & 1u);
                tc::mbar_wait(&X.vfull[b], (TT >> 1) & 1u);
                tc::fence_after();
                if (ln == 0) {  // O += P . V
                    const uint32_t vb = sbase + TcSmem::V0 + b * TcSmem::VSZ;
                    const uint32_t pb = sbase + TcSmem::P0 + b * TcSmem::PSZ;
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        const uint64_t phi = tc::desc_sw128(pb + s * 32, 16, 1024);
                        const uint64_t plo = tc::desc_sw128(pb + 8192 + s * 32, 16, 1024);
                        const uint64_t vhi = tc::desc_sw128(vb + s * 2048, 8192, 1024);
                        const uint64_t vlo = tc::desc_sw128(vb + 16384 + s * 2048, 8192, 1024);
                        tc::mma_bf16(tO, phi, vhi, id_pv, (t > 0 || s > 0) ? 1u : 0u);
                        tc::mma_bf16(tO, plo, vhi, id_pv, 1);
                        tc::mma_bf16(tO, phi, vlo, id_pv, 1);
                    }
                    tc::commit(&X.vempty[b]);  // V and P slots free; O stable up to tile t
                    if (tp && it_no == 0 && t < 10) tp[80 + t * 8 + 3] = gtime();
                    if (t + 1 == ntile) tc::commit(&X.odone);
                }
                __syncwarp();
                if (t + 2 < ntile) qk(t + 2);
            }
            T += ntile;
        } else {
            // ================= math (thread = member = TMEM lane) =================
            const uint32_t j = tid;  // member
            const uint32_t lane_off = (static_cast<uint32_t>(w) * 32u) << 16;
            float m = -FLT_MAX, s = 0.0f;
            for (uint32_t t = 0; t < ntile; ++t, ++T) {
                const uint32_t b = T & 1u, u0 = t * TC_TILE;
                // selection bits of this member over the tile's rows
                uint32_t bits0 = 0, bits1 = 0;
#pragma unroll 8
                for (int rr = 0; rr < 32; ++rr) {
                    const uint32_t u = u0 + rr, u2 = u0 + 32 + rr;
                    bits0 |= (u < nu ? static_cast<uint32_t>(mask[u] >> j) & 1u : 0u) << rr;
                    bits1 |= (u2 < nu ? static_cast<uint32_t>(mask[u2] >> j) & 1u : 0u) << rr;
                }
                tc::mbar_wait(&X.sfull[b], (T >> 1) & 1u);
                tc::fence_after();
                if (tp && it_no == 0 && t < 10 && tid == 0) tp[80 + t * 8 + 1] = gtime();
                float mx = -FLT_MAX;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float a[32];
                    tc::tmem_ld32(tS + b * 64 + 32 * h + lane_off, a);
                    const uint32_t bits = h ? bits1 : bits0;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if ((bits >> i) & 1u) mx = fmaxf(mx, a[i]);
                }
                // lazy rescale of this member's O row and sum; the TMEM accesses
                // are warp-collective, so a warp rescales together (f = 1 elsewhere)
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
                    for (int c = 0; c < 128; c += 32) {
                        tc::tmem_ld32(tO + c + lane_off, o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= f;
                        tc::tmem_st32(tO + c + lane_off, o);
                    }
                }
                // P row: 64 tile rows, 8 per 16-byte store (hi and lo)
                if (T >= 2) tc::mbar_wait(&X.vempty[b], ((T >> 1) - 1) & 1u);  // PV(T-2) read this P slot
                const uint32_t pb = sbase + TcSmem::P0 + b * TcSmem::PSZ;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float a[32];
                    tc::tmem_ld32(tS + b * 64 + 32 * h + lane_off, a);
                    const uint32_t bits = h ? bits1 : bits0;
#pragma unroll
                    for (int c = 0; c < 32; c += 8) {
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
                        const uint32_t off = tc::kmaj_off(j, 32 * h + c, 64);
                        sts128(pb + off, hh);
                        sts128(pb + 8192 + off, ll);
                    }
                }
                tc::fence_smem_async();
                tc::fence_before();
                mbar_arrive(&X.pfull[b]);
                if (tp && it_no == 0 && t < 10 && tid == 0) tp[80 + t * 8 + 2] = gtime();
            }
            // ---- item epilogue: O row of this member -> partial ----
            tc::mbar_wait(&X.odone, items & 1u);
            tc::fence_after();
            if (rec) tp[it_no * 4 + 2] = gtime();
            const uint32_t kk = X.kidx[j];
            float* pp = kk != UN_NONE ? parts + (static_cast<size_t>(kk) * nrange + r) * UN_PART : nullptr;
            float o[32];
#pragma unroll
            for (int c = 0; c < 128; c += 32) {
                tc::tmem_ld32(tO + c + lane_off, o);
                if (pp)
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        *reinterpret_cast<float4*>(pp + 4 + c + i) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
            }
            if (pp) {
                pp[0] = s > 0.0f ? m : -FLT_MAX;
                pp[1] = s;
            }
        }
        ++items;
        tc::fence_before();
        __syncthreads();  // item done: marks, rows, Q and O may be rewritten
        tc::fence_after();
        if (rec) tp[it_no * 4 + 3] = gtime();
        ++it_no;
    }
    tc::fence_before();
    __syncthreads();
    if (w == 0) tc::tmem_free<256>(X.tbase);
}

// ---- appended rows (>= P) of every member: one warp each ----
__global__ void attend_tail_kernel(const DecodeProblem* __restrict__ probs,
                                   const uint32_t* __restrict__ members, uint32_t n,
                                   const uint32_t* __restrict__ bnd, uint32_t nrange,
                                   float* __restrict__ tails) {
    const uint32_t k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int ln = threadIdx.x & 31;
    if (k >= n) return;
    const DecodeProblem& Pb = probs[members[k]];
    const SessionDev& sd = *Pb.s;
    const uint32_t K = Pb.K, P0 = sd.P;
    const uint32_t first = bnd[static_cast<size_t>(k) * (nrange + 1) + div_up(P0, UN_RANGE)];
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

// ---- per member (one warp): range partials in range order, then the tail ----
__global__ void __launch_bounds__(128)
union_merge_kernel(const DecodeProblem* __restrict__ probs, const uint32_t* __restrict__ members,
                   const uint32_t* __restrict__ mgroup, const uint32_t* __restrict__ gP, uint32_t n,
                   uint32_t nrange, const float* __restrict__ parts, const float* __restrict__ tails) {
    __shared__ float wsh[4][UN_MAX_RANGES + 1];
    const uint32_t k = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (k >= n) return;
    const DecodeProblem& Pb = probs[members[k]];
    const uint32_t nr = div_up(gP[mgroup[k]], UN_RANGE);
    auto part = [&](uint32_t r) {
        return r < nr ? parts + (static_cast<size_t>(k) * nrange + r) * UN_PART
                      : tails + static_cast<size_t>(k) * UN_PART;
    };
    float gm = -FLT_MAX;
    for (uint32_t r = ln; r <= nr; r += 32) {
        const float* pp = part(r);
        if (pp[1] > 0.0f) gm = fmaxf(gm, pp[0]);
    }
    for (int o = 16; o; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    float gs = 0.0f;
    for (uint32_t r = ln; r <= nr; r += 32) {
        const float* pp = part(r);
        const float f = pp[1] > 0.0f ? ex2(pp[0] - gm) : 0.0f;
        wsh[w][r] = f;
        gs = fmaf(pp[1], f, gs);
    }
    for (int o = 16; o; o >>= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
    __syncwarp();
    float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t r = 0;
    for (; r + 4 <= nr + 1; r += 4) {  // 4 partials in flight
        float4 a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = reinterpret_cast<const float4*>(part(r + u) + 4)[ln];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float f = wsh[w][r + u];  // 0 for empty partials (their acc is 0)
            o4.x = fmaf(f, a[u].x, o4.x);
            o4.y = fmaf(f, a[u].y, o4.y);
            o4.z = fmaf(f, a[u].z, o4.z);
            o4.w = fmaf(f, a[u].w, o4.w);
        }
    }
    for (; r <= nr; ++r) {
        const float f = wsh[w][r];
        const float4 a = reinterpret_cast<const float4*>(part(r) + 4)[ln];
        o4.x = fmaf(f, a.x, o4.x);
        o4.y = fmaf(f, a.y, o4.y);
        o4.z = fmaf(f, a.z, o4.z);
        o4.w = fmaf(f, a.w, o4.w);
    }
    const float inv = 1.0f / gs;
    if (Pb.out)
        reinterpret_cast<float4*>(Pb.out)[ln] =
            make_float4(o4.x * inv, o4.y * inv, o4.z * inv, o4.w * inv);
}

cudaError_t launch_attend_union(const DecodeProblem* probs, uint32_t ngroups, const uint32_t* gP,
                                const uint32_t* gmember, const uint32_t* members,
                                const uint32_t* mgroup, uint32_t nmembers, uint32_t nrange,
                                uint32_t* bnd, float* parts, float* tails, int num_sms,
                                unsigned long long* tprof, cudaStream_t st) {
    if (nrange > UN_MAX_RANGES) return cudaErrorInvalidValue;
    static bool attr = false;
    const int smem = static_cast<int>(TcSmem::BYTES + 1024);
    if (!attr) {
        const cudaError_t e =
            cudaFuncSetAttribute(attend_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    union_bounds_kernel<<<nmembers, 256, 0, st>>>(probs, members, mgroup, gP, nrange, bnd);
    const uint32_t items = ngroups * nrange;
    // CSATTN_UNION_CTAS caps the persistent grid (tests: many items per CTA)
    const char* cenv = std::getenv("CSATTN_UNION_CTAS");
    const uint32_t cap = cenv ? static_cast<uint32_t>(std::atoi(cenv)) : 0u;
    uint32_t grid = items < static_cast<uint32_t>(num_sms) ? items : static_cast<uint32_t>(num_sms);
    if (cap && cap < grid) grid = cap;
    attend_tc_kernel<<<grid, TC_THREADS, smem, st>>>(
        probs, members, gmember, gP, bnd, ngroups, nrange, parts, tprof);
    attend_tail_kernel<<<div_up(nmembers, 8), 256, 0, st>>>(probs, members, nmembers, bnd, nrange,
                                                            tails);
    union_merge_kernel<<<div_up(nmembers, 4), 128, 0, st>>>(probs, members, mgroup, gP, nmembers,
                                                            nrange, parts, tails);
    return cudaGetLastError();
}

}  // namespace csa
