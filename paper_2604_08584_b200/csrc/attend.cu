// attend.cu — CSAttention decode, part 2: sparse attention over the selected
// rows (masked dense_attention, core.cpp:118-169) on sm_100a.
//
// Split-K flash decoding: the K selected rows of every problem are cut into
// ATT_ROWS-row chunks and every chunk is one 128-thread CTA, so a layer step
// (512 problems x ~52 chunks at 128K) is a grid of ~27K independent CTAs with
// high memory-level parallelism. Each warp streams 32 rows: one coalesced load
// of its 32 row indices, then ATT_U rows at a time with one float4 per lane of
// the K row and of the V row in flight (a 512-byte row = one warp-wide 128-bit
// load), online softmax in fp32. The CTA reduces its 4 warps into one partial
// (max, sum, acc[d]); the last CTA to finish a problem (device-scope counter)
// merges the partials in chunk order — a deterministic log-sum-exp merge —
// writes the output, the softmax weights (if requested: logits are parked in
// the weights buffer and normalized in place) and resets the counter.
#include <cuda_runtime.h>

#include <type_traits>

#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace csa {

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int ATT_THREADS = 128;
constexpr int ATT_WARPS = ATT_THREADS / 32;
constexpr int ATT_U = 4;

__device__ __forceinline__ float wsum(float v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Each lane holds NC x VEC elements of the head dim: element (cc, v) is
// cc*32*VEC + lane*VEC + v (VEC = 4 when d % 4 == 0: 128-bit loads).
template <int VEC>
__device__ __forceinline__ void ld_vec(float (&x)[VEC], const float* p) {
    if constexpr (VEC == 4) {
        const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
        x[0] = t.x;
        x[1] = t.y;
        x[2] = t.z;
        x[3] = t.w;
    } else {
        x[0] = __ldcs(p);
    }
}

template <int NC, int VEC>
__global__ void __launch_bounds__(ATT_THREADS)
attend_kernel(const DecodeProblem* __restrict__ probs, const uint32_t* __restrict__ chunk_prob,
              const uint32_t* __restrict__ chunk_base, float* __restrict__ part,
              uint32_t* __restrict__ counters, uint32_t rows) {
    __shared__ float wm[ATT_WARPS], ws[ATT_WARPS];
    __shared__ float wacc[ATT_WARPS][NC * 32 * VEC];
    __shared__ uint32_t is_last;
    const uint32_t c = blockIdx.x;
    // chunk entry: problem | chunk index << 20 (chunks may come in any order)
    const uint32_t cpk = chunk_prob[c];
    const uint32_t p = cpk & 0xfffffu;
    const DecodeProblem& P = probs[p];
    const SessionDev& sd = *P.s;
    const uint32_t d = sd.d, K = P.K, P0 = sd.P;
    const uint32_t j = cpk >> 20;
    const uint32_t nch = chunk_base[p + 1] - chunk_base[p];
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    const uint32_t rw = j * rows + w * (rows / ATT_WARPS);  // this warp's first row
    const uint32_t nrw = rw < K ? min(rows / ATT_WARPS, K - rw) : 0u;
    const bool want_w = (P.mode & MODE_WEIGHTS) && P.weights;

    float q[NC][VEC];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            const uint32_t e = cc * 32 * VEC + ln * VEC + v;
            q[cc][v] = e < d ? P.q[e] : 0.0f;
        }
    const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(d)));

    float m = -FLT_MAX, s = 0.0f;
    float acc[NC][VEC];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[cc][v] = 0.0f;

    for (uint32_t b0 = 0; b0 < nrw; b0 += 32) {  // 32-row index batches
    const uint32_t r0 = rw + b0;
    const uint32_t nr = min(32u, nrw - b0);
    const uint32_t myidx = ln < nr ? __ldg(P.sel + r0 + ln) : 0u;
    for (uint32_t i0 = 0; i0 < nr; i0 += ATT_U) {
        float kv[ATT_U][NC][VEC], vv[ATT_U][NC][VEC];
#pragma unroll
        for (int u = 0; u < ATT_U; ++u) {
            const uint32_t i = __shfl_sync(0xffffffffu, myidx, (i0 + u) & 31);
            const bool ok = i0 + u < nr;
            const float* kr = i < P0 ? sd.kpre + static_cast<size_t>(i) * d
                                     : sd.ktail + static_cast<size_t>(i - P0) * d;
            const float* vr = i < P0 ? sd.vpre + static_cast<size_t>(i) * d
                                     : sd.vtail + static_cast<size_t>(i - P0) * d;
#pragma unroll
            for (int cc = 0; cc < NC; ++cc) {
                const uint32_t e = cc * 32 * VEC + ln * VEC;
                if (ok && e < d) {
                    ld_vec<VEC>(kv[u][cc], kr + e);
                    ld_vec<VEC>(vv[u][cc], vr + e);
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) kv[u][cc][v] = vv[u][cc][v] = 0.0f;
                }
            }
        }
        float lg[ATT_U];
#pragma unroll
        for (int u = 0; u < ATT_U; ++u) {
            float dp = 0.0f;
#pragma unroll
            for (int cc = 0; cc < NC; ++cc)
#pragma unroll
                for (int v = 0; v < VEC; ++v) dp = fmaf(q[cc][v], kv[u][cc][v], dp);
            lg[u] = wsum(dp) * scale;
        }
        float mn = m;
#pragma unroll
        for (int u = 0; u < ATT_U; ++u)
            if (i0 + u < nr) mn = fmaxf(mn, lg[u]);
        const float f = expf(m - mn);
        s *= f;
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[cc][v] *= f;
#pragma unroll
        for (int u = 0; u < ATT_U; ++u) {
            if (i0 + u >= nr) continue;
            const float pu = expf(lg[u] - mn);
            s += pu;
#pragma unroll
            for (int cc = 0; cc < NC; ++cc)
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[cc][v] = fmaf(pu, vv[u][cc][v], acc[cc][v]);
            if (want_w && ln == 0) P.weights[r0 + i0 + u] = lg[u];  // logit, normalized later
        }
        m = mn;
    }
    }
    // ---- CTA partial ----
    if (ln == 0) {
        wm[w] = nrw ? m : -FLT_MAX;
        ws[w] = nrw ? s : 0.0f;
    }
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int v = 0; v < VEC; ++v) wacc[w][cc * 32 * VEC + ln * VEC + v] = acc[cc][v];
    __syncthreads();
    float M = -FLT_MAX;
#pragma unroll
    for (int i = 0; i < ATT_WARPS; ++i) M = fmaxf(M, wm[i]);
    float* pp = part + static_cast<size_t>(chunk_base[p] + j) * (d + 2);
    if (threadIdx.x == 0) {
        float S = 0.0f;
        for (int i = 0; i < ATT_WARPS; ++i)
            if (ws[i] > 0.0f) S += ws[i] * expf(wm[i] - M);
        pp[0] = M;
        pp[1] = S;
    }
    for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) {
        float a = 0.0f;
        for (int i = 0; i < ATT_WARPS; ++i)
            if (ws[i] > 0.0f) a += wacc[i][t] * expf(wm[i] - M);
        pp[2 + t] = a;
    }
    // ---- last CTA of the problem merges all partials in chunk order ----
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(counters + p, 1u) == nch - 1) ? 1u : 0u;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const float* pb = part + static_cast<size_t>(chunk_base[p]) * (d + 2);
    float GM = -FLT_MAX;
    for (uint32_t k = 0; k < nch; ++k) GM = fmaxf(GM, __ldcg(pb + k * (d + 2)));
    float GS = 0.0f;
    for (uint32_t k = 0; k < nch; ++k) {
        const float sk = __ldcg(pb + k * (d + 2) + 1);
        if (sk > 0.0f) GS += sk * expf(__ldcg(pb + k * (d + 2)) - GM);
    }
    const float inv = 1.0f / GS;
    if ((P.mode & MODE_PARTIAL) && P.out && threadIdx.x == 0) {
        P.out[0] = GM;  // (max, sum, acc[d]) for the cross-shard merge
        P.out[1] = GS;
    }
    for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) {
        float o = 0.0f;
        for (uint32_t k = 0; k < nch; ++k) {
            const float sk = __ldcg(pb + k * (d + 2) + 1);
            if (sk > 0.0f) o += __ldcg(pb + k * (d + 2) + 2 + t) * expf(__ldcg(pb + k * (d + 2)) - GM);
        }
        if (P.out) {
            if (P.mode & MODE_PARTIAL) P.out[2 + t] = o;  // shard partial: unnormalised
            else P.out[t] = o * inv;
        }
    }
    if (want_w)
        for (uint32_t r = threadIdx.x; r < K; r += blockDim.x)
            P.weights[r] = expf(__ldcg(P.weights + r) - GM) * inv;
    if (threadIdx.x == 0) counters[p] = 0;  // ready for the next step
}

// Fast path, d == 128: lane l owns elements [4l, 4l+4) of every row. Rows go
// in groups of 8: eight 128-bit K loads and eight V loads per lane in flight,
// partial dots reduced across the warp by a transposed butterfly (9 shuffles
// for 8 rows: after it, lane l holds the logit of row ((l>>4)&1)*4 +
// ((l>>3)&1)*2 + ((l>>2)&1)), so exp / max / sum run lane-parallel.
// GR rows per group: 8 (72 regs, 7 CTAs/SM) or 4 (<= 64 regs, 8 CTAs/SM)
__device__ __forceinline__ float4 ld_row4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

// GR=8 capped at 72 registers (7 CTAs/SM, an 8-byte spill): more warps in
// flight beat the 90-register / 5-CTA build on this memory-latency-bound
// loop (c3 250 -> 221 us; 6 CTAs: 231, 8 CTAs at 64 registers: 235)
// WARP (GQA sessions of ATT_WARPS query heads): a CTA is (session, chunk j)
// and warp h attends head h's rows [j*rows/4, (j+1)*rows/4): the four heads
// of a KV head read largely the same rows at about the same time on one SM,
// so the rows they share are served from L1. Each warp writes its own
// (problem, chunk) partial; the last warp of a problem merges them.
template <bool PARTIAL, int GR, bool WARP = false>  // PARTIAL: sharded steps write (max, sum, acc[d]) unnormalised
__global__ void __launch_bounds__(ATT_THREADS, GR == 4 ? 8 : 7)
attend128_kernel(const DecodeProblem* __restrict__ probs, const uint32_t* __restrict__ chunk_prob,
                 const uint32_t* __restrict__ chunk_base, float* __restrict__ part,
                 uint32_t* __restrict__ counters, uint32_t rows) {
    static_assert(!(WARP && PARTIAL), "WARP: unsharded steps only");
    constexpr int NC = 1, VEC = 4;
    __shared__ float wm[ATT_WARPS], ws[ATT_WARPS];
    __shared__ float wacc[ATT_WARPS][NC * 32 * VEC];
    __shared__ uint32_t is_last;
    const uint32_t c = blockIdx.x;
    // chunk entry: problem | chunk index << 20 (chunks may come in any order)
    const uint32_t cpk = chunk_prob[c];
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    const uint32_t p = (cpk & 0xfffffu) + (WARP ? static_cast<uint32_t>(w) : 0u);
    const DecodeProblem& P = probs[p];
    const SessionDev& sd = *P.s;
    const uint32_t d = 128, K = P.K, P0 = sd.P;
    const uint32_t j = cpk >> 20;
    const uint32_t nch = chunk_base[p + 1] - chunk_base[p];
    if (WARP && j >= nch) return;  // (heads of a session share K: never taken)
    const uint32_t rw = WARP ? j * (rows / ATT_WARPS) : j * rows + w * (rows / ATT_WARPS);  // this warp's first row
    const uint32_t nrw = rw < K ? min(rows / ATT_WARPS, K - rw) : 0u;
    const bool want_w = (P.mode & MODE_WEIGHTS) && P.weights;
    const float* const kpre = sd.kpre;
    const float* const vpre = sd.vpre;
    const float* const ktail = sd.ktail;
    const float* const vtail = sd.vtail;
    // base-2 logits: q pre-scaled by log2(e)/sqrt(d), exp2 = one MUFU op;
    // partials leave the kernel in natural-log units (x ln 2)
    float4 q4 = ld_row4(P.q + 4 * ln);
    {
        const float c2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(d)));
        q4.x *= c2;
        q4.y *= c2;
        q4.z *= c2;
        q4.w *= c2;
    }
    constexpr float LN2 = 0.6931471805599453f;
    // this lane's row slot within a group after the butterfly
    const int myrow = GR == 8 ? ((ln >> 4) & 1) * 4 + ((ln >> 3) & 1) * 2 + ((ln >> 2) & 1)
                              : ((ln >> 4) & 1) * 2 + ((ln >> 3) & 1);
    const bool up16 = ln & 16, up8 = ln & 8, up4 = ln & 4;

    float m = -FLT_MAX, s = 0.0f;
    float acc[NC][VEC] = {{0.0f, 0.0f, 0.0f, 0.0f}};
    for (uint32_t b0 = 0; b0 < nrw; b0 += 32) {  // 32-row index batches
    const uint32_t r0 = rw + b0;
    const uint32_t nr = min(32u, nrw - b0);
    // each lane resolves one row: element offset within its store (32-bit),
    // top bit = appended row (tail store); K and V share the offset
    uint32_t myoff = 0;
    if (ln < nr) {
        const uint32_t i = __ldg(P.sel + r0 + ln);
        myoff = i < P0 ? i * d : ((i - P0) * d) | 0x80000000u;
    }
    // lanes past the batch repeat row r0 (always present): every load is
    // unconditional, and those rows drop out through their zero probability
    {
        const uint32_t o0 = __shfl_sync(0xffffffffu, myoff, 0);
        if (ln >= nr) myoff = o0;
    }
    // sel is ascending, so appended rows form a suffix: nearly every batch is
    // prefill-only and takes the loop without per-row store selection
    const bool mixed = __any_sync(0xffffffffu, (myoff & 0x80000000u) != 0u);
    auto groups = [&](auto mixed_c, auto weights_c) {
    constexpr bool MIXED = decltype(mixed_c)::value;
    constexpr bool WTS = decltype(weights_c)::value;
    for (uint32_t g0 = 0; g0 < nr; g0 += GR) {
        float4 kk[GR], vv[GR];
#pragma unroll
        for (int u = 0; u < GR; ++u) {
            const uint32_t o = __shfl_sync(0xffffffffu, myoff, (g0 + u) & 31);
            if constexpr (MIXED) {
                const bool tl = o & 0x80000000u;
                const uint32_t e = (o & 0x7fffffffu) + 4 * ln;
                kk[u] = ld_row4((tl ? ktail : kpre) + e);
                vv[u] = ld_row4((tl ? vtail : vpre) + e);
            } else {
                kk[u] = ld_row4(kpre + (o + 4 * ln));
                vv[u] = ld_row4(vpre + (o + 4 * ln));
            }
        }
        float pd[GR];
#pragma unroll
        for (int u = 0; u < GR; ++u)
            pd[u] = fmaf(q4.w, kk[u].w, fmaf(q4.z, kk[u].z, fmaf(q4.y, kk[u].y, q4.x * kk[u].x)));
        // transposed butterfly: GR -> ... -> 1 partials, then a plain sum
        float lg;
        if constexpr (GR == 8) {
            float h4[4], h2[2];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float send = up16 ? pd[t] : pd[t + 4];
                const float keep = up16 ? pd[t + 4] : pd[t];
                h4[t] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const float send = up8 ? h4[t] : h4[t + 2];
                const float keep = up8 ? h4[t + 2] : h4[t];
                h2[t] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            const float send = up4 ? h2[0] : h2[1];
            const float keep = up4 ? h2[1] : h2[0];
            lg = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        } else {
            float h2[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const float send = up16 ? pd[t] : pd[t + 2];
                const float keep = up16 ? pd[t + 2] : pd[t];
                h2[t] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
            const float send = up8 ? h2[0] : h2[1];
            const float keep = up8 ? h2[1] : h2[0];
            lg = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            lg += __shfl_xor_sync(0xffffffffu, lg, 4);
        }
        lg += __shfl_xor_sync(0xffffffffu, lg, 2);
        lg += __shfl_xor_sync(0xffffffffu, lg, 1);
        const bool valid = g0 + myrow < nr;
        float gm = valid ? lg : -FLT_MAX;
        if constexpr (GR == 8) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, 4));
        gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, 8));
        gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, 16));
        if (__builtin_expect(gm > m, 0)) {  // warp-uniform: rescale only when the running max grows
            const float f = ex2f(m - gm);
            s *= f;
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[0][v] *= f;
            m = gm;
        }
        const float pr = valid ? ex2f(lg - m) : 0.0f;
        float ps = pr;  // rows replicated over the low lane bits: sum the row bits
        if constexpr (GR == 8) ps += __shfl_xor_sync(0xffffffffu, ps, 4);
        ps += __shfl_xor_sync(0xffffffffu, ps, 8);
        ps += __shfl_xor_sync(0xffffffffu, ps, 16);
        s += ps;
#pragma unroll
        for (int u = 0; u < GR; ++u) {
            const int src = GR == 8 ? ((u >> 2) & 1) * 16 + ((u >> 1) & 1) * 8 + (u & 1) * 4
                                    : ((u >> 1) & 1) * 16 + (u & 1) * 8;
            const float pu = __shfl_sync(0xffffffffu, pr, src);
            acc[0][0] = fmaf(pu, vv[u].x, acc[0][0]);
            acc[0][1] = fmaf(pu, vv[u].y, acc[0][1]);
            acc[0][2] = fmaf(pu, vv[u].z, acc[0][2]);
            acc[0][3] = fmaf(pu, vv[u].w, acc[0][3]);
        }
        if constexpr (WTS)
            if (valid && (ln & (GR == 8 ? 3 : 7)) == 0)
                P.weights[r0 + g0 + myrow] = lg * LN2;  // natural-log logit, normalized later
    }
    };
    if (want_w)
        groups(std::true_type{}, std::true_type{});
    else if (mixed)
        groups(std::true_type{}, std::false_type{});
    else
        groups(std::false_type{}, std::false_type{});
    }
    if constexpr (WARP) {
        // ---- warp partial of (problem, chunk j); the last warp merges ----
        float* pw = part + static_cast<size_t>(chunk_base[p] + j) * (d + 2);
        if (ln == 0) {
            pw[0] = nrw ? m * LN2 : -FLT_MAX;
            pw[1] = nrw ? s : 0.0f;
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) pw[2 + ln * VEC + v] = acc[0][v];
        __threadfence();
        __syncwarp();
        uint32_t lastw = 0;
        if (ln == 0) lastw = atomicAdd(counters + p, 1u) == nch - 1 ? 1u : 0u;
        if (!__shfl_sync(0xffffffffu, lastw, 0)) return;
        __threadfence();
        const float* pb = part + static_cast<size_t>(chunk_base[p]) * (d + 2);
        float GM = -FLT_MAX;
        for (uint32_t k = ln; k < nch; k += 32) GM = fmaxf(GM, __ldcg(pb + k * (d + 2)));
        for (int o = 16; o; o >>= 1) GM = fmaxf(GM, __shfl_xor_sync(0xffffffffu, GM, o));
        float GS = 0.0f, o4[VEC] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (uint32_t k = 0; k < nch; ++k) {  // chunk order
            const float sk = __ldcg(pb + k * (d + 2) + 1);
            if (sk > 0.0f) {
                const float f = expf(__ldcg(pb + k * (d + 2)) - GM);
                GS += sk * f;
#pragma unroll
                for (int v = 0; v < VEC; ++v) o4[v] += __ldcg(pb + k * (d + 2) + 2 + ln * VEC + v) * f;
            }
        }
        const float inv = 1.0f / GS;
        if (P.out)
#pragma unroll
            for (int v = 0; v < VEC; ++v) P.out[ln * VEC + v] = o4[v] * inv;
        if (want_w)
            for (uint32_t r = ln; r < K; r += 32) P.weights[r] = expf(__ldcg(P.weights + r) - GM) * inv;
        if (ln == 0) counters[p] = 0;  // ready for the next step
        return;
    }
    // ---- CTA partial ----
    if (ln == 0) {
        wm[w] = nrw ? m : -FLT_MAX;
        ws[w] = nrw ? s : 0.0f;
    }
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int v = 0; v < VEC; ++v) wacc[w][cc * 32 * VEC + ln * VEC + v] = acc[cc][v];
    __syncthreads();
    float M = -FLT_MAX;
#pragma unroll
    for (int i = 0; i < ATT_WARPS; ++i) M = fmaxf(M, wm[i]);
    float* pp = part + static_cast<size_t>(chunk_base[p] + j) * (d + 2);
    if (threadIdx.x == 0) {
        float S = 0.0f;
        for (int i = 0; i < ATT_WARPS; ++i)
            if (ws[i] > 0.0f) S += ws[i] * ex2f(wm[i] - M);
        pp[0] = M * LN2;  // natural-log units for the chunk / shard merges
        pp[1] = S;
    }
    for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) {
        float a = 0.0f;
        for (int i = 0; i < ATT_WARPS; ++i)
            if (ws[i] > 0.0f) a += wacc[i][t] * ex2f(wm[i] - M);
        pp[2 + t] = a;
    }
    // ---- last CTA of the problem merges all partials in chunk order ----
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(counters + p, 1u) == nch - 1) ? 1u : 0u;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const float* pb = part + static_cast<size_t>(chunk_base[p]) * (d + 2);
    float GM = -FLT_MAX;
    for (uint32_t k = 0; k < nch; ++k) GM = fmaxf(GM, __ldcg(pb + k * (d + 2)));
    float GS = 0.0f;
    for (uint32_t k = 0; k < nch; ++k) {
        const float sk = __ldcg(pb + k * (d + 2) + 1);
        if (sk > 0.0f) GS += sk * expf(__ldcg(pb + k * (d + 2)) - GM);
    }
    const float inv = 1.0f / GS;
    if (PARTIAL && P.out && threadIdx.x == 0) {
        P.out[0] = GM;  // (max, sum, acc[d]) for the cross-shard merge
        P.out[1] = GS;
    }
    for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) {
        float o = 0.0f;
        for (uint32_t k = 0; k < nch; ++k) {
            const float sk = __ldcg(pb + k * (d + 2) + 1);
            if (sk > 0.0f) o += __ldcg(pb + k * (d + 2) + 2 + t) * expf(__ldcg(pb + k * (d + 2)) - GM);
        }
        if (P.out) {
            if (PARTIAL) P.out[2 + t] = o;  // shard partial: unnormalised
            else P.out[t] = o * inv;
        }
    }
    if (want_w)
        for (uint32_t r = threadIdx.x; r < K; r += blockDim.x)
            P.weights[r] = expf(__ldcg(P.weights + r) - GM) * inv;
    if (threadIdx.x == 0) counters[p] = 0;  // ready for the next step
}

// Cross-shard log-sum-exp merge of the shards' (max, sum, acc[d]) partials
// (all-gathered: shard j's partial of problem p at parts[(j*nprob + p)*(d+2)]),
// in shard order: the sharded step's output.
__global__ void shard_merge_kernel(const float* __restrict__ parts, uint32_t nshard, uint32_t nprob,
                                   uint32_t d, float* __restrict__ out, size_t out_stride) {
    const uint32_t p = blockIdx.x;
    float GM = -FLT_MAX;
    for (uint32_t j = 0; j < nshard; ++j) {
        const float* pp = parts + (static_cast<size_t>(j) * nprob + p) * (d + 2);
        if (__ldcg(pp + 1) > 0.0f) GM = fmaxf(GM, __ldcg(pp));
    }
    float GS = 0.0f;
    for (uint32_t j = 0; j < nshard; ++j) {
        const float* pp = parts + (static_cast<size_t>(j) * nprob + p) * (d + 2);
        const float sj = __ldcg(pp + 1);
        if (sj > 0.0f) GS += sj * expf(__ldcg(pp) - GM);
    }
    const float inv = 1.0f / GS;
    for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) {
        float o = 0.0f;
        for (uint32_t j = 0; j < nshard; ++j) {
            const float* pp = parts + (static_cast<size_t>(j) * nprob + p) * (d + 2);
            const float sj = __ldcg(pp + 1);
            if (sj > 0.0f) o += __ldcg(pp + 2 + t) * expf(__ldcg(pp) - GM);
        }
        out[p * out_stride + t] = o * inv;
    }
}

cudaError_t launch_shard_merge(const float* parts, uint32_t nshard, uint32_t nprob, uint32_t d,
                               float* out, cudaStream_t st) {
    shard_merge_kernel<<<nprob, 128, 0, st>>>(parts, nshard, nprob, d, out, d);
    return cudaGetLastError();
}

cudaError_t launch_attend(const DecodeProblem* probs, const uint32_t* chunk_prob,
                          const uint32_t* chunk_base, uint32_t nchunks, float* part,
                          uint32_t* counters, uint32_t d, cudaStream_t st, bool partial,
                          uint32_t rows, bool warp_heads) {
#define CSA_ATT(NC, VEC) \
    attend_kernel<NC, VEC><<<nchunks, ATT_THREADS, 0, st>>>(probs, chunk_prob, chunk_base, part, counters, rows)
    // GR=8 at 72 registers (7 CTAs/SM): c3 attend 250 -> 221 us, c4 1692 ->
    // 1550 us per model step against GR=4 at 64 registers (8 CTAs/SM);
    // CSATTN_ATT_GR=4 forces the 4-row groups
    const int gr_env = std::getenv("CSATTN_ATT_GR") ? std::atoi(std::getenv("CSATTN_ATT_GR")) : 0;
    const int gr = gr_env == 4 ? 4 : 8;
    if (d == 128 && warp_heads && !partial) {
        if (gr == 4) attend128_kernel<false, 4, true><<<nchunks, ATT_THREADS, 0, st>>>(probs, chunk_prob, chunk_base, part, counters, rows);
        else attend128_kernel<false, 8, true><<<nchunks, ATT_THREADS, 0, st>>>(probs, chunk_prob, chunk_base, part, counters, rows);
    } else if (d == 128 && partial) {
        if (gr == 4) attend128_kernel<true, 4><<<nchunks, ATT_THREADS, 0, st>>>(probs, chunk_prob, chunk_base, part, counters, rows);
        else attend128_kernel<true, 8><<<nchunks, ATT_THREADS, 0, st>>>(probs, chunk_prob, chunk_base, part, counters, rows);
    } else if (d == 128) {
        if (gr == 4) attend128_kernel<false, 4><<<nchunks, ATT_THREADS, 0, st>>>(probs, chunk_prob, chunk_base, part, counters, rows);
        else attend128_kernel<false, 8><<<nchunks, ATT_THREADS, 0, st>>>(probs, chunk_prob, chunk_base, part, counters, rows);
    } else if (d % 4 == 0) {
        if (d <= 128) CSA_ATT(1, 4);
        else if (d <= 256) CSA_ATT(2, 4);
        else CSA_ATT(4, 4);
    } else {
        if (d <= 32) CSA_ATT(1, 1);
        else if (d <= 128) CSA_ATT(4, 1);
        else CSA_ATT(16, 1);
    }
#undef CSA_ATT
    return cudaGetLastError();
}

}  // namespace csa
