// route.cu — CSAttention decode, part 0: centroid routing (select_centroids,
// retrieval.cpp:40-87) + gather planning, one CTA per (session, query head).
//
// Per subspace b: normalize the query slice (fp64 sum of squares, f32 store,
// l2_normalize core.cpp:109-116), m*C sequential-fp64 centroid dots, argmax
// with strict > (lower j wins) or the top-tau backoff below the threshold.
// The gathered lists (b-major, selection order — gather_lists :95-109) and
// bounds on the accumulated scores are written to a per-problem plan that
// select.cu streams from.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace csa {

constexpr int RT_THREADS = 256;
constexpr int RT_WARPS = RT_THREADS / 32;

__global__ void __launch_bounds__(RT_THREADS)
route_kernel(const DecodeProblem* __restrict__ probs, RoutePlan* __restrict__ plans, int trig) {
    __shared__ float q[DMAX], qn[DMAX];
    __shared__ double csc[MAX_TABLES];
    __shared__ uint32_t ids[MAXM * MAXTAU], nids[MAXM], zero_mask;
    __shared__ uint32_t lists[MAXL], lsub[MAXL], nl, llive[MAXL];
    __shared__ double lmin[MAXL], lmax[MAXL];
    // the select launch that follows may start its prologue now (it waits
    // for this grid's completion before reading the plans)
    if (trig == 1) asm volatile("griddepcontrol.launch_dependents;");
    const DecodeProblem& P = probs[blockIdx.x];
    if (!(P.mode & MODE_SEARCH)) return;
    const SessionDev& sd = *P.s;
    const uint32_t m = sd.m, C = sd.C, d = sd.d, tid = threadIdx.x;
    RoutePlan& plan = plans[blockIdx.x];
    DecodeReport* Rp = reinterpret_cast<DecodeReport*>(P.rep);
    // q and the layout in one round trip (later phases read them from smem)
    __shared__ uint32_t soff[MAXM], swid[MAXM];
    for (uint32_t t = tid; t < d; t += blockDim.x) q[t] = P.q[t];
    if (tid < m) {
        soff[tid] = sd.offs[tid];
        swid[tid] = sd.widths[tid];
    }
    if (tid == 0) zero_mask = 0;
    __syncthreads();
    if (tid < m) {
        const uint32_t off = soff[tid], w = swid[tid];
        double n2 = 0.0;
        for (uint32_t t = 0; t < w; ++t) {
            const double x = q[off + t];
            n2 = __fma_rn(x, x, n2);  // x*x is exact in fp64
        }
        if (n2 == 0.0) {
            atomicOr(&zero_mask, 1u << tid);
        } else {
            const double inv = 1.0 / sqrt(n2);
            for (uint32_t t = 0; t < w; ++t)
                qn[off + t] = __double2float_rn(__dmul_rn(static_cast<double>(q[off + t]), inv));
        }
    }
    __syncthreads();
    for (uint32_t x = tid; x < m * C; x += blockDim.x) {
        const uint32_t b = x / C, j = x - b * C;
        if (zero_mask & (1u << b)) continue;
        const uint32_t off = soff[b], w = swid[b];
        const float* c = sd.cent + static_cast<size_t>(C) * off + static_cast<size_t>(j) * w;
        double acc = 0.0;
        if ((w & 3u) == 0u && ((C * off + j * w) & 3u) == 0u) {  // 16-byte rows: vector loads
            const float4* c4 = reinterpret_cast<const float4*>(c);
#pragma unroll 4
            for (uint32_t t4 = 0; t4 < w / 4; ++t4) {
                const float4 v = __ldg(c4 + t4);
                const float* qs = qn + off + 4 * t4;
                acc = __fma_rn((double)qs[0], (double)v.x, acc);
                acc = __fma_rn((double)qs[1], (double)v.y, acc);
                acc = __fma_rn((double)qs[2], (double)v.z, acc);
                acc = __fma_rn((double)qs[3], (double)v.w, acc);
            }
        } else {
            for (uint32_t t = 0; t < w; ++t) acc = __fma_rn((double)qn[off + t], (double)__ldg(c + t), acc);
        }
        csc[x] = acc;
    }
    __syncthreads();
    const int wid = tid >> 5, ln = tid & 31;
    for (uint32_t b = wid; b < m; b += RT_WARPS) {
        if (zero_mask & (1u << b)) {  // degenerate slice: centroid 0, no backoff
            if (ln == 0) {
                ids[b * MAXTAU] = 0;
                nids[b] = 1;
                Rp->best_cos[b] = 1.0;
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
                for (uint32_t u = 0; u < r; ++u) used |= (ids[b * MAXTAU + u] == j);
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
            if (ln == 0) ids[b * MAXTAU + r] = bj;
            __syncwarp();
            if (r == 0) {
                if (ln == 0) Rp->best_cos[b] = bv;
                if (bv >= sd.threshold) {
                    if (ln == 0) nids[b] = 1;
                    break;
                }
            }
            if (ln == 0) nids[b] = r + 1;
        }
        __syncwarp();
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t n = 0;
        unsigned long long dots = 0;
        for (uint32_t b = 0; b < m; ++b) {
            if (!(zero_mask & (1u << b))) dots += static_cast<unsigned long long>(C) * swid[b];
            for (uint32_t r = 0; r < nids[b]; ++r) {
                lists[n] = b * C + ids[b * MAXTAU + r];
                lsub[n] = b;
                ++n;
            }
        }
        nl = n;
        plan.nl = n;
        Rp->nl = n;
        Rp->dot_ops_lo = static_cast<uint32_t>(dots);
        Rp->dot_ops_hi = static_cast<uint32_t>(dots >> 32);
    }
    __syncthreads();
    if (trig == 2) asm volatile("griddepcontrol.launch_dependents;");
    if (tid < nl) {
        plan.lists[tid] = lists[tid];
        plan.lsub[tid] = lsub[tid];
        Rp->lists[tid] = lists[tid];
    }
    // bounds on every accumulated score: a pool key's score is a sum of
    // w_l * score over a non-empty subset of the gathered lists, each score in
    // [tmin_l, tmax_l] (the lists' live score bounds)
    // the lists' live lengths and score bounds, loaded lane-parallel (one
    // round trip); the sums below stay sequential in list order
    if (tid < nl) {
        const uint32_t t = lists[tid];
        const uint32_t lv = __ldcg(sd.live_g + t);
        const float2 mm = __ldcg(sd.tmm + t);
        const double w = sd.weights[lsub[tid]];
        lmin[tid] = lv ? w * static_cast<double>(mm.x) : 0.0;
        lmax[tid] = lv ? w * static_cast<double>(mm.y) : 0.0;
        llive[tid] = lv;
    }
    __syncthreads();
    if (tid == 0) {
        double neg = 0.0, pos = 0.0, amin = DBL_MAX, bmax = -DBL_MAX;
        bool any = false, any_neg = false, any_pos = false;
        for (uint32_t l = 0; l < nl; ++l) {
            if (llive[l] == 0) continue;
            const double a = lmin[l], b = lmax[l];
            any = true;
            if (a < 0.0) { neg += a; any_neg = true; }
            if (b > 0.0) { pos += b; any_pos = true; }
            amin = fmin(amin, a);
            bmax = fmax(bmax, b);
        }
        double lo = any ? (any_neg ? neg : amin) : 0.0;
        double hi = any ? (any_pos ? pos : bmax) : 0.0;
        if (!sd.passthrough) {  // window keys compete at score 0 when absent
            lo = fmin(lo, 0.0);
            hi = fmax(hi, 0.0);
        }
        plan.lo = lo;
        plan.hi = hi;
    }
    if (wid == 0) {  // gathered_entries (CostCounters): live lengths of the lists
        uint32_t g = 0;
        for (uint32_t l = ln; l < nl; l += 32) g += llive[l];
        for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
        if (ln == 0) {
            Rp->gathered_lo = g;
            Rp->gathered_hi = 0;
        }
    }
}

cudaError_t launch_route(const DecodeProblem* probs, RoutePlan* plans, uint32_t nprob,
                         cudaStream_t st, int trig) {
    route_kernel<<<nprob, RT_THREADS, 0, st>>>(probs, plans, trig);
    return cudaGetLastError();
}

}  // namespace csa
