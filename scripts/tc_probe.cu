// tc_probe.cu — checks the tcgen05 encodings in csrc/tc.cuh on a B200:
//   S^T[128 rows][64 cols] = K[128x128] . Q[64x128]^T   (A K-major, B K-major)
//   O^T[128 dims][64 cols] = V^T . P^T with V[128 rows][128 dims] as an
//                            MN-major A operand and P[64][128] K-major B
// against a double-precision host product of the same bf16-rounded inputs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2604_08584_b200/csrc
//        scripts/tc_probe.cu -o scripts/tc_probe
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc.cuh"

using namespace csa;

__global__ void __launch_bounds__(128, 1)
probe(const float* K, const float* Q, const float* V, const float* P, float* S_out, float* O_out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sK = sm;            // 128 x 128 bf16 K-major: 32 KB
    unsigned char* sQ = sm + 32768;    // 64 x 128 K-major: 16 KB
    unsigned char* sV = sm + 49152;    // V as MN-major A (M = dims 128, K = rows 128): 32 KB
    unsigned char* sP = sm + 81920;    // P as K-major B (N = 64, K = rows 128): 16 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 128 * 128; i += 128) {
        const int r = i / 128, k = i % 128;
        *reinterpret_cast<__nv_bfloat16*>(sK + tc::kmaj_off(r, k, 128)) = __float2bfloat16(K[i]);
        *reinterpret_cast<__nv_bfloat16*>(sV + tc::mnmaj_off(k, r, 128)) = __float2bfloat16(V[i]);
    }
    for (int i = tid; i < 64 * 128; i += 128) {
        const int r = i / 128, k = i % 128;
        *reinterpret_cast<__nv_bfloat16*>(sQ + tc::kmaj_off(r, k, 64)) = __float2bfloat16(Q[i]);
        *reinterpret_cast<__nv_bfloat16*>(sP + tc::kmaj_off(r, k, 64)) = __float2bfloat16(P[i]);
    }
    if (tid == 0) tc::mbar_init(&bar, 1);
    if (tid < 32) tc::tmem_alloc<128>(&tbase);
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tS = tbase, tO = tbase + 64;
    if (tid == 0) {
        const uint32_t id1 = tc::idesc_bf16(128, 64, false, false);
        for (int s = 0; s < 8; ++s) {
            const uint32_t koff = (s >> 2) * 128 * 128 + (s & 3) * 32;
            const uint32_t qoff = (s >> 2) * 64 * 128 + (s & 3) * 32;
            tc::mma_bf16(tS, tc::desc_sw128(tc::smem_u32(sK) + koff, 16, 1024),
                         tc::desc_sw128(tc::smem_u32(sQ) + qoff, 16, 1024), id1, s > 0);
        }
        const uint32_t id2 = tc::idesc_bf16(128, 64, true, false);
        for (int s = 0; s < 8; ++s) {
            const uint32_t voff = s * 2048;
            const uint32_t poff = (s >> 2) * 64 * 128 + (s & 3) * 32;
            tc::mma_bf16(tO, tc::desc_sw128(tc::smem_u32(sV) + voff, 128 * 128, 1024),
                         tc::desc_sw128(tc::smem_u32(sP) + poff, 16, 1024), id2, s > 0);
        }
        tc::commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after();
    const int w = tid >> 5;
    const uint32_t lane_base = static_cast<uint32_t>(w * 32) << 16;
    for (int c = 0; c < 64; c += 32) {
        float v[32];
        tc::tmem_ld32(tS + lane_base + c, v);
        for (int i = 0; i < 32; ++i) S_out[tid * 64 + c + i] = v[i];
        tc::tmem_ld32(tO + lane_base + c, v);
        for (int i = 0; i < 32; ++i) O_out[tid * 64 + c + i] = v[i];
    }
    tc::fence_before();
    __syncthreads();
    if (tid < 32) tc::tmem_free<128>(tbase);
}

// MMA throughput for the union kernel's shapes: QK (M=128, N=64, K=16, A and B
// K-major) and PV (M=128, N=128, K=16, B MN-major), n iterations each
__global__ void __launch_bounds__(128, 1) mma_rate(int n, int kind, unsigned long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
    if (tid == 0) tc::mbar_init(&bar, 1);
    if (tid < 32) tc::tmem_alloc<256>(&tbase);
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
        const uint32_t b = tc::smem_u32(sm);
        const uint32_t idq = tc::idesc_bf16(128, 64, false, false);
        const uint32_t idp = tc::idesc_bf16(128, 128, false, true);
        const uint32_t idm = tc::idesc_bf16(128, 256, false, false);
        unsigned long long t0 = clock64();
        for (int it = 0; it < n; ++it) {
            if (kind == 0)
                tc::mma_bf16(tbase, tc::desc_sw128(b + (it & 3) * 32, 16, 1024),
                             tc::desc_sw128(b + 32768 + (it & 3) * 32, 16, 1024), idq, 1);
            else if (kind == 1)
                tc::mma_bf16(tbase + 128, tc::desc_sw128(b + (it & 3) * 32, 16, 1024),
                             tc::desc_sw128(b + 32768 + (it & 3) * 2048, 8192, 1024), idp, 1);
            else if (kind == 2)
                tc::mma_bf16(tbase, tc::desc_sw128(b + (it & 3) * 32, 16, 1024),
                             tc::desc_sw128(b + 16384 + (it & 3) * 32, 16, 1024), idm, 1);
            else if (kind == 3)  // QK shape, 2 alternating accumulators
                tc::mma_bf16(tbase + 64 * (it & 1), tc::desc_sw128(b + (it & 3) * 32, 16, 1024),
                             tc::desc_sw128(b + 32768 + (it & 3) * 32, 16, 1024), idq, 1);
            else if (kind == 4)  // QK shape, 4 alternating accumulators
                tc::mma_bf16(tbase + 64 * (it & 3), tc::desc_sw128(b + (it & 3) * 32, 16, 1024),
                             tc::desc_sw128(b + 32768 + (it & 3) * 32, 16, 1024), idq, 1);
            else if (kind == 5)  // PV shape, 2 alternating accumulators
                tc::mma_bf16(tbase + 128 * (it & 1), tc::desc_sw128(b + (it & 3) * 32, 16, 1024),
                             tc::desc_sw128(b + 32768 + (it & 3) * 2048, 8192, 1024), idp, 1);
            else  // QK shape, A operand in no-swizzle... same as 0 but enable=0 each time (no accumulate)
                tc::mma_bf16(tbase, tc::desc_sw128(b + (it & 3) * 32, 16, 1024),
                             tc::desc_sw128(b + 32768 + (it & 3) * 32, 16, 1024), idq, 0);
        }
        tc::commit(&bar);
        tc::mbar_wait(&bar, 0);
        cycles[kind] = clock64() - t0;
    }
    tc::fence_before();
    __syncthreads();
    if (tid < 32) tc::tmem_free<256>(tbase);
}

// O[128][128] = P[128 x 64] . V[64 x 128]: P from TMEM (tcgen05.st), V MN-major B
__global__ void __launch_bounds__(128, 1) probe_ts(const float* Pm, const float* V, float* O_out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sV = sm;  // V as MN-major B (N = dims 128, K = rows 64): 16 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 64 * 128; i += 128) {
        const int r = i / 128, c = i % 128;
        *reinterpret_cast<__nv_bfloat16*>(sV + tc::mnmaj_off(c, r, 64)) = __float2bfloat16(V[i]);
    }
    if (tid == 0) tc::mbar_init(&bar, 1);
    if (tid < 32) tc::tmem_alloc<256>(&tbase);
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int w = tid >> 5;
    const uint32_t lane = static_cast<uint32_t>(w * 32) << 16;
    const uint32_t tP = tbase, tO = tbase + 128;
    for (int s = 0; s < 4; ++s) {  // k-step s: P[tid][16s .. 16s+15] -> columns 8s .. 8s+7
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) {
            const __nv_bfloat162 h = __floats2bfloat162_rn(Pm[tid * 64 + 16 * s + 2 * i], Pm[tid * 64 + 16 * s + 2 * i + 1]);
            v[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        tc::tmem_st8(tP + lane + 8 * s, v);
    }
    tc::tmem_st_wait();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
        const uint32_t id = tc::idesc_bf16(128, 128, false, true);
        for (int s = 0; s < 4; ++s)
            tc::mma_bf16_ts(tO, tP + 8 * s, tc::desc_sw128(tc::smem_u32(sV) + s * 2048, 64 * 128, 1024), id, s > 0);
        tc::commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after();
    for (int c = 0; c < 128; c += 32) {
        float v[32];
        tc::tmem_ld32(tO + lane + c, v);
        for (int i = 0; i < 32; ++i) O_out[tid * 128 + c + i] = v[i];
    }
    tc::fence_before();
    __syncthreads();
    if (tid < 32) tc::tmem_free<256>(tbase);
}

static float bf(float x) {
    return __bfloat162float(__float2bfloat16(x));
}

int main() {
    std::vector<float> K(128 * 128), Q(64 * 128), V(128 * 128), P(64 * 128);
    srand(1);
    auto rnd = [] { return (rand() / (float)RAND_MAX) * 2.0f - 1.0f; };
    for (auto& x : K) x = rnd();
    for (auto& x : Q) x = rnd();
    for (auto& x : V) x = rnd();
    for (auto& x : P) x = rnd();
    float *dK, *dQ, *dV, *dP, *dS, *dO;
    cudaMalloc(&dK, K.size() * 4);
    cudaMalloc(&dQ, Q.size() * 4);
    cudaMalloc(&dV, V.size() * 4);
    cudaMalloc(&dP, P.size() * 4);
    cudaMalloc(&dS, 128 * 64 * 4);
    cudaMalloc(&dO, 128 * 64 * 4);
    cudaMemcpy(dK, K.data(), K.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dQ, Q.data(), Q.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dP, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
    probe<<<1, 128, 98304>>>(dK, dQ, dV, dP, dS, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> S(128 * 64), O(128 * 64);
    cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double es = 0, eo = 0;
    int bad = 0;
    for (int r = 0; r < 128; ++r)
        for (int j = 0; j < 64; ++j) {
            double s = 0, o = 0;
            for (int k = 0; k < 128; ++k) {
                s += (double)bf(K[r * 128 + k]) * bf(Q[j * 128 + k]);
                o += (double)bf(V[k * 128 + r]) * bf(P[j * 128 + k]);  // O^T[dim r][col j]
            }
            const double d1 = fabs(s - S[r * 64 + j]), d2 = fabs(o - O[r * 64 + j]);
            es = fmax(es, d1);
            eo = fmax(eo, d2);
            if ((d1 > 1e-3 || d2 > 1e-3) && bad++ < 5)
                printf("r=%d j=%d S %.5f vs %.5f | O %.5f vs %.5f\n", r, j, S[r * 64 + j], s,
                       O[r * 64 + j], o);
        }
    printf("max |S err| %.3g  max |O err| %.3g  %s\n", es, eo, (es < 1e-3 && eo < 1e-3) ? "OK" : "FAIL");
    {  // A from TMEM
        std::vector<float> Pm(128 * 64), V2(64 * 128), O2(128 * 128);
        for (auto& x : Pm) x = rnd();
        for (auto& x : V2) x = rnd();
        float *dPm, *dV2, *dO2;
        cudaMalloc(&dPm, Pm.size() * 4);
        cudaMalloc(&dV2, V2.size() * 4);
        cudaMalloc(&dO2, O2.size() * 4);
        cudaMemcpy(dPm, Pm.data(), Pm.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dV2, V2.data(), V2.size() * 4, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(probe_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
        probe_ts<<<1, 128, 32768>>>(dPm, dV2, dO2);
        cudaError_t e2 = cudaDeviceSynchronize();
        cudaMemcpy(O2.data(), dO2, O2.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int m = 0; m < 128; ++m)
            for (int j = 0; j < 128; ++j) {
                double o = 0;
                for (int k = 0; k < 64; ++k) o += (double)bf(Pm[m * 64 + k]) * bf(V2[k * 128 + j]);
                err = fmax(err, fabs(o - O2[m * 128 + j]));
            }
        printf("A-from-TMEM PV: %s max |err| %.3g %s\n", cudaGetErrorString(e2), err, err < 1e-3 ? "OK" : "FAIL");
    }
    unsigned long long* dc;
    cudaMalloc(&dc, 64);
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const char* names[7] = {"QK  M128 N64  K16 (A,B K-major)", "PV  M128 N128 K16 (B MN-major)", "ref M128 N256 K16 (K-major)",
                            "QK  2 accumulators", "QK  4 accumulators", "PV  2 accumulators", "QK  no accumulate"};
    for (int kind = 0; kind < 7; ++kind) {
        const int n = 4096;
        mma_rate<<<1, 128, 65536>>>(n, kind, dc);
        unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaDeviceSynchronize();
        cudaMemcpy(c, dc, 64, cudaMemcpyDeviceToHost);
        const int N = (kind == 1 || kind == 5) ? 128 : kind == 2 ? 256 : 64;
        printf("%s: %.1f cycles/MMA (pacing-law floor %d)\n", names[kind], (double)c[kind] / n, 128 * N / 256);
    }
    return 0;
}
