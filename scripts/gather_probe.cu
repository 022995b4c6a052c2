// gather_probe.cu — achievable HBM bandwidth for gathers of random rows of
// B bytes from a large table (the access pattern of the attention and union
// kernels: 512-byte K/V rows), vs a contiguous stream. Diagnostics only.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/gather_probe.cu -o scripts/gather_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

template <int F4>  // float4 per row
__global__ void gather(const float4* __restrict__ tab, const unsigned* __restrict__ idx, unsigned nrow,
                       float* __restrict__ out) {
    // each warp gathers rows; lane l reads float4 l, l+32, ... of the row
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    for (unsigned r0 = warp * 8; r0 < nrow; r0 += nw * 8) {
        float4 v[8][F4 / 32 > 0 ? F4 / 32 : 1];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const unsigned r = r0 + u < nrow ? idx[r0 + u] : 0;
#pragma unroll
            for (int c = 0; c < (F4 / 32 > 0 ? F4 / 32 : 1); ++c)
                v[u][c] = __ldg(tab + static_cast<size_t>(r) * F4 + c * 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < (F4 / 32 > 0 ? F4 / 32 : 1); ++c) {
                acc.x += v[u][c].x;
                acc.y += v[u][c].y;
            }
    }
    if (acc.x == 12345.f) out[0] = acc.y;
}

int main() {
    const size_t tab_bytes = 1ull << 30;  // 1 GB table
    float4* tab;
    cudaMalloc(&tab, tab_bytes);
    cudaMemset(tab, 0, tab_bytes);
    float* out;
    cudaMalloc(&out, 16);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](auto kern, int row_bytes, bool sorted, const char* name) {
        const unsigned rows_in_tab = static_cast<unsigned>(tab_bytes / row_bytes);
        const unsigned n = static_cast<unsigned>((512ull << 20) / row_bytes);  // 512 MB gathered
        std::vector<unsigned> h(n);
        srand(7);
        for (unsigned i = 0; i < n; ++i) h[i] = sorted ? i % rows_in_tab : (unsigned)(((unsigned long long)rand() * 2654435761ull) % rows_in_tab);
        unsigned* d;
        cudaMalloc(&d, n * 4ull);
        cudaMemcpy(d, h.data(), n * 4ull, cudaMemcpyHostToDevice);
        for (int occ : {4, 8, 16}) {
            kern<<<sms * occ, 256>>>(tab, d, n, out);
            cudaEventRecord(a);
            for (int it = 0; it < 5; ++it) kern<<<sms * occ, 256>>>(tab, d, n, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%-28s row %5d B, %2d CTA/SM: %7.1f GB/s\n", name, row_bytes, occ,
                   5.0 * n * (double)row_bytes / (ms * 1e-3) / 1e9);
        }
        cudaFree(d);
    };
    run(gather<32>, 512, false, "random rows");
    run(gather<64>, 1024, false, "random rows");
    run(gather<256>, 4096, false, "random rows");
    run(gather<32>, 512, true, "sequential rows");
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
