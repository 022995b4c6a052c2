// csat_dev.cu — the tables section of a CSAT v1 image written on the device
// (index file I/O on device).
//
// A session's tables live index-sorted with tombstones (select.cu). The image
// stores each table as a TopList (score desc, idx asc; TopList::from_scores /
// try_insert order, index.cpp:17-62) followed by its length prefix
// (serialize_index, index.cpp:308-312). Here:
//   csat_keys_kernel    one 64-bit key per entry: ~ordered(score) << 32 | idx,
//                       tombstones -> ~0 (sort last)
//   CUB segmented radix sort of the keys, one segment per table
//   csat_write_kernel   one CTA per table: len u32 | indices u32 x len |
//                       scores (f32, or IEEE half RNE) x len at the table's
//                       byte offset (exclusive prefix of the table sizes)
// The host prepends the header and centroid rows (csat.cpp).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "common.cuh"
#include "csat_half.h"
#include "kernels.h"

namespace csa {

__device__ __forceinline__ uint32_t ordered_asc(uint32_t u) {  // float bits -> ascending uint
    return (u & 0x80000000u) ? ~u : (u ^ 0x80000000u);
}
__device__ __forceinline__ uint32_t float_of_ordered(uint32_t o) {
    return (o & 0x80000000u) ? (o ^ 0x80000000u) : ~o;
}

__global__ void csat_keys_kernel(const uint2* __restrict__ ent, const uint32_t* __restrict__ n_used,
                                 uint32_t cap2, unsigned long long* __restrict__ keys) {
    const uint32_t t = blockIdx.x;
    const uint32_t n = n_used[t];
    for (uint32_t p = threadIdx.x; p < cap2; p += blockDim.x) {
        unsigned long long k = ~0ull;
        if (p < n) {
            const uint2 e = ent[static_cast<size_t>(t) * cap2 + p];
            if (!(e.x & TOMB))
                k = (static_cast<unsigned long long>(~ordered_asc(e.y)) << 32) | e.x;
        }
        keys[static_cast<size_t>(t) * cap2 + p] = k;
    }
}

__global__ void csat_write_kernel(const unsigned long long* __restrict__ sorted,
                                  const uint32_t* __restrict__ live, const unsigned long long* __restrict__ off,
                                  uint32_t cap2, int half, unsigned char* __restrict__ out) {
    const uint32_t t = blockIdx.x;
    const uint32_t n = live[t];
    unsigned char* base = out + off[t];
    const unsigned long long* k = sorted + static_cast<size_t>(t) * cap2;
    if (threadIdx.x == 0) {
        base[0] = n & 0xff;
        base[1] = (n >> 8) & 0xff;
        base[2] = (n >> 16) & 0xff;
        base[3] = (n >> 24) & 0xff;
    }
    unsigned char* ib = base + 4;
    unsigned char* sb = ib + 4ull * n;
    for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) {
        const unsigned long long key = k[r];
        const uint32_t idx = static_cast<uint32_t>(key);
        const uint32_t bits = float_of_ordered(~static_cast<uint32_t>(key >> 32));
        for (int i = 0; i < 4; ++i) ib[4ull * r + i] = (idx >> (8 * i)) & 0xff;
        if (half) {
            const uint16_t h = csa_half::to_half(csa_half::bits_f32(bits));
            sb[2ull * r] = h & 0xff;
            sb[2ull * r + 1] = h >> 8;
        } else {
            for (int i = 0; i < 4; ++i) sb[4ull * r + i] = (bits >> (8 * i)) & 0xff;
        }
    }
}

size_t csat_sort_temp_bytes(uint32_t ntables, uint32_t cap2) {
    size_t bytes = 0;
    const uint32_t n = ntables * cap2;
    cub::DeviceSegmentedRadixSort::SortKeys(nullptr, bytes, static_cast<const unsigned long long*>(nullptr),
                                            static_cast<unsigned long long*>(nullptr), static_cast<int>(n),
                                            static_cast<int>(ntables), static_cast<const int*>(nullptr),
                                            static_cast<const int*>(nullptr));
    return bytes;
}

cudaError_t launch_csat_tables(const uint2* ent, const uint32_t* n_used, const uint32_t* live,
                               uint32_t ntables, uint32_t cap2, const int* seg_begin, const int* seg_end,
                               const unsigned long long* off, int half, unsigned long long* keys,
                               unsigned long long* sorted, void* temp, size_t temp_bytes,
                               unsigned char* out, cudaStream_t st) {
    csat_keys_kernel<<<ntables, 256, 0, st>>>(ent, n_used, cap2, keys);
    cudaError_t e = cub::DeviceSegmentedRadixSort::SortKeys(temp, temp_bytes, keys, sorted,
                                                            static_cast<int>(ntables * cap2),
                                                            static_cast<int>(ntables), seg_begin, seg_end, 0,
                                                            64, st);
    if (e != cudaSuccess) return e;
    csat_write_kernel<<<ntables, 256, 0, st>>>(sorted, live, off, cap2, half, out);
    return cudaGetLastError();
}

}  // namespace csa
