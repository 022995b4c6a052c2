// csat_half.h — IEEE binary16 <-> binary32 for the CSAT image, shared by the
// host codec (csat.cpp) and the device table writer (csat_dev.cu) so both
// produce identical bytes. Round to nearest even from f32, NaN -> quiet NaN
// with the sign kept, overflow -> inf, underflow -> signed zero: the
// conversion the reference's f32_to_f16 / f16_to_f32 perform (util.cpp:8-74).
#pragma once
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define CSA_HD __host__ __device__ __forceinline__
#else
#define CSA_HD inline
#endif

namespace csa_half {

CSA_HD uint32_t f32_bits(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    return x;
}
CSA_HD float bits_f32(uint32_t x) {
    float f;
    memcpy(&f, &x, 4);
    return f;
}

CSA_HD uint16_t to_half(float f) {
    const uint32_t x = f32_bits(f);
    const uint32_t sign = (x >> 16) & 0x8000u;
    const uint32_t e8 = (x >> 23) & 0xffu;
    uint32_t frac = x & 0x7fffffu;
    if (e8 == 0xffu) return static_cast<uint16_t>(sign | (frac ? 0x7e00u : 0x7c00u));  // nan / inf
    const int e = static_cast<int>(e8) - 127;
    if (e > 15) return static_cast<uint16_t>(sign | 0x7c00u);  // overflow
    if (e >= -14) {                                           // normal
        uint32_t h = sign | (static_cast<uint32_t>(e + 15) << 10) | (frac >> 13);
        const uint32_t rem = frac & 0x1fffu;
        h += (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ? 1u : 0u;  // RNE, may carry into the exponent
        return static_cast<uint16_t>(h);
    }
    if (e >= -24) {  // subnormal half
        frac |= 0x800000u;
        const int sh = 13 + (-14 - e);
        uint32_t h = sign | (frac >> sh);
        const uint32_t rem = frac & ((1u << sh) - 1u), mid = 1u << (sh - 1);
        h += (rem > mid || (rem == mid && (h & 1u))) ? 1u : 0u;
        return static_cast<uint16_t>(h);
    }
    return static_cast<uint16_t>(sign);  // underflow
}

CSA_HD float from_half(uint16_t h) {
    const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
    const uint32_t e5 = (h >> 10) & 0x1fu;
    uint32_t frac = h & 0x3ffu;
    uint32_t x;
    if (e5 == 0x1fu) {
        x = sign | 0x7f800000u | (frac << 13);
    } else if (e5 != 0) {
        x = sign | ((e5 + 112u) << 23) | (frac << 13);
    } else if (frac == 0) {
        x = sign;
    } else {  // subnormal: normalise
        uint32_t e = 113;
        while (!(frac & 0x400u)) {
            frac <<= 1;
            --e;
        }
        x = sign | (e << 23) | ((frac & 0x3ffu) << 13);
    }
    return bits_f32(x);
}

}  // namespace csa_half
