// csat.cpp — the CSAT v1 index image, host side.
//
// Byte layout (little endian), as written by the reference's serialize_index
// (index.cpp:289-318) and validated by deserialize_index (:320-396):
//   "CSAT" | version u16 = 1 | flags u16 (bit 0: 16-bit scores AND centroid
//   elements, bit 1: keys normalized) | m u32 | C u32 | L u32 | d u32 |
//   prefill u64 | widths u32 x m | centroid rows (C x width_b per subspace) |
//   per table (subspace-major): len u32, indices u32 x len, scores x len.
// 16-bit values are IEEE half, round-to-nearest-even from f32 (util.cpp:8-43).
// The parser follows the reference's check order exactly, so the first
// violation raises the same error class with the same message.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "csattn_b200.h"
#include "errors.hpp"
#include "csat_half.h"
#include "csat.h"

namespace {

using csa_host::fail;

constexpr uint16_t kVersion = 1;
constexpr uint16_t kHalf = 1u << 0, kNormalized = 1u << 1;

using csa_half::from_half;
using csa_half::to_half;

struct Writer {
    uint8_t* p;
    uint64_t cap, n = 0;
    void bytes(const void* src, uint64_t k) {
        if (p && n + k <= cap) std::memcpy(p + n, src, k);
        n += k;
    }
    void u16(uint16_t v) {
        const uint8_t b[2] = {static_cast<uint8_t>(v), static_cast<uint8_t>(v >> 8)};
        bytes(b, 2);
    }
    void u32(uint32_t v) {
        uint8_t b[4];
        for (int i = 0; i < 4; ++i) b[i] = static_cast<uint8_t>(v >> (8 * i));
        bytes(b, 4);
    }
    void u64(uint64_t v) {
        uint8_t b[8];
        for (int i = 0; i < 8; ++i) b[i] = static_cast<uint8_t>(v >> (8 * i));
        bytes(b, 8);
    }
    void value(float f, bool half) {
        if (half) {
            u16(to_half(f));
        } else {
            uint32_t b;
            std::memcpy(&b, &f, 4);
            u32(b);
        }
    }
};

struct Reader {
    const uint8_t* p;
    uint64_t n, pos = 0;
    void need(uint64_t k, const char* what) const {
        if (n - pos < k)
            fail(CSATTN_ERR_TRUNCATED, "file ends at byte " + std::to_string(pos) + " while reading " + what);
    }
    uint64_t le(int k, const char* what) {
        need(static_cast<uint64_t>(k), what);
        uint64_t v = 0;
        for (int i = 0; i < k; ++i) v |= static_cast<uint64_t>(p[pos + i]) << (8 * i);
        pos += static_cast<uint64_t>(k);
        return v;
    }
    float value(bool half, const char* what) {
        if (half) return from_half(static_cast<uint16_t>(le(2, what)));
        const uint32_t b = static_cast<uint32_t>(le(4, what));
        float f;
        std::memcpy(&f, &b, 4);
        return f;
    }
};

void check_header(const csattn_csat_header* h) {
    if (h->m == 0 || h->m > CSATTN_CSAT_MAX_SUBSPACES)
        fail(CSATTN_ERR_PARAMETER, "CSAT header: subspace count out of range");
    uint64_t sum = 0;
    for (uint64_t b = 0; b < h->m; ++b) sum += h->widths[b];
    if (sum != h->dim) fail(CSATTN_ERR_DIMENSION, "CSAT header: widths do not sum to the dimension");
    if (h->score_bits != 16 && h->score_bits != 32)
        fail(CSATTN_ERR_PARAMETER, "CSAT header: score_bits must be 16 or 32");
}

// The header fields of an image (reference check order through the widths).
void parse_header(Reader& in, csattn_csat_header* h) {
    in.need(4, "magic");
    if (std::memcmp(in.p, "CSAT", 4) != 0) fail(CSATTN_ERR_BAD_MAGIC, "not an index file (bad magic at byte 0)");
    in.pos = 4;
    const uint16_t version = static_cast<uint16_t>(in.le(2, "version"));
    if (version != kVersion) fail(CSATTN_ERR_VERSION, "unsupported index version " + std::to_string(version));
    const uint16_t flags = static_cast<uint16_t>(in.le(2, "flags"));
    if (flags & ~(kHalf | kNormalized))
        fail(CSATTN_ERR_CORRUPT, "unknown flag bits set: 0x" + std::to_string(flags));
    const uint32_t m = static_cast<uint32_t>(in.le(4, "subspace count"));
    const uint32_t c = static_cast<uint32_t>(in.le(4, "centroid count"));
    const uint32_t cap = static_cast<uint32_t>(in.le(4, "list capacity"));
    const uint32_t d = static_cast<uint32_t>(in.le(4, "dimension"));
    const uint64_t prefill = in.le(8, "prefill length");
    if (m == 0 || c == 0 || cap == 0 || d == 0 || prefill == 0)
        fail(CSATTN_ERR_CORRUPT, "zero field in header (m, C, L, d, prefill)");
    if (m > CSATTN_CSAT_MAX_SUBSPACES)
        fail(CSATTN_ERR_PARAMETER, "B200 path supports m <= " + std::to_string(CSATTN_CSAT_MAX_SUBSPACES));
    uint64_t sum = 0;
    for (uint32_t b = 0; b < m; ++b) {
        h->widths[b] = in.le(4, "subspace width");
        sum += h->widths[b];
    }
    if (sum != d)
        fail(CSATTN_ERR_CORRUPT, "subspace widths sum to " + std::to_string(sum) + ", expected " + std::to_string(d));
    h->m = m;
    h->centroids = c;
    h->list_capacity = cap;
    h->dim = d;
    h->prefill_len = prefill;
    h->score_bits = (flags & kHalf) ? 16 : 32;
    h->normalize_keys = (flags & kNormalized) ? 1 : 0;
}

void write_prefix(Writer& w, const csattn_csat_header* h, const float* centroids) {
    const bool half = h->score_bits == 16;
    w.bytes("CSAT", 4);
    w.u16(kVersion);
    w.u16(static_cast<uint16_t>((half ? kHalf : 0u) | (h->normalize_keys ? kNormalized : 0u)));
    w.u32(static_cast<uint32_t>(h->m));
    w.u32(static_cast<uint32_t>(h->centroids));
    w.u32(static_cast<uint32_t>(h->list_capacity));
    w.u32(static_cast<uint32_t>(h->dim));
    w.u64(h->prefill_len);
    for (uint64_t b = 0; b < h->m; ++b) w.u32(static_cast<uint32_t>(h->widths[b]));
    for (uint64_t i = 0; i < h->centroids * h->dim; ++i) w.value(centroids[i], half);
}

}  // namespace

namespace csa_host {
uint64_t csat_prefix(const csattn_csat_header* h, const float* centroids, uint8_t* out) {
    check_header(h);
    Writer w{out, out ? ~0ull : 0ull};
    write_prefix(w, h, centroids);
    return w.n;
}
}  // namespace csa_host

extern "C" {

uint16_t csattn_f32_to_f16(float value) { return to_half(value); }
float csattn_f16_to_f32(uint16_t bits) { return from_half(bits); }

csattn_status csattn_csat_read_header(const uint8_t* bytes, uint64_t n, csattn_csat_header* h) {
    return csa_host::guard([&] {
        Reader in{bytes, n};
        parse_header(in, h);
    });
}

csattn_status csattn_csat_footprint(const csattn_csat_header* h, const uint32_t* lens,
                                    uint64_t* header_bytes, uint64_t* centroid_bytes,
                                    uint64_t* entry_bytes) {
    return csa_host::guard([&] {
        check_header(h);
        const uint64_t sb = h->score_bits == 16 ? 2 : 4, T = h->m * h->centroids;
        uint64_t e = 0;
        for (uint64_t t = 0; t < T; ++t) e += static_cast<uint64_t>(lens[t]) * (4 + sb);
        *header_bytes = 4 + 2 + 2 + 4 + 4 + 4 + 4 + 8 + 4 * h->m + 4 * T;
        *centroid_bytes = sb * h->centroids * h->dim;
        *entry_bytes = e;
    });
}

csattn_status csattn_csat_encode(const csattn_csat_header* h, const float* centroids,
                                 const uint32_t* lens, const uint32_t* indices, const float* scores,
                                 uint64_t stride, uint8_t* out, uint64_t capacity, uint64_t* size) {
    return csa_host::guard([&] {
        check_header(h);
        const bool half = h->score_bits == 16;
        Writer w{out, capacity};
        write_prefix(w, h, centroids);
        const uint64_t T = h->m * h->centroids;
        for (uint64_t t = 0; t < T; ++t) {
            const uint32_t len = lens[t];
            if (len > stride) fail(CSATTN_ERR_PARAMETER, "CSAT encode: list longer than the stride");
            w.u32(len);
            for (uint32_t r = 0; r < len; ++r) w.u32(indices[t * stride + r]);
            for (uint32_t r = 0; r < len; ++r) w.value(scores[t * stride + r], half);
        }
        *size = w.n;
        if (out && w.n > capacity)
            fail(CSATTN_ERR_PARAMETER, "CSAT encode: output buffer holds " + std::to_string(capacity) +
                                           " bytes, image needs " + std::to_string(w.n));
    });
}

csattn_status csattn_csat_decode(const uint8_t* bytes, uint64_t n, csattn_csat_header* h,
                                 float* centroids, uint32_t* lens, uint32_t* indices,
                                 float* scores, uint64_t stride) {
    return csa_host::guard([&] {
        Reader in{bytes, n};
        parse_header(in, h);
        const bool half = h->score_bits == 16;
        if (stride < h->list_capacity) fail(CSATTN_ERR_PARAMETER, "CSAT decode: stride below the list capacity");
        for (uint64_t i = 0; i < h->centroids * h->dim; ++i) centroids[i] = in.value(half, "centroid row");
        const uint64_t T = h->m * h->centroids;
        std::vector<uint32_t> seen;
        for (uint64_t t = 0; t < T; ++t) {
            const uint32_t len = static_cast<uint32_t>(in.le(4, "list length"));
            if (len > h->list_capacity)
                fail(CSATTN_ERR_CORRUPT, "table " + std::to_string(t) + " holds " + std::to_string(len) +
                                             " entries, capacity " + std::to_string(h->list_capacity));
            uint32_t* ix = indices + t * stride;
            float* sc = scores + t * stride;
            for (uint32_t r = 0; r < len; ++r) ix[r] = static_cast<uint32_t>(in.le(4, "list index"));
            for (uint32_t r = 0; r < len; ++r) sc[r] = in.value(half, "list score");
            for (uint32_t r = 1; r < len; ++r)
                if (sc[r] > sc[r - 1])
                    fail(CSATTN_ERR_CORRUPT, "table " + std::to_string(t) + " scores are not sorted descending");
            seen.assign(ix, ix + len);
            std::sort(seen.begin(), seen.end());
            if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
                fail(CSATTN_ERR_CORRUPT, "table " + std::to_string(t) + " repeats a key index");
            lens[t] = len;
        }
        if (in.pos != n) fail(CSATTN_ERR_CORRUPT, "unexpected trailing bytes at offset " + std::to_string(in.pos));
    });
}

}  // extern "C"
