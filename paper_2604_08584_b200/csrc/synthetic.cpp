// synthetic.cpp — make_synthetic (synthetic.cpp:18-74 in the reference):
// the planted-cluster Q/K/V workload the measurement configs are defined on
// (SURVEY.md §8(d)). Host-side input generation, bit-identical to the
// reference: mt19937_64 from the standard library, the reference's
// hand-rolled draws (util.hpp:28-52) and l2_normalize (core.cpp:109-116).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "csattn_b200.h"

namespace {

struct Draws {
    std::mt19937_64 g;
    double spare = 0.0;
    bool have = false;
    explicit Draws(uint64_t seed) : g(seed) {}
    double unit() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
    uint64_t index(uint64_t n) {
        return static_cast<uint64_t>((static_cast<unsigned __int128>(g()) * n) >> 64);
    }
    double normal() {
        if (have) {
            have = false;
            return spare;
        }
        double u1 = unit();
        const double u2 = unit();
        while (u1 <= 0.0) u1 = unit();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(a);
        have = true;
        return r * std::cos(a);
    }
};

uint64_t mix(uint64_t seed, uint64_t salt) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

bool normalize(float* v, size_t n) {
    double n2 = 0.0;
    for (size_t i = 0; i < n; ++i) n2 += static_cast<double>(v[i]) * static_cast<double>(v[i]);
    if (n2 == 0.0) return true;
    const double inv = 1.0 / std::sqrt(n2);
    for (size_t i = 0; i < n; ++i) v[i] = static_cast<float>(v[i] * inv);
    return false;
}

}  // namespace

extern "C" csattn_status csattn_make_synthetic(const csattn_synthetic_spec* spec, float* queries,
                                               float* keys, float* values) {
    if (spec->rows == 0 || spec->dim == 0 || spec->clusters == 0) return CSATTN_ERR_PARAMETER;
    if (spec->dwell == 0) return CSATTN_ERR_PARAMETER;
    if (!(spec->plant_fraction >= 0.0 && spec->plant_fraction <= 1.0)) return CSATTN_ERR_PARAMETER;
    const uint64_t d = spec->dim;
    // salts of the three independent streams (directions, rows, block map)
    const uint64_t kDir = 0x64697273, kRow = 0x726f7773, kBlock = 0x626c6b73;
    Draws dr(mix(spec->seed, kDir));
    std::vector<float> dirs(spec->clusters * d);
    for (uint64_t c = 0; c < spec->clusters; ++c) {
        float* row = dirs.data() + c * d;
        do {
            for (uint64_t t = 0; t < d; ++t) row[t] = static_cast<float>(dr.normal());
        } while (normalize(row, d));
    }
    Draws rng(mix(spec->seed, kRow));
    for (uint64_t i = 0; i < spec->rows; ++i) {
        const uint64_t block = i / spec->dwell;
        const uint64_t qc = mix(spec->seed, kBlock + block) % spec->clusters;
        const float* qd = dirs.data() + qc * d;
        float* q = queries + i * d;
        for (uint64_t t = 0; t < d; ++t)
            q[t] = qd[t] + static_cast<float>(spec->query_noise * rng.normal());
        float* k = keys + i * d;
        if (rng.unit() < spec->plant_fraction) {
            const float* kd = dirs.data() + rng.index(spec->clusters) * d;
            for (uint64_t t = 0; t < d; ++t)
                k[t] = static_cast<float>(spec->plant_scale) * kd[t] + static_cast<float>(rng.normal());
        } else {
            for (uint64_t t = 0; t < d; ++t) k[t] = static_cast<float>(rng.normal());
        }
        float* v = values + i * d;
        for (uint64_t t = 0; t < d; ++t) v[t] = static_cast<float>(rng.normal());
    }
    return CSATTN_OK;
}
