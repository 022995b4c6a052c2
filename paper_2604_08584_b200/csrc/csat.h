// csat.h — host CSAT v1 pieces used by the session calls in capi.cpp.
#pragma once
#include <cstdint>

#include "csattn_b200.h"

namespace csa_host {
// Bytes before the first table (fixed header, widths, centroid rows); writes
// them to out when out != nullptr (out must hold the returned size).
uint64_t csat_prefix(const csattn_csat_header* h, const float* centroids, uint8_t* out);
}  // namespace csa_host
