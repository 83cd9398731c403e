#pragma once
// Host twin of the device fill kernel (kernels/fill.cu): element (r, c) of a
// block at (row0, col0) in a matrix with `total_cols` columns is draw
// (row0+r)*total_cols + col0+c of Rng(seed), mapped to float(2u - 1).
#include <cstdint>

#include "poas/rng.hpp"

namespace poas_b200 {

inline float uniform_pm1_at(std::uint64_t seed, std::uint64_t index) {
  const std::uint64_t z = poas::splitmix64_at(seed, index);
  const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
  return static_cast<float>(2.0 * u - 1.0);
}

inline void fill_uniform_host(float* dst, std::int64_t ld, std::int64_t rows, std::int64_t cols,
                              std::int64_t row0, std::int64_t col0, std::int64_t total_cols,
                              std::uint64_t seed) {
#pragma omp parallel for schedule(static)
  for (std::int64_t r = 0; r < rows; ++r) {
    const std::uint64_t base = static_cast<std::uint64_t>((row0 + r) * total_cols + col0);
    float* out = dst + r * ld;
    for (std::int64_t c = 0; c < cols; ++c) out[c] = uniform_pm1_at(seed, base + c);
  }
}

}  // namespace poas_b200
