#pragma once
// Counter-based splitmix64 stream with Box-Muller normals. Bit-compatible
// with the reference generator (proj/include/poas/rng.hpp:13-56) because
// seeded input matrices and golden plans depend on it; the device fill
// kernel (kernels/fill.cu) evaluates the same counter directly.

#include <cmath>
#include <cstdint>
#include <string_view>

namespace poas {

inline constexpr std::uint64_t kSplitmixGamma = 0x9e3779b97f4a7c15ULL;

// Draw number `index` (0-based) of a stream started at `seed`.
constexpr std::uint64_t splitmix64_at(std::uint64_t seed, std::uint64_t index) {
  std::uint64_t z = seed + (index + 1) * kSplitmixGamma;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : state_(seed) {}

  std::uint64_t next_u64() {
    const std::uint64_t out = splitmix64_at(state_, 0);
    state_ += kSplitmixGamma;
    return out;
  }

  // [0, 1) with 53 random bits.
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

  double next_range(double lo, double hi) { return lo + (hi - lo) * next_unit(); }

  // Inclusive integer range.
  std::int64_t next_int(std::int64_t lo, std::int64_t hi) {
    const std::uint64_t span = static_cast<std::uint64_t>(hi - lo + 1);
    return lo + static_cast<std::int64_t>(next_u64() % span);
  }

  // One standard normal per call (no cached partner).
  double next_gaussian() {
    const double u1 = 1.0 - next_unit();
    const double u2 = next_unit();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
  }

  // Independent stream per named consumer: FNV-1a of the name folded into
  // the master seed. The 19-digit offset is the reference's constant.
  static Rng for_stream(std::uint64_t master_seed, std::string_view name) {
    return Rng(master_seed ^ name_hash(name));
  }

  static std::uint64_t name_hash(std::string_view name) {
    std::uint64_t h = 1469598103934665603ULL;
    for (const char ch : name) {
      h ^= static_cast<std::uint64_t>(static_cast<unsigned char>(ch));
      h *= 1099511628211ULL;
    }
    return h;
  }

  std::uint64_t state() const { return state_; }

 private:
  std::uint64_t state_;
};

}  // namespace poas
