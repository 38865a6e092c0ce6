// meshforge::CounterRng for the B200 library: draw i is a pure function of
// (seed, i) - the splitmix64 finaliser applied to mix(seed) ^ mix(i + c), as
// specified by proj/include/meshforge/core/rng.h:10-29 (same streams, so the
// reference's fixtures and ours generate identical inputs).
#pragma once

#include <cstdint>

namespace meshforge {

namespace rng_detail {
constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr std::uint64_t kMulA = 0xBF58476D1CE4E5B9ull;
constexpr std::uint64_t kMulB = 0x94D049BB133111EBull;
constexpr std::uint64_t kStream = 0x632BE59BD9B4E019ull;
constexpr std::uint64_t splitmix64(std::uint64_t z) {
  return [](std::uint64_t a) {
    a = (a ^ (a >> 30)) * kMulA;
    a = (a ^ (a >> 27)) * kMulB;
    return a ^ (a >> 31);
  }(z + kGolden);
}
}  // namespace rng_detail

struct CounterRng {
  std::uint64_t seed = 0;

  explicit CounterRng(std::uint64_t s = 0) : seed(s) {}

  static std::uint64_t mix(std::uint64_t z) { return rng_detail::splitmix64(z); }
  std::uint64_t bits(std::uint64_t i) const {
    return rng_detail::splitmix64(rng_detail::splitmix64(seed) ^ rng_detail::splitmix64(i + rng_detail::kStream));
  }
  // uniform double in [0, 1) from the top 53 bits
  double uniform(std::uint64_t i) const { return static_cast<double>(bits(i) >> 11) * 0x1.0p-53; }
  std::uint64_t below(std::uint64_t i, std::uint64_t n) const { return bits(i) % n; }
};

}  // namespace meshforge
