// Host Gaussian streams. xoshiro256++ (Blackman & Vigna, 2019) seeded through
// splitmix64; normals by Box-Muller (both published algorithms).
#include "grf/random.hpp"

#include <cmath>
#include <numbers>

namespace grf {

namespace {

inline std::uint64_t rotl64(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

inline std::uint64_t splitmix64_next(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

Xoshiro256Stream::Xoshiro256Stream(std::uint64_t seed, std::uint64_t substream) : seed_(seed) {
  // Two splitmix64 passes keep (seed, substream) -> state injective in practice.
  std::uint64_t mix = seed;
  const std::uint64_t salt = splitmix64_next(mix) ^ (substream * 0xD1342543DE82EF95ull + 0x632BE59BD9B4E019ull);
  std::uint64_t st = salt;
  for (auto& w : s_) w = splitmix64_next(st);
  if ((s_[0] | s_[1] | s_[2] | s_[3]) == 0) s_[0] = 1;
}

std::uint64_t Xoshiro256Stream::next_u64() {
  const std::uint64_t out = rotl64(s_[0] + s_[3], 23) + s_[0];
  const std::uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl64(s_[3], 45);
  return out;
}

double Xoshiro256Stream::uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

double Xoshiro256Stream::draw() {
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  const double u1 = 1.0 - uniform01();  // (0, 1]
  const double u2 = uniform01();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 2.0 * std::numbers::pi * u2;
  spare_ = r * std::sin(a);
  have_spare_ = true;
  return r * std::cos(a);
}

}  // namespace grf
