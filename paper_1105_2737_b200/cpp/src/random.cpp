// Host Gaussian streams of the drop-in.
//
// Xoshiro256Stream reproduces the reference's seeded stream bit for bit
// (/root/reference/proj/core/src/random.cpp:56-108), so reference programs
// that seed a Xoshiro256Stream and call the stream overload of synthesize get
// the reference's noise:
//   * state: four splitmix64 outputs (Steele, Lea & Flood 2014) from the single
//     word seed XOR golden-gamma * (substream + 1); an all-zero state is fixed
//     up to state[0] = 1;
//   * generator: xoshiro256++ (Blackman & Vigna 2019), uniforms = top 53 bits;
//   * normals: the Marsaglia–Tsang (2000) 256-layer ziggurat over a signed
//     64-bit draw (layer = low 8 bits, magnitude vs the layer's 2^63-scaled
//     acceptance bound), with Marsaglia's exponential tail beyond r.
// The layer tables are rebuilt here from the two published constants (r, v)
// by the standard top-down recursion, in the same IEEE operation order, so
// every table entry — and hence every draw — matches.
#include "grf/random.hpp"

#include <cmath>
#include <cstdlib>

namespace grf {

namespace {

constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;

std::uint64_t splitmix_step(std::uint64_t& s) {
  s += kGolden;
  std::uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

constexpr std::uint64_t rot(std::uint64_t v, unsigned r) { return (v << r) | (v >> (64u - r)); }

// Ziggurat layers: accept[i] = |draw| bound for the fast path, scale[i] =
// x per unit of draw, pdf[i] = exp(-x_i^2/2) at the layer's outer edge.
class Layers {
 public:
  static constexpr double r = 3.6541528853610088;     // start of the tail
  static constexpr double v = 4.928673233974655e-3;   // area of every layer
  std::uint64_t accept[256];
  double scale[256];
  double pdf[256];

  Layers() {
    const double two63 = 9223372036854775808.0;
    double x = r;      // current layer edge, walking inwards
    double outer = r;  // edge of the layer above
    const double base = v / std::exp(-0.5 * x * x);  // width of the base strip incl. tail
    accept[0] = static_cast<std::uint64_t>((x / base) * two63);
    accept[1] = 0;
    scale[0] = base / two63;
    scale[255] = x / two63;
    pdf[0] = 1.0;
    pdf[255] = std::exp(-0.5 * x * x);
    for (int layer = 254; layer >= 1; --layer) {
      x = std::sqrt(-2.0 * std::log(v / x + std::exp(-0.5 * x * x)));
      accept[layer + 1] = static_cast<std::uint64_t>((x / outer) * two63);
      outer = x;
      pdf[layer] = std::exp(-0.5 * x * x);
      scale[layer] = x / two63;
    }
  }
};

const Layers& layers() {
  static const Layers t;
  return t;
}

}  // namespace

Xoshiro256Stream::Xoshiro256Stream(std::uint64_t seed, std::uint64_t substream) : seed_(seed) {
  std::uint64_t mix = seed ^ (kGolden * (substream + 1));
  for (std::uint64_t& w : s_) w = splitmix_step(mix);
  if ((s_[0] | s_[1] | s_[2] | s_[3]) == 0) s_[0] = 1;
  (void)layers();  // tables ready before the first draw
}

std::uint64_t Xoshiro256Stream::next_u64() {
  std::uint64_t* const s = s_;
  const std::uint64_t out = rot(s[0] + s[3], 23) + s[0];
  const std::uint64_t shifted = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= shifted;
  s[3] = rot(s[3], 45);
  return out;
}

double Xoshiro256Stream::uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

double Xoshiro256Stream::draw() {
  const Layers& L = layers();
  while (true) {
    const auto w = static_cast<std::int64_t>(next_u64());
    if (w == INT64_MIN) continue;  // no representable magnitude
    const unsigned layer = static_cast<unsigned>(w & 0xff);
    const double x = static_cast<double>(w) * L.scale[layer];
    if (static_cast<std::uint64_t>(std::llabs(w)) < L.accept[layer]) return x;
    if (layer == 0) {
      // tail |x| > r: x = r + E1/r with E1, E2 exponential, accepted when 2 E2 >= (E1/r)^2
      double e1, e2;
      do {
        double u = uniform01();
        while (u == 0.0) u = uniform01();
        double u2 = uniform01();
        while (u2 == 0.0) u2 = uniform01();
        e1 = -std::log(u) / Layers::r;
        e2 = -std::log(u2);
      } while (e2 + e2 < e1 * e1);
      return w > 0 ? Layers::r + e1 : -(Layers::r + e1);
    }
    // wedge between layers: accept under the density
    if (L.pdf[layer] + uniform01() * (L.pdf[layer - 1] - L.pdf[layer]) < std::exp(-0.5 * x * x)) return x;
  }
}

}  // namespace grf
