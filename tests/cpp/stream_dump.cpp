// Prints n normals and n raw words of the drop-in's grf::Xoshiro256Stream(seed,
// substream) as hex doubles / decimal words (tests/test_streams.py compares
// them with the reference's own stream).
#include <cinttypes>
#include <cstdio>
#include <cstdlib>

#include "grf/random.hpp"

int main(int argc, char** argv) {
  if (argc != 4) {
    std::fprintf(stderr, "usage: stream_dump seed substream n\n");
    return 2;
  }
  const std::uint64_t seed = std::strtoull(argv[1], nullptr, 10), sub = std::strtoull(argv[2], nullptr, 10);
  const std::uint64_t n = std::strtoull(argv[3], nullptr, 10);
  grf::Xoshiro256Stream a(seed, sub), b(seed, sub);
  for (std::uint64_t i = 0; i < n; ++i) std::printf("%a\n", a.next());
  for (std::uint64_t i = 0; i < n; ++i) std::printf("%" PRIu64 "\n", b.next_u64());
  if (a.draws_consumed() != n) return 1;
  return 0;
}
