// Host-only unit checks of engine building blocks that have no GPU
// dependency (compiled and run by tests/test_host_units.py):
//   * fastmod_u64 == the hardware remainder for random and edge-case inputs
//   * Rng streams equal the reference's documented xoshiro256** / splitmix64
//     (first draws of Rng(42) recorded from the compiled reference)
#include <cinttypes>
#include <cstdio>
#include <cstdlib>

#include "../paper_2512_12476_b200/csrc/rng.hpp"

int main(int argc, char** argv) {
  using namespace hpg;
  const auto& t = fastmod_table();
  Rng r(12345);
  uint64_t bad = 0, checked = 0;
  const uint64_t edge[] = {0ull, 1ull, 2ull, 0x7fffffffffffffffull, 0x8000000000000000ull,
                           0xffffffffffffffffull, 0xfffffffffffffffeull, 1ull << 53};
  for (int d = 1; d <= FastModTable::kMax; ++d) {
    for (uint64_t a : edge) {
      ++checked;
      if (fastmod_u64(a, t.m[d], d) != a % d) ++bad;
    }
    for (int k = 0; k < 20000; ++k) {
      const uint64_t a = r.next();
      ++checked;
      if (fastmod_u64(a, t.m[d], d) != a % d) ++bad;
      const uint64_t b = (a % (4ull * d)) + (k & 1 ? 0ull : ~0ull - 4ull * d);
      ++checked;
      if (fastmod_u64(b, t.m[d], d) != b % d) ++bad;
    }
  }
  std::printf("fastmod checked %" PRIu64 " mismatches %" PRIu64 "\n", checked, bad);
  // stream pin: Rng(seed).next() x3 and fork
  const uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 42;
  Rng s(seed);
  // draw into named values: argument evaluation order is unspecified
  const uint64_t a = s.next(), b = s.next(), c = s.next();
  std::printf("draws %" PRIu64 " %" PRIu64 " %" PRIu64 "\n", a, b, c);
  Rng f = Rng(seed).fork(7);
  const uint64_t x = f.next();
  const uint64_t y = f.bounded(100);
  const double z = f.uniform();
  std::printf("fork7 %" PRIu64 " bounded100 %" PRIu64 " uniform %.17g\n", x, y, z);
  return bad == 0 ? 0 : 1;
}
