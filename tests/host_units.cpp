// Host-only unit checks of engine building blocks that have no GPU
// dependency (compiled and run by tests/test_host_units.py):
//   * fastmod_u64 == the hardware remainder for random and edge-case inputs
//   * Rng streams equal the reference's documented xoshiro256** / splitmix64
//     (first draws of Rng(42) recorded from the compiled reference)
//   * jump-ahead polynomials (rng_jump.hpp) == stepping the stream D times
#include <cinttypes>
#include <cstdio>
#include <cstdlib>

#include "../paper_2512_12476_b200/csrc/rng.hpp"
#include "../paper_2512_12476_b200/csrc/rng_jump.hpp"

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
  // jump-ahead: x^D mod p applied to a state == D draws; table x^(L*D)
  uint64_t jbad = 0;
  Rng jr(777);
  for (int trial = 0; trial < 64; ++trial) {
    const uint64_t D = trial < 4 ? static_cast<uint64_t>(trial) : jr.next() % 3000;
    Rng a0(jr.next()), b0 = a0;
    for (uint64_t k = 0; k < D; ++k) a0.next();
    const Poly256 q = jump_poly(D);
    rng_apply_jump(b0, q.data());
    for (int w = 0; w < 4; ++w) jbad += a0.s[w] != b0.s[w];
    const JumpTable tbp = jump_table(D, 31);
    const std::vector<Poly256>& tb = *tbp;
    for (int L : {1, 7, 31}) {
      Rng c0(jr.next()), d0 = c0;
      for (uint64_t k = 0; k < D * L; ++k) c0.next();
      rng_apply_jump(d0, tb[L - 1].data());
      for (int w = 0; w < 4; ++w) jbad += c0.s[w] != d0.s[w];
    }
  }
  std::printf("jump mismatches %" PRIu64 "\n", jbad);
  return bad == 0 && jbad == 0 ? 0 : 1;
}
