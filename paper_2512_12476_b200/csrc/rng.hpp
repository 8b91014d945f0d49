// Deterministic streams, bit-identical to the reference's Rng
// (proj/include/hetplan/rng.hpp:10-65): splitmix64 finalizer for seeding and
// forking, xoshiro256** for draws, bounded(n) = next() % n (modulo bias kept
// on purpose), uniform() = (next() >> 11) * 2^-53, descending Fisher-Yates.
// Usable on host and device; the device path replaces the 64-bit modulo by a
// multiply-high with a tabulated reciprocal (exact, see bounded_fast).
#pragma once

#include <cstdint>

#include "common.hpp"

namespace hpg {

HPG_HD uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct Rng {
  uint64_t seed;
  uint64_t s[4];

  HPG_HD Rng() : seed(0), s{0, 0, 0, 0} {}
  HPG_HD explicit Rng(uint64_t sd) : seed(sd) {
    uint64_t v = sd;
    for (int i = 0; i < 4; ++i) {
      s[i] = mix64(v);
      v = s[i];
    }
  }
  HPG_HD static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  HPG_HD uint64_t next() {
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  HPG_HD uint64_t bounded(uint64_t n) { return next() % n; }
  HPG_HD double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  HPG_HD double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  // Rng::fork (rng.hpp:64): derived from the original seed, not the state.
  HPG_HD Rng fork(uint64_t salt) const { return Rng(mix64(seed ^ mix64(salt))); }
  template <typename T>
  HPG_HD void shuffle(T* v, int n) {
    for (int i = n; i > 1; --i) {
      const int j = static_cast<int>(bounded(static_cast<uint64_t>(i)));
      T tmp = v[i - 1];
      v[i - 1] = v[j];
      v[j] = tmp;
    }
  }
};

}  // namespace hpg
