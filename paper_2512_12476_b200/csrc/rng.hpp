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

#ifndef __CUDA_ARCH__
// Exact 64-bit remainder by a precomputed 128-bit reciprocal (Lemire,
// Kaser & Kurz, "Faster remainder by direct computation", 2019): for every
// 64-bit a and d >= 1, fastmod(a) == a % d. Replaces the hardware divide in
// the host-side candidate generator (thousands of bounded() draws per
// candidate); results are identical by construction and checked in
// tests/test_host_units.py.
struct FastModTable {
  static constexpr int kMax = 1024;
  unsigned __int128 m[kMax + 1];
  FastModTable() {
    m[0] = 0;
    for (int d = 1; d <= kMax; ++d) m[d] = ~static_cast<unsigned __int128>(0) / d + 1;
  }
};
inline const FastModTable& fastmod_table() {
  static const FastModTable t;
  return t;
}
inline uint64_t fastmod_u64(uint64_t a, unsigned __int128 M, uint64_t d) {
  const unsigned __int128 low = M * a;
  unsigned __int128 bottom = (low & 0xFFFFFFFFFFFFFFFFull) * d;
  bottom >>= 64;
  const unsigned __int128 top = (low >> 64) * d;
  return static_cast<uint64_t>((bottom + top) >> 64);
}
#endif

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
  HPG_HD uint64_t bounded(uint64_t n) {
#ifndef __CUDA_ARCH__
    if (n <= FastModTable::kMax) return fastmod_u64(next(), fastmod_table().m[n], n);
#endif
    return next() % n;
  }
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
