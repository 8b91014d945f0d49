// xoshiro256 jump-ahead by an arbitrary count (host side): the transition is
// linear over GF(2); its characteristic polynomial p (degree 256) comes from
// Berlekamp-Massey on one output bit, and advancing a state by D steps is
// q(T) applied to it, q = x^D mod p (the construction behind xoshiro's own
// jump()). Used to give each lane of a device GA init chunk its candidate's
// start state (ga_kernel.cuh ga_init_chunk).
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "rng.hpp"

namespace hpg {

using Poly256 = std::array<uint64_t, 4>;  // coefficients of x^0..x^255

namespace jump_detail {

inline uint64_t bit(const uint64_t* w, int i) { return (w[i >> 6] >> (i & 63)) & 1u; }

// low 256 coefficients of p (p = x^256 + ...)
inline const Poly256& charpoly() {
  static const Poly256 p = [] {
    // 512 terms of one output bit of the state sequence
    Rng r(0x9E3779B97F4A7C15ull);
    std::vector<uint8_t> sq(512);
    for (int i = 0; i < 512; ++i) {
      sq[i] = static_cast<uint8_t>(r.s[0] & 1u);
      r.next();
    }
    // Berlekamp-Massey over GF(2): connection polynomial C (C[0] = 1)
    std::vector<uint8_t> C(513, 0), B(513, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < 512; ++n) {
      uint8_t d = sq[n];
      for (int i = 1; i <= L; ++i) d ^= C[i] & sq[n - i];
      if (!d) {
        ++m;
        continue;
      }
      T = C;
      for (int i = 0; i + m <= 512; ++i) C[i + m] ^= B[i];
      if (2 * L <= n) {
        L = n + 1 - L;
        B = T;
        m = 1;
      } else {
        ++m;
      }
    }
    // the characteristic polynomial is the reciprocal of C: p_i = C[L - i]
    Poly256 out{0, 0, 0, 0};
    if (L != 256) return out;  // never: xoshiro256's polynomial is primitive
    for (int i = 0; i < 256; ++i)
      if (C[256 - i]) out[i >> 6] |= 1ull << (i & 63);
    return out;
  }();
  return p;
}

// a * b mod p
// x^(256 + 8k) * v mod p for byte position k of the high half and byte
// value v: the reduction becomes 32 table lookups (256 KB, built once)
inline const std::vector<Poly256>& reduce_table() {
  static const std::vector<Poly256> t = [] {
    const Poly256& p = charpoly();
    // x^(256 + j) mod p for j = 0..255, by repeated multiplication by x
    std::vector<Poly256> xj(256);
    Poly256 cur = p;  // x^256 = p (mod p) with the x^256 term dropped
    for (int j = 0; j < 256; ++j) {
      xj[j] = cur;
      const uint64_t top = cur[3] >> 63;
      for (int k = 3; k > 0; --k) cur[k] = (cur[k] << 1) | (cur[k - 1] >> 63);
      cur[0] <<= 1;
      if (top)
        for (int k = 0; k < 4; ++k) cur[k] ^= p[k];
    }
    std::vector<Poly256> out(32 * 256, Poly256{0, 0, 0, 0});
    for (int k = 0; k < 32; ++k)
      for (int v = 1; v < 256; ++v) {
        const Poly256& lo = out[k * 256 + (v & (v - 1))];
        const Poly256& x = xj[8 * k + __builtin_ctz(static_cast<unsigned>(v))];
        for (int w = 0; w < 4; ++w) out[k * 256 + v][w] = lo[w] ^ x[w];
      }
    return out;
  }();
  return t;
}

// a * b mod p over GF(2): 4-bit windowed carry-less product, then the high
// 256 bits folded back through reduce_table()
inline Poly256 mulmod(const Poly256& a, const Poly256& b) {
  uint64_t win[16][5];
  for (int w = 0; w < 5; ++w) win[0][w] = 0;
  for (int v = 1; v < 16; ++v) {
    // win[v] = b * v: b shifted by each set bit of v
    const int bitpos = 31 - __builtin_clz(static_cast<unsigned>(v));
    const int rest = v ^ (1 << bitpos);
    for (int w = 0; w < 5; ++w) {
      const uint64_t bw = w < 4 ? b[w] : 0;
      const uint64_t bl = w > 0 ? b[w - 1] : 0;
      const uint64_t sh = bitpos ? (bw << bitpos) | (bl >> (64 - bitpos)) : bw;
      win[v][w] = win[rest][w] ^ sh;
    }
  }
  uint64_t prod[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < 64; ++i) {
    const unsigned nib = static_cast<unsigned>(a[i >> 4] >> (4 * (i & 15))) & 15u;
    if (!nib) continue;
    const int w0 = (4 * i) >> 6, s = (4 * i) & 63;
    for (int w = 0; w < 5; ++w) {
      prod[w0 + w] ^= win[nib][w] << s;
      if (s) prod[w0 + w + 1] ^= win[nib][w] >> (64 - s);
    }
  }
  const std::vector<Poly256>& t = reduce_table();
  Poly256 r{prod[0], prod[1], prod[2], prod[3]};
  for (int k = 0; k < 32; ++k) {
    const unsigned v = static_cast<unsigned>(prod[4 + (k >> 3)] >> (8 * (k & 7))) & 255u;
    if (!v) continue;
    const Poly256& x = t[k * 256 + v];
    for (int w = 0; w < 4; ++w) r[w] ^= x[w];
  }
  return r;
}

}  // namespace jump_detail

// x^D mod p
inline Poly256 jump_poly(uint64_t D) {
  Poly256 r{1, 0, 0, 0}, base{2, 0, 0, 0};  // 1 and x
  while (D) {
    if (D & 1) r = jump_detail::mulmod(r, base);
    base = jump_detail::mulmod(base, base);
    D >>= 1;
  }
  return r;
}

// the state advanced by q(T) (q = jump_poly(D) advances D steps)
HPG_HD void rng_apply_jump(Rng& r, const uint64_t* q) {
  uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int i = 0; i < 256; ++i) {
    if ((q[i >> 6] >> (i & 63)) & 1u) {
      a0 ^= r.s[0];
      a1 ^= r.s[1];
      a2 ^= r.s[2];
      a3 ^= r.s[3];
    }
    r.next();
  }
  r.s[0] = a0;
  r.s[1] = a1;
  r.s[2] = a2;
  r.s[3] = a3;
}

// x^(L*D) mod p for L = 1..n (cached per D, process-wide). Entries are
// immutable once published: a caller keeps its table alive through the
// shared_ptr even if a later call for the same D publishes a longer one.
using JumpTable = std::shared_ptr<const std::vector<Poly256>>;
inline JumpTable jump_table(uint64_t D, int n) {
  static std::mutex m;
  static std::map<uint64_t, JumpTable> cache;
  {
    std::lock_guard<std::mutex> lk(m);
    auto it = cache.find(D);
    if (it != cache.end() && static_cast<int>(it->second->size()) >= n) return it->second;
  }
  // built outside the lock so callers can fill several tables in parallel
  auto v = std::make_shared<std::vector<Poly256>>();
  const Poly256 q = jump_poly(D);
  v->push_back(q);
  while (static_cast<int>(v->size()) < n) v->push_back(jump_detail::mulmod(v->back(), q));
  std::lock_guard<std::mutex> lk(m);
  JumpTable& slot = cache[D];
  if (!slot || slot->size() < v->size()) slot = std::move(v);
  return slot;
}

}  // namespace hpg
