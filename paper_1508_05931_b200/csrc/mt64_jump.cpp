// mt19937_64 jump-ahead over GF(2), host side; see mt64_jump.h.
#include "mt64_jump.h"

#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <utility>

namespace gscan {
namespace mt64 {
namespace {

using Poly = std::vector<uint64_t>;  // bit i = coefficient of t^i

inline bool getb(const Poly& p, int i) { return (p[i >> 6] >> (i & 63)) & 1u; }

// phi via Berlekamp-Massey over GF(2) on bit 0 of 2 * kDeg engine outputs.
// The output bit is a non-zero linear functional of the state and phi is
// primitive, so the sequence's minimal polynomial is phi itself.
Poly charpoly() {
  const int n = 2 * kDeg;
  std::mt19937_64 eng(5489u);
  std::vector<uint8_t> s(n);
  for (int i = 0; i < n; ++i) s[i] = (uint8_t)(eng() & 1u);
  const int W = (n + 64) / 64 + 1;
  Poly C(W, 0), B(W, 0), T(W, 0);
  C[0] = B[0] = 1;
  int L = 0, m = -1;
  for (int i = 0; i < n; ++i) {
    uint32_t d = s[i];  // s_i + sum_{k=1..L} c_k s_{i-k}
    for (int k = 1; k <= L; ++k) d ^= (uint32_t)(getb(C, k) & s[i - k]);
    if (!d) continue;
    T = C;
    const int sh = i - m;  // C ^= B << sh
    const int ws = sh >> 6, bs = sh & 63;
    for (int w = W - 1; w >= ws; --w) {
      uint64_t v = B[w - ws] << bs;
      if (bs && w - ws - 1 >= 0) v |= B[w - ws - 1] >> (64 - bs);
      C[w] ^= v;
    }
    if (2 * L <= i) {
      L = i + 1 - L;
      m = i;
      B = T;
    }
  }
  // connection polynomial C(x) = 1 + c1 x + ... + cL x^L; the characteristic
  // polynomial is its reciprocal: phi(t) = t^L + c1 t^(L-1) + ... + cL
  Poly phi(kWords, 0);
  for (int k = 0; k <= L; ++k)
    if (getb(C, k)) phi[(L - k) >> 6] |= 1ull << ((L - k) & 63);
  return phi;  // L == kDeg for mt19937_64
}

const Poly& phi_poly() {
  static const Poly p = charpoly();
  return p;
}

// a * a mod phi (a of degree < kDeg)
Poly sqr_mod(const Poly& a) {
  const Poly& phi = phi_poly();
  Poly r(2 * kWords + 1, 0);
  for (int i = 0; i < kDeg; ++i)
    if (getb(a, i)) r[(2 * i) >> 6] |= 1ull << ((2 * i) & 63);
  // reduce: for every set bit at degree d >= kDeg, add phi * t^(d - kDeg)
  for (int d = 2 * kDeg - 2; d >= kDeg; --d) {
    if (!((r[d >> 6] >> (d & 63)) & 1u)) continue;
    const int sh = d - kDeg, ws = sh >> 6, bs = sh & 63;
    for (int w = 0; w < kWords; ++w) {
      if (!phi[w]) continue;
      r[w + ws] ^= phi[w] << bs;
      if (bs) r[w + ws + 1] ^= phi[w] >> (64 - bs);
    }
  }
  r.resize(kWords);
  return r;
}

Poly mul_t_mod(const Poly& a) {  // a * t mod phi
  const Poly& phi = phi_poly();
  Poly r(kWords + 1, 0);
  for (int w = kWords - 1; w >= 0; --w) {
    r[w + 1] |= a[w] >> 63;
    r[w] |= a[w] << 1;
  }
  if ((r[kDeg >> 6] >> (kDeg & 63)) & 1u)
    for (int w = 0; w < kWords; ++w) r[w] ^= phi[w];
  r.resize(kWords);
  return r;
}

// t^e mod phi by left-to-right square-and-multiply
Poly pow_t(uint64_t e) {
  Poly r(kWords, 0);
  r[0] = 1;
  for (int b = 63; b >= 0; --b) {
    r = sqr_mod(r);
    if ((e >> b) & 1u) r = mul_t_mod(r);
  }
  return r;
}

inline uint64_t twist(uint64_t a, uint64_t b) {
  const uint64_t y = (a & kUpper) | (b & kLower);
  return (y >> 1) ^ ((b & 1u) ? kMatrixA : 0ull);
}

}  // namespace

void seed_state(uint64_t seed, uint64_t* st) {
  st[0] = seed;
  for (int i = 1; i < kN; ++i) st[i] = 6364136223846793005ull * (st[i - 1] ^ (st[i - 1] >> 62)) + (uint64_t)i;
}

const std::vector<uint64_t>& jump_table(uint64_t L, int nb) {
  static std::mutex mu;
  static std::map<std::pair<uint64_t, int>, std::vector<uint64_t>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({L, nb});
  if (it != cache.end()) return it->second;
  std::vector<uint64_t> tab((size_t)nb * kWords);
  Poly g = pow_t(L);
  for (int b = 0; b < nb; ++b) {
    std::memcpy(&tab[(size_t)b * kWords], g.data(), kWords * 8);
    if (b + 1 < nb) g = sqr_mod(g);
  }
  return cache.emplace(std::make_pair(L, nb), std::move(tab)).first->second;
}

void apply_jump_host(const uint64_t* g, uint64_t* state) {
  std::vector<uint64_t> x(kDeg + 2 * kN);
  for (int k = 0; k < kN; ++k) x[k] = state[k];
  for (int i = 0; i + kN < (int)x.size(); ++i) x[i + kN] = x[i + kM] ^ twist(x[i], x[i + 1]);
  uint64_t out[kN] = {};
  for (int i = 0; i < kDeg; ++i)
    if ((g[i >> 6] >> (i & 63)) & 1u)
      for (int k = 0; k < kN; ++k) out[k] ^= x[i + k];
  std::memcpy(state, out, sizeof(out));
}

}  // namespace mt64
}  // namespace gscan

// Host self-check of the jump machinery (CPU tests): the state after
// `blocks` * L words (L = 2^20, jumps by the table's powers of two) must
// reproduce the next 312 outputs of a sequentially advanced std::mt19937_64.
// Returns the number of mismatching outputs (0 = exact).
extern "C" int gscan_mt64_jump_check(uint64_t seed, uint64_t blocks) {
  using namespace gscan::mt64;
  const uint64_t L = 1ull << 20;
  int nb = 1;
  while ((1ull << nb) <= blocks) ++nb;
  const std::vector<uint64_t>& tab = jump_table(L, nb);
  uint64_t st[kN];
  seed_state(seed, st);
  for (int b = 0; b < nb; ++b)
    if ((blocks >> b) & 1u) apply_jump_host(&tab[(size_t)b * kWords], st);
  std::mt19937_64 eng(seed);
  eng.discard(blocks * L);
  uint64_t x[2 * kN];
  for (int k = 0; k < kN; ++k) x[k] = st[k];
  for (int i = 0; i < kN; ++i) {
    const uint64_t y = (x[i] & kUpper) | (x[i + 1] & kLower);
    x[i + kN] = x[i + kM] ^ (y >> 1) ^ ((x[i + 1] & 1u) ? kMatrixA : 0ull);
  }
  int bad = 0;
  for (int k = 0; k < kN; ++k) {
    uint64_t y = x[kN + k];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    bad += (eng() != y);
  }
  return bad;
}
