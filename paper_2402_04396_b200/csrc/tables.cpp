// Codebook and Hadamard tables, rebuilt from the reference's construction
// rules (not copied): E8P pattern table (core/src/e8p.cpp:37-79), the
// e8-1bit lattice ball (core/src/codebook.cpp:162-243), Hadamard bases
// (core/src/hadamard.cpp:14-154) and the planner (hadamard.cpp:156-168),
// with the registry extended by order 172 (had172_data.h).
#include <algorithm>
#include <bit>
#include <cmath>
#include <map>
#include <mutex>

#include "had172_data.h"
#include "internal.hpp"

namespace q8p {
namespace detail {
namespace {

// Padding rows 227..255 (sum of squares 48).  Their order is part of the
// artifact format (codewords index into it), so this list is format data:
// e8p.cpp:17-33, pinned by tests/acceptance.cpp:137-151.
constexpr std::int8_t kE8PTail[29][8] = {
    {3, 1, 1, 1, 3, 3, 3, 3}, {1, 3, 1, 1, 3, 3, 3, 3}, {1, 1, 3, 1, 3, 3, 3, 3},
    {1, 1, 1, 3, 3, 3, 3, 3}, {3, 3, 3, 1, 3, 3, 1, 1}, {3, 3, 3, 1, 3, 1, 3, 1},
    {3, 3, 3, 1, 1, 3, 3, 1}, {3, 3, 3, 1, 3, 1, 1, 3}, {3, 3, 3, 1, 1, 3, 1, 3},
    {3, 3, 3, 1, 1, 1, 3, 3}, {3, 3, 1, 3, 3, 3, 1, 1}, {3, 3, 1, 3, 3, 1, 3, 1},
    {3, 3, 1, 3, 1, 3, 3, 1}, {3, 3, 1, 3, 3, 1, 1, 3}, {3, 3, 1, 3, 1, 3, 1, 3},
    {3, 3, 1, 3, 1, 1, 3, 3}, {3, 1, 3, 3, 3, 3, 1, 1}, {3, 1, 3, 3, 3, 1, 3, 1},
    {3, 1, 3, 3, 1, 3, 3, 1}, {3, 1, 3, 3, 3, 1, 1, 3}, {3, 1, 3, 3, 1, 3, 1, 3},
    {1, 3, 3, 3, 1, 1, 3, 3}, {1, 3, 3, 3, 3, 3, 1, 1}, {1, 3, 3, 3, 3, 1, 3, 1},
    {1, 3, 3, 3, 1, 3, 3, 1}, {1, 3, 3, 3, 3, 1, 1, 3}, {1, 3, 3, 3, 1, 3, 1, 3},
    {1, 1, 3, 3, 1, 3, 3, 3}, {3, 3, 1, 1, 3, 3, 3, 1},
};

E8PTable build_e8p_table() {
  E8PTable t{};
  // Sorted {1,3,5}^8 patterns with sum of squares <= 40: walk the patterns
  // as base-3 numbers (coordinate 7 least significant), which visits them in
  // lexicographic order, and keep those inside the ball.
  std::size_t rows = 0;
  std::array<int, 8> digit{};
  for (int code = 0; code < 6561; ++code) {
    int rem = code, ss = 0;
    for (int c = 7; c >= 0; --c) {
      digit[c] = 1 + 2 * (rem % 3);
      rem /= 3;
      ss += digit[c] * digit[c];
    }
    if (ss > 40) continue;
    if (rows >= 227) throw Error("e8p table: too many ball rows");
    for (int c = 0; c < 8; ++c) t.doubled[rows][c] = static_cast<std::int8_t>(digit[c]);
    ++rows;
  }
  if (rows != 227) throw Error("e8p table: expected 227 ball rows");
  for (int i = 0; i < 29; ++i)
    for (int c = 0; c < 8; ++c) t.doubled[227 + i][c] = kE8PTail[i][c];
  for (int i = 0; i < 256; ++i) {
    int s = 0;
    for (int c = 0; c < 8; ++c) s += t.doubled[i][c];
    t.odd_parity[i] = static_cast<std::uint8_t>((s & 3) == 2);
  }
  return t;
}

std::array<std::array<std::int8_t, 8>, 256> build_e8_1bit() {
  // E8 points (doubled: all-even or all-odd coordinates, sum = 0 mod 4) with
  // doubled squared norm <= 32; that set has >= 256 points, so the first 256
  // by (norm, lexicographic doubled tuple) are the table.
  std::vector<std::array<std::int8_t, 8>> pts;
  std::array<std::int8_t, 8> cur{};
  auto rec = [&](auto&& self, int pos, int parity, int rem, int sum) -> void {
    if (pos == 8) {
      if (((sum % 4) + 4) % 4 == 0) pts.push_back(cur);
      return;
    }
    int tmax = static_cast<int>(std::sqrt(static_cast<double>(rem)));
    while (tmax * tmax > rem) --tmax;
    if ((tmax & 1) != parity) --tmax;
    for (int v = -tmax; v <= tmax; v += 2) {
      cur[pos] = static_cast<std::int8_t>(v);
      self(self, pos + 1, parity, rem - v * v, sum + v);
    }
  };
  rec(rec, 0, 0, 32, 0);
  rec(rec, 0, 1, 32, 0);
  auto norm = [](const std::array<std::int8_t, 8>& v) {
    int s = 0;
    for (int x : v) s += x * x;
    return s;
  };
  std::sort(pts.begin(), pts.end(), [&](const auto& a, const auto& b) {
    const int na = norm(a), nb = norm(b);
    return na != nb ? na < nb : a < b;
  });
  if (pts.size() < 256) throw Error("e8-1bit table: ball too small");
  std::array<std::array<std::int8_t, 8>, 256> out{};
  for (int i = 0; i < 256; ++i) out[i] = pts[i];
  return out;
}

int legendre(long a, long p) {
  a %= p;
  if (a < 0) a += p;
  if (a == 0) return 0;
  long r = 1, b = a, e = (p - 1) / 2;
  while (e) {
    if (e & 1) r = r * b % p;
    b = b * b % p;
    e >>= 1;
  }
  return r == 1 ? 1 : -1;
}

std::vector<std::int8_t> build_base(std::size_t q) {
  std::vector<std::int8_t> b(q * q);
  auto at = [&](std::size_t i, std::size_t j) -> std::int8_t& { return b[i * q + j]; };
  switch (q) {
    case 1:
      b[0] = 1;
      break;
    case 4:  // Sylvester: H[i][j] = (-1)^popcount(i & j)
      for (std::size_t i = 0; i < 4; ++i)
        for (std::size_t j = 0; j < 4; ++j) at(i, j) = std::popcount(i & j) & 1 ? -1 : 1;
      break;
    case 12:
    case 20: {  // Paley I over GF(q-1): [[1, 1^T], [-1, Q + I]], Q[i][j] = chi(i - j)
      const long p = static_cast<long>(q) - 1;
      for (std::size_t i = 0; i < q; ++i)
        for (std::size_t j = 0; j < q; ++j) {
          if (i == 0)
            at(i, j) = 1;
          else if (j == 0)
            at(i, j) = -1;
          else
            at(i, j) = static_cast<std::int8_t>(
                i == j ? 1 : legendre(static_cast<long>(i) - static_cast<long>(j), p));
        }
      break;
    }
    case 28: {  // Paley II over GF(13): symmetric conference matrix, 2x2 blocks
      const long p = 13;
      const std::size_t m = 14;
      for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < m; ++j) {
          int s;
          if (i == 0 || j == 0)
            s = (i == j) ? 0 : 1;
          else
            s = i == j ? 0 : legendre(static_cast<long>(j) - static_cast<long>(i), p);
          const int blk[2][2] = {{s == 0 ? 1 : s, s == 0 ? -1 : s}, {s == 0 ? -1 : s, s == 0 ? -1 : -s}};
          for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 2; ++c) at(2 * i + a, 2 * j + c) = static_cast<std::int8_t>(blk[a][c]);
        }
      break;
    }
    case 172:
      for (std::size_t i = 0; i < q; ++i)
        for (std::size_t j = 0; j < q; ++j)
          at(i, j) = (q8p_had172_bits[i][j / 64] >> (j % 64)) & 1 ? -1 : 1;
      break;
    default:
      throw SizeError("hadamard_base: order " + std::to_string(q) + " not in registry");
  }
  // Self-check B * B^T = q I, as the reference does once per order (hadamard.cpp:99-112).
  for (std::size_t i = 0; i < q; ++i)
    for (std::size_t j = 0; j < q; ++j) {
      long dot = 0;
      for (std::size_t k = 0; k < q; ++k) dot += long(b[i * q + k]) * b[j * q + k];
      if (dot != (i == j ? long(q) : 0L)) throw Error("hadamard base self-check failed");
    }
  return b;
}

constexpr std::size_t kRegistry[] = {1, 4, 12, 20, 28, 172};

}  // namespace

const E8PTable& e8p_table() {
  static const E8PTable t = build_e8p_table();
  return t;
}

void e8p_decode_host(std::uint16_t word, float out[8]) {
  const E8PTable& t = e8p_table();
  const unsigned idx = word >> 8, sb = (word >> 1) & 0x7Fu;
  const float shift = (word & 1u) ? 0.25f : -0.25f;
  int neg0 = (std::popcount(sb) & 1) != t.odd_parity[idx];
  for (int c = 0; c < 8; ++c) {
    const bool neg = c == 0 ? neg0 : ((sb >> (7 - c)) & 1u);
    const float a = 0.5f * t.doubled[idx][c];
    out[c] = (neg ? -a : a) + shift;
  }
}

const std::array<std::array<std::int8_t, 8>, 256>& e8_1bit_doubled() {
  static const auto t = build_e8_1bit();
  return t;
}

const std::vector<std::int8_t>& hadamard_base(std::size_t q) {
  static std::map<std::size_t, std::vector<std::int8_t>> cache;
  static std::mutex mu;
  std::scoped_lock lock(mu);
  auto it = cache.find(q);
  if (it == cache.end()) it = cache.emplace(q, build_base(q)).first;
  return it->second;
}

}  // namespace detail

HadamardSpec plan_hadamard(std::size_t n) {
  if (n == 0) throw SizeError("plan_hadamard: n must be positive");
  for (std::size_t p = std::size_t{1} << std::countr_zero(n); p >= 1; p >>= 1) {
    const std::size_t q = n / p;
    for (std::size_t order : detail::kRegistry)
      if (order == q) return HadamardSpec{n, p, q};
    if (p == 1) break;
  }
  throw SizeError("plan_hadamard: no power-of-two x base factorization for " + std::to_string(n));
}

}  // namespace q8p
