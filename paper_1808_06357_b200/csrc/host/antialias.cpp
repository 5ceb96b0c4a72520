// Minimal-l2 anti-aliasing set, SPEC.md:163-222 / PAPER.md:1321-1326.
//
// SPEC's rule: walk integer vectors by ascending squared norm, lexicographic
// inside a shell, first vector to hit a residue wins. That order is a total
// order on (||h||^2, h), so the winner for residue chi is simply the minimum
// of (||h||^2, h) over the vectors with that residue. We therefore enumerate
// the ball ||h||^2 <= S once (in any order, in parallel) and keep, per
// residue, the minimum of a packed 64-bit key (norm2, lex digits of h) with an
// atomic compare-and-swap. S grows geometrically until every residue is hit;
// SPEC's radius cap 4 n^(1/d) + 16 raises radius_exhausted.
#include <algorithm>
#include <atomic>
#include <cmath>

#include "lattdse/setup.hpp"

namespace lattdse {

namespace {

constexpr int kMaxRank = 64;

struct Enum {
  int d, r;
  i64 S;           // squared radius
  i64 H;           // max |h_j| = floor(sqrt(S))
  std::uint64_t base;  // 2H+1
  std::vector<std::vector<i64>> zmod;  // [i][j] = z_ij mod n_i
  std::vector<i64> mod, fw;            // moduli, flat weights
  std::atomic<std::uint64_t>* key;
  std::uint64_t lexspan;  // base^d

  void rec(int j, i64 rem, const i64* part, std::uint64_t lex, i64 norm) const {
    i64 mm = static_cast<i64>(std::sqrt(static_cast<double>(rem)));
    while ((mm + 1) * (mm + 1) <= rem) ++mm;
    while (mm * mm > rem) --mm;
    i64 nxt[kMaxRank];
    for (i64 x = -mm; x <= mm; ++x) {
      for (int i = 0; i < r; ++i) {
        i64 v = (part[i] + x * zmod[i][j]) % mod[i];
        nxt[i] = v < 0 ? v + mod[i] : v;
      }
      const std::uint64_t lx = lex * base + static_cast<std::uint64_t>(x + H);
      const i64 nn = norm + x * x;
      if (j + 1 < d) {
        rec(j + 1, rem - x * x, nxt, lx, nn);
      } else {
        i64 chi = 0;
        for (int i = 0; i < r; ++i) chi += nxt[i] * fw[i];
        const std::uint64_t k = static_cast<std::uint64_t>(nn) * lexspan + lx;
        auto& slot = key[chi];
        std::uint64_t cur = slot.load(std::memory_order_relaxed);
        while (k < cur && !slot.compare_exchange_weak(cur, k, std::memory_order_relaxed)) {
        }
      }
    }
  }
};

}  // namespace

AntiAliasSet AntiAliasSet::build(const Lattice& lat, bool with_vectors, double cap_radius) {
  const int d = lat.dim(), r = lat.rank();
  const i64 N = lat.n_total();
  if (cap_radius <= 0) cap_radius = 4.0 * std::pow(static_cast<double>(N), 1.0 / d) + 16.0;
  const i64 cap2 = static_cast<i64>(std::floor(cap_radius * cap_radius));

  // starting radius: ball volume ~ 2N
  const double vd = std::pow(M_PI, d / 2.0) / std::tgamma(d / 2.0 + 1.0);
  i64 S = std::max<i64>(1, static_cast<i64>(std::ceil(std::pow(2.0 * N / vd, 2.0 / d))));

  if (r > kMaxRank) raise(Errc::unsupported, "anti-aliasing build supports rank <= 64");
  std::vector<std::atomic<std::uint64_t>> key(N);
  for (;;) {
    S = std::min(S, cap2);
    Enum e;
    e.d = d;
    e.r = r;
    e.S = S;
    e.H = static_cast<i64>(std::floor(std::sqrt(static_cast<double>(S))));
    while ((e.H + 1) * (e.H + 1) <= S) ++e.H;
    e.base = static_cast<std::uint64_t>(2 * e.H + 1);
    long double span = std::pow(static_cast<long double>(e.base), d);
    if (span * (static_cast<long double>(S) + 1) >= 1.8e19L)
      raise(Errc::unsupported, "anti-aliasing key does not fit 64 bits for this (d, radius)");
    e.lexspan = 1;
    for (int j = 0; j < d; ++j) e.lexspan *= e.base;
    e.mod = lat.moduli();
    e.fw = lat.flat_weights();
    e.zmod.assign(r, std::vector<i64>(d));
    for (int i = 0; i < r; ++i) {
      auto col = lat.gen_column(i);
      for (int j = 0; j < d; ++j) e.zmod[i][j] = ((col[j] % e.mod[i]) + e.mod[i]) % e.mod[i];
    }
    e.key = key.data();
    for (auto& k : key) k.store(~std::uint64_t(0), std::memory_order_relaxed);

    const i64 H = e.H;
#pragma omp parallel for schedule(dynamic, 1)
    for (i64 x0 = -H; x0 <= H; ++x0) {
      i64 part[kMaxRank];
      for (int i = 0; i < r; ++i) {
        i64 v = (x0 * e.zmod[i][0]) % e.mod[i];
        part[i] = v < 0 ? v + e.mod[i] : v;
      }
      const std::uint64_t lx = static_cast<std::uint64_t>(x0 + H);
      if (d == 1) {
        i64 chi = 0;
        for (int i = 0; i < r; ++i) chi += part[i] * e.fw[i];
        const std::uint64_t k = static_cast<std::uint64_t>(x0 * x0) * e.lexspan + lx;
        auto& slot = key[chi];
        std::uint64_t cur = slot.load(std::memory_order_relaxed);
        while (k < cur && !slot.compare_exchange_weak(cur, k, std::memory_order_relaxed)) {
        }
      } else {
        e.rec(1, S - x0 * x0, part, lx, x0 * x0);
      }
    }

    bool full = true;
    for (i64 c = 0; c < N && full; ++c)
      if (key[c].load(std::memory_order_relaxed) == ~std::uint64_t(0)) full = false;
    if (full) {
      AntiAliasSet out;
      out.n_total = N;
      out.dim = d;
      out.norm2.resize(N);
      if (with_vectors) out.h.resize(static_cast<size_t>(N) * d);
      std::uint32_t mx = 0;
#pragma omp parallel for schedule(static) reduction(max : mx)
      for (i64 c = 0; c < N; ++c) {
        std::uint64_t k = key[c].load(std::memory_order_relaxed);
        const std::uint64_t nn = k / e.lexspan;
        std::uint64_t lx = k % e.lexspan;
        out.norm2[c] = static_cast<std::uint32_t>(nn);
        mx = std::max<std::uint32_t>(mx, static_cast<std::uint32_t>(nn));
        if (with_vectors)
          for (int j = d - 1; j >= 0; --j) {
            out.h[static_cast<size_t>(c) * d + j] = static_cast<std::int16_t>(static_cast<i64>(lx % e.base) - H);
            lx /= e.base;
          }
      }
      out.max_norm2 = mx;
      return out;
    }
    if (S >= cap2)
      raise(Errc::radius_exhausted, "anti-aliasing set incomplete at the radius cap " + std::to_string(cap_radius));
    S = static_cast<i64>(std::ceil(S * 1.35)) + 1;
  }
}

bool AntiAliasSet::verify_minimal(const Lattice& lat, int bound) const {
  const int d = lat.dim();
  const i64 N = lat.n_total();
  if (static_cast<i64>(norm2.size()) != N) return false;
  // every residue present exactly once with matching residue
  if (!h.empty())
    for (i64 c = 0; c < N; ++c) {
      std::vector<i64> hv(h.begin() + c * d, h.begin() + (c + 1) * d);
      if (lat.flat_residue(hv) != c) return false;
      i64 nn = 0;
      for (i64 x : hv) nn += x * x;
      if (static_cast<std::uint32_t>(nn) != norm2[c]) return false;
    }
  // brute force: no vector in the box has a smaller norm than the table
  std::vector<i64> hv(d, -bound);
  for (;;) {
    i64 nn = 0;
    for (i64 x : hv) nn += x * x;
    if (static_cast<std::uint64_t>(nn) < norm2[lat.flat_residue(hv)]) return false;
    int j = d - 1;
    while (j >= 0 && hv[j] == bound) hv[j--] = -bound;
    if (j < 0) break;
    ++hv[j];
  }
  return true;
}

std::uint64_t AntiAliasSet::norm_hash() const {
  std::uint64_t hsh = 14695981039346656037ULL;
  for (std::uint32_t v : norm2)
    for (int b = 0; b < 4; ++b) {
      hsh ^= (v >> (8 * b)) & 0xffu;
      hsh *= 1099511628211ULL;
    }
  return hsh;
}

}  // namespace lattdse
