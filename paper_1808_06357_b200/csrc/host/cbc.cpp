// Component-by-component construction of rank-1 generating vectors,
// SPEC.md:104-161 (criterion SPEC.md:117-126, greedy SPEC.md:128-137),
// extended to prime n as BASELINE.json's configs require (candidates
// 1..n-1, same criterion, same smallest-candidate tie-break).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "hostfft.hpp"
#include "lattdse/setup.hpp"

namespace lattdse::cbc {

namespace {

const long double kPi2L = 9.869604401089358618834490999876151135L;  // pi^2

bool is_prime(i64 n) {
  if (n < 2) return false;
  for (i64 p : {2, 3, 5, 7, 11, 13})
    if (n % p == 0) return n == p;
  for (i64 f = 17; f * f <= n; f += 2)
    if (n % f == 0) return false;
  return true;
}

i64 powmod(i64 b, i64 e, i64 m) {
  __int128 r = 1, x = b % m;
  while (e) {
    if (e & 1) r = r * x % m;
    x = x * x % m;
    e >>= 1;
  }
  return static_cast<i64>(r);
}

i64 primitive_root(i64 p) {
  std::vector<i64> fac;
  i64 m = p - 1;
  for (i64 f = 2; f * f <= m; ++f)
    if (m % f == 0) {
      fac.push_back(f);
      while (m % f == 0) m /= f;
    }
  if (m > 1) fac.push_back(m);
  for (i64 g = 2; g < p; ++g) {
    bool ok = true;
    for (i64 f : fac)
      if (powmod(g, (p - 1) / f, p) == 1) {
        ok = false;
        break;
      }
    if (ok) return g;
  }
  return 1;  // p == 2
}

std::vector<double> omega_table(i64 n) {
  std::vector<double> om(n);
#pragma omp parallel for schedule(static) if (n > 4096)
  for (i64 j = 0; j < n; ++j) om[j] = omega(j, n);
  return om;
}

// Index of the winning candidate among (value, candidate) pairs: smallest
// value; values within kTieRel of the minimum count as ties -> smallest c.
i64 pick(const std::vector<std::pair<double, i64>>& scored) {
  double best = scored.front().first;
  for (auto& s : scored) best = std::min(best, s.first);
  const double tol = kTieRel * std::fabs(best);
  i64 winner = -1;
  for (auto& s : scored)
    if (s.first <= best + tol && (winner < 0 || s.second < winner)) winner = s.second;
  return winner;
}

}  // namespace

double omega(std::int64_t j, std::int64_t n) {
  const __int128 nn = n, jj = j % n;
  const __int128 num = 6 * jj * (jj - nn) + nn * nn;  // 6 n^2 B2(j/n)
  return static_cast<double>(static_cast<long double>(num) * (kPi2L / (3.0L * static_cast<long double>(n) *
                                                                          static_cast<long double>(n))));
}

double wce_squared(std::span<const i64> z, i64 n) {
  if (n < 1) raise(Errc::invalid_argument, "wce_squared: n must be >= 1");
  for (i64 c : z) {
    i64 r = ((c % n) + n) % n;
    if (n > 1 && std::gcd(r, n) != 1)
      raise(Errc::non_coprime_component, "wce_squared: component " + std::to_string(c) + " not coprime to n");
  }
  const auto om = omega_table(n);
  long double acc = 0;
  for (i64 k = 0; k < n; ++k) {
    long double prod = 1;
    for (i64 c : z) {
      i64 r = static_cast<i64>((static_cast<__int128>(k) * (((c % n) + n) % n)) % n);
      prod *= 1.0L + static_cast<long double>(om[r]);
    }
    acc += prod;
  }
  return static_cast<double>(acc / static_cast<long double>(n) - 1.0L);
}

double score_naive(const std::vector<double>& P, i64 c, i64 n, const std::vector<double>& om) {
  long double acc = 0;
  i64 r = 0;  // k*c mod n, incrementally
  for (i64 k = 0; k < n; ++k) {
    acc += static_cast<long double>(P[k]) * (1.0L + static_cast<long double>(om[r]));
    r += c;
    if (r >= n) r -= n;
  }
  return static_cast<double>(acc / static_cast<long double>(n) - 1.0L);
}

Result construct(i64 n, int d_max) {
  if (n < 2) raise(Errc::invalid_argument, "cbc: n must be >= 2");
  if (d_max < 1) raise(Errc::invalid_argument, "cbc: d_max must be >= 1");
  const auto om = omega_table(n);
  std::vector<double> P(n, 1.0);
  Result res;
  auto apply = [&](i64 c) {
    i64 r = 0;
    for (i64 k = 0; k < n; ++k) {
      P[k] = P[k] * (1.0 + om[r]);
      r += c;
      if (r >= n) r -= n;
    }
  };
  res.z.push_back(1);
  apply(1);
  res.wce.push_back(score_naive(std::vector<double>(n, 1.0), 1, n, om));

  const bool prime = is_prime(n);
  const i64 g = prime ? primitive_root(n) : 0;
  std::vector<i64> gpow;  // g^a mod n, a = 0..n-2
  if (prime && d_max > 1) {
    gpow.resize(n - 1);
    i64 x = 1;
    for (i64 a = 0; a < n - 1; ++a) {
      gpow[a] = x;
      x = static_cast<i64>(static_cast<__int128>(x) * g % n);
    }
  }

  for (int s = 2; s <= d_max; ++s) {
    std::vector<std::pair<double, i64>> shortlist;
    if (prime && n > 64) {
      // corr(e) = sum_a P(g^a) om(g^(a+e)): cyclic correlation of length n-1.
      const i64 L = n - 1;
      std::vector<hostfft::cd> pa(L), wa(L);
      for (i64 a = 0; a < L; ++a) {
        pa[a] = P[gpow[a]];
        wa[a] = om[gpow[a]];
      }
      hostfft::dft(pa, -1);
      hostfft::dft(wa, -1);
      for (i64 a = 0; a < L; ++a) pa[a] = std::conj(pa[a]) * wa[a];
      hostfft::dft(pa, +1);
      long double base = 0;
      for (i64 k = 0; k < n; ++k) base += P[k];
      base += static_cast<long double>(P[0]) * om[0];
      std::vector<double> approx(L);
      double best = INFINITY;
      for (i64 e = 0; e < L; ++e) {
        approx[e] = static_cast<double>((base + pa[e].real() / static_cast<double>(L)) / n - 1.0L);
        best = std::min(best, approx[e]);
      }
      const double window = std::max(1e-9 * std::fabs(best), 1e-13);
      std::vector<i64> cands;
      for (i64 e = 0; e < L; ++e)
        if (approx[e] <= best + window) cands.push_back(gpow[e]);
      std::sort(cands.begin(), cands.end());
      shortlist.resize(cands.size());
#pragma omp parallel for schedule(dynamic)
      for (size_t q = 0; q < cands.size(); ++q) shortlist[q] = {score_naive(P, cands[q], n, om), cands[q]};
    } else {
      std::vector<i64> cands;
      for (i64 c = 1; c < n; ++c)
        if (std::gcd(c, n) == 1) cands.push_back(c);
      shortlist.resize(cands.size());
#pragma omp parallel for schedule(dynamic, 16)
      for (size_t q = 0; q < cands.size(); ++q) shortlist[q] = {score_naive(P, cands[q], n, om), cands[q]};
    }
    const i64 zs = pick(shortlist);
    double val = 0;
    for (auto& sc : shortlist)
      if (sc.second == zs) val = sc.first;
    res.z.push_back(zs);
    res.wce.push_back(val);
    apply(zs);
  }
  return res;
}

}  // namespace lattdse::cbc
