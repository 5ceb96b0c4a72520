// Seeded potential / initial-condition families of BASELINE.json, plugged
// into the callable slots of SPEC.md:313-317 (ProblemSpec). The paper's own
// families are not in any configuration.
//
// Trigonometric arguments are formed from exact integer numerators reduced
// mod the lattice denominator before conversion.
#include <cmath>

#include "lattdse/setup.hpp"

namespace lattdse::problems {

namespace {
const long double kPiL = 3.141592653589793238462643383279502884L;
}

std::uint64_t SplitMix64::next() {
  state += 0x9E3779B97F4A7C15ULL;
  std::uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double SplitMix64::uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

double SplitMix64::uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

int SplitMix64::integer(int lo, int hi) {
  const int span = hi - lo + 1;
  int k = static_cast<int>(std::floor(uniform() * span));
  if (k >= span) k = span - 1;
  return lo + k;
}

Potential draw_potential(SplitMix64& rng, int d) {
  Potential v;
  for (int j = 0; j < d; ++j) v.a.push_back(rng.uniform(0.5, 1.5));
  for (int j = 0; j + 1 < d; ++j) v.b.push_back(rng.uniform(0.0, 0.5));
  return v;
}

Initial draw_initial(SplitMix64& rng, int d, double c_lo, double c_hi, int p_max, double sigma) {
  Initial g;
  g.sigma = sigma;
  for (int j = 0; j < d; ++j) g.c.push_back(rng.uniform(c_lo, c_hi));
  for (int j = 0; j < d; ++j) g.p.push_back(rng.integer(-p_max, p_max));
  return g;
}

std::uint64_t member_seed(std::uint64_t base, std::int64_t member) {
  SplitMix64 s(base ^ static_cast<std::uint64_t>(member + 1));
  return s.next();
}

double cos2pi_frac(i64 a, i64 L) {
  i64 r = a % L;
  if (r < 0) r += L;
  return static_cast<double>(cosl(2.0L * kPiL * static_cast<long double>(r) / static_cast<long double>(L)));
}

std::complex<double> cis2pi_frac(i64 a, i64 L) {
  i64 r = a % L;
  if (r < 0) r += L;
  const long double t = 2.0L * kPiL * static_cast<long double>(r) / static_cast<long double>(L);
  return {static_cast<double>(cosl(t)), static_cast<double>(sinl(t))};
}

double eval_v(const Potential& v, const i64* num, int d, i64 L) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) acc += v.a[j] * (1.0 - cos2pi_frac(num[j], L));
  for (int j = 0; j + 1 < d; ++j) acc += v.b[j] * cos2pi_frac(num[j] - num[j + 1], L);
  return acc;
}

std::complex<double> eval_g_unnormalized(const Initial& g, const i64* num, int d, i64 L) {
  long double expo = 0;
  __int128 phase = 0;
  const long double inv2s2 = 1.0L / (2.0L * static_cast<long double>(g.sigma) * g.sigma);
  for (int j = 0; j < d; ++j) {
    const long double x = static_cast<long double>(num[j]) / static_cast<long double>(L);
    const long double s = sinl(kPiL * (x - static_cast<long double>(g.c[j])));
    expo -= s * s * inv2s2;
    phase += static_cast<__int128>(g.p[j]) * num[j];
  }
  const i64 ph = static_cast<i64>(((phase % L) + L) % L);
  const double amp = static_cast<double>(expl(expo));
  return amp * cis2pi_frac(ph, L);
}

std::vector<double> sample_v(const Lattice& lat, const Potential& v) {
  const auto num = lat.point_numerators();
  const int d = lat.dim();
  const i64 N = lat.n_total(), L = lat.denom();
  std::vector<double> out(N);
#pragma omp parallel for schedule(static)
  for (i64 k = 0; k < N; ++k) out[k] = eval_v(v, num.data() + k * d, d, L);
  return out;
}

std::vector<std::complex<double>> sample_g(const Lattice& lat, Initial& g) {
  const auto num = lat.point_numerators();
  const int d = lat.dim();
  const i64 N = lat.n_total(), L = lat.denom();
  std::vector<std::complex<double>> out(N);
#pragma omp parallel for schedule(static)
  for (i64 k = 0; k < N; ++k) out[k] = eval_g_unnormalized(g, num.data() + k * d, d, L);
  // (1/N) sum |g|^2 by fixed-block partial sums (deterministic under OpenMP)
  const i64 blk = 4096, nb = (N + blk - 1) / blk;
  std::vector<long double> part(nb, 0);
#pragma omp parallel for schedule(static)
  for (i64 b = 0; b < nb; ++b) {
    long double s = 0;
    for (i64 k = b * blk; k < std::min(N, (b + 1) * blk); ++k) s += std::norm(out[k]);
    part[b] = s;
  }
  long double tot = 0;
  for (auto s : part) tot += s;
  if (!(tot > 0)) raise(Errc::non_normalizable, "initial condition vanishes on the lattice");
  g.C = static_cast<double>(1.0L / sqrtl(tot / static_cast<long double>(N)));
#pragma omp parallel for schedule(static)
  for (i64 k = 0; k < N; ++k) out[k] *= g.C;
  return out;
}

}  // namespace lattdse::problems
