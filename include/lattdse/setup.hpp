// Setup-side modules of the reference spec that feed the hot path:
//   cbc        -- SPEC.md:104-161 (wce_squared, cbc_construct), extended to
//                 prime n (candidates 1..n-1) as BASELINE.json's configs need
//   antialias  -- SPEC.md:163-222 (minimal-l2 anti-aliasing set)
//   problems   -- seeded potential / initial-condition families of
//                 BASELINE.json plugged into SPEC.md:313-317's callables
// All host C++; they run once per configuration, never inside a step.
#pragma once

#include <complex>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "lattice.hpp"

namespace lattdse {

// ------------------------------------------------------------------ cbc
namespace cbc {

/// omega(j/n) = 2 pi^2 B2(j/n), B2(x) = x^2 - x + 1/6, from the exact integer
/// numerator 6j^2 - 6jn + n^2 (so omega(j) == omega(n-j) bit for bit).
double omega(std::int64_t j, std::int64_t n);

/// P_1(z) = -1 + (1/n) sum_k prod_j (1 + omega(k z_j mod n)).
/// Raises non_coprime_component if some gcd(z_j, n) != 1.
double wce_squared(std::span<const i64> z, i64 n);

struct Result {
  std::vector<i64> z;          // generating vector, z[0] = 1
  std::vector<double> wce;     // criterion value after each component
};

/// Greedy component-by-component construction: z_1 = 1;
/// z_s = argmin over candidates c in [1,n) with gcd(c,n)=1 of the criterion,
/// ties (relative difference <= kTieRel) to the smallest c. Prime n uses the
/// O(n log n) Rader-permuted correlation to shortlist candidates, then the
/// shortlist is re-scored with the exact sequential sum (cbc::score_naive),
/// so the result equals the exhaustive naive construction.
Result construct(i64 n, int d_max);

constexpr double kTieRel = 1e-13;

/// The same construction on CUDA device `device` for prime n (csrc/cuda/
/// solver.cu): the length-(n-1) correlation runs through the solver's
/// length-M four-step FFT (M >= 2n-1, zero-padded linear correlation), the
/// shortlist is re-scored by a compensated device sum (host long-double
/// total). For n where the host construction is out of reach (config 4:
/// n ~ 2^30, d = 20); equal to construct() on the sizes tests/ compare.
Result construct_device(i64 n, int d_max, int device = 0);

/// Exact criterion of candidate c given the running products P (double) --
/// sequential long double sum over k = 0..n-1.
double score_naive(const std::vector<double>& P, i64 c, i64 n, const std::vector<double>& om);

}  // namespace cbc

// ------------------------------------------------------------ antialias
/// Minimal-l2 anti-aliasing set of full cardinality.
/// For every flattened residue chi: h^(chi) is the first vector in the order
/// (||h||^2 ascending, then lexicographic ascending) with residue chi.
struct AntiAliasSet {
  i64 n_total = 0;
  int dim = 0;
  std::vector<std::uint32_t> norm2;  // ||h^(chi)||^2, exact
  std::vector<std::int16_t> h;       // n_total x dim, row-major (empty if not requested)
  std::uint32_t max_norm2 = 0;

  /// cap_radius <= 0 selects SPEC's default 4*n^(1/d) + 16.
  static AntiAliasSet build(const Lattice& lat, bool with_vectors = true, double cap_radius = -1.0);
  /// Norms only, built on CUDA device `device` (rank-1; csrc/cuda/aaset_dev.cu).
  /// Same norm2 table as build(). A Solver given an AntiAliasSet whose norm2
  /// is empty builds this table on its own device instead.
  static AntiAliasSet build_norms_device(const Lattice& lat, int device = 0, double cap_radius = -1.0);
  /// Brute-force minimality check over ||h||_inf <= bound.
  bool verify_minimal(const Lattice& lat, int bound) const;
  /// FNV-1a over the norm table (u32 little endian), for golden fixtures.
  std::uint64_t norm_hash() const;
};

// ------------------------------------------------------------- problems
namespace problems {

/// SplitMix64 stream; doubles from the top 53 bits.
struct SplitMix64 {
  std::uint64_t state;
  explicit SplitMix64(std::uint64_t seed) : state(seed) {}
  std::uint64_t next();
  double uniform();                       // [0,1)
  double uniform(double lo, double hi);   // [lo,hi)
  int integer(int lo, int hi);            // inclusive
};

/// v(x) = sum_j a_j (1 - cos 2 pi x_j) + sum_{j<d} b_j cos 2 pi (x_j - x_{j+1})
struct Potential {
  std::vector<double> a, b;
};
/// g(x) = C prod_j exp(-sin^2(pi (x_j - c_j)) / (2 sigma^2)) exp(2 pi i p_j x_j)
struct Initial {
  std::vector<double> c;
  std::vector<int> p;
  double sigma = 0.1;
  double C = 1.0;  // set by normalize_on_lattice
};

/// Seed schedule: one stream seeded with `seed` draws
/// a_1..a_d ~ U[0.5,1.5], b_1..b_{d-1} ~ U[0,0.5], then c_1..c_d ~ U[c_lo,c_hi],
/// p_1..p_d ~ U{-p_max..p_max}. Ensemble member m draws its own (c, p) from a
/// stream seeded with member_seed(seed, m).
Potential draw_potential(SplitMix64& rng, int d);
Initial draw_initial(SplitMix64& rng, int d, double c_lo, double c_hi, int p_max, double sigma);
std::uint64_t member_seed(std::uint64_t base, std::int64_t member);

/// cos(2 pi a / L) with a reduced exactly mod L.
double cos2pi_frac(i64 a, i64 L);
/// exp(2 pi i a / L) with a reduced exactly mod L.
std::complex<double> cis2pi_frac(i64 a, i64 L);

double eval_v(const Potential& v, const i64* num, int d, i64 L);
std::complex<double> eval_g_unnormalized(const Initial& g, const i64* num, int d, i64 L);

/// v at every lattice point (kappa order).
std::vector<double> sample_v(const Lattice& lat, const Potential& v);
/// Normalised g at every lattice point; sets g.C so (1/N) sum |g|^2 = 1.
std::vector<std::complex<double>> sample_g(const Lattice& lat, Initial& g);

}  // namespace problems

}  // namespace lattdse
