// The C++ drop-in claim, exercised: code written against the reference's
// public header (include/lattdse/lattice.hpp mirrors lattice.hpp:17-86,
// errors.hpp:8-34) plus the solver/setup headers, compiled with g++ -std=c++20
// and linked to the in-tree library (tests/test_cxx_consumer.py).
//   ./cxx_consumer          lattice-core + setup (CPU)
//   ./cxx_consumer --gpu    + a Strang propagation on device 0
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <vector>

#include "lattdse/errors.hpp"
#include "lattdse/lattice.hpp"
#include "lattdse/setup.hpp"
#include "lattdse/solver.hpp"

using namespace lattdse;

static int fail(const char* what) {
  std::printf("FAIL %s\n", what);
  return 1;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  // the paper's Fig. 1 lattice, as a reference caller builds it (lattice.hpp:35)
  Lattice fig1 = Lattice::create(2, 1, {{1, 34}}, {55});
  std::printf("fig1 hash=0x%016llx n=%lld\n", (unsigned long long)fig1.hash(), (long long)fig1.n_total());
  LatticePoint p7 = fig1.point(7);
  if (p7.num.size() != 2 || p7.num[0] != 7 || p7.num[1] != (7 * 34) % 55) return fail("point(7)");
  const std::vector<i64> h = {3, -1};
  if (fig1.flat_residue(h) != ((3 - 34) % 55 + 55) % 55) return fail("flat_residue");
  Lattice back = Lattice::from_json(fig1.to_json());
  if (!(back == fig1)) return fail("json round trip");
  // errors cross the library boundary as lattdse::Error with the reference codes
  try {
    Lattice::create(2, 2, {{1, 0}, {0, 1}}, {4, 8});
    return fail("non-divisible moduli accepted");
  } catch (const Error& e) {
    if (e.code() != Errc::non_divisible_moduli) return fail("error code");
    std::printf("caught %s\n", e.what());
  }
  // setup: prime-n CBC and the anti-aliasing norm table
  cbc::Result z = cbc::construct(4099, 2);
  std::printf("C0 z=(%lld,%lld)\n", (long long)z.z[0], (long long)z.z[1]);
  Lattice c0 = Lattice::rank1(z.z, 4099);
  AntiAliasSet aa = AntiAliasSet::build(c0, false);
  std::printf("aaset max norm2=%u hash=0x%016llx\n", aa.max_norm2, (unsigned long long)aa.norm_hash());
  if (!gpu) {
    std::printf("cpu ok\n");
    return 0;
  }
  ProblemSpec prob;
  prob.eps = 0.1;
  problems::SplitMix64 rng(0x180806357ull);
  prob.potential = problems::draw_potential(rng, 2);
  prob.initial.push_back(problems::draw_initial(rng, 2, 0.4, 0.6, 2, 0.1));
  Solver S(c0, aa, prob);
  S.set_dt(1.0 / 256);
  S.discretize_initial();
  std::vector<TrajectoryRow> tr = S.propagate(64, 16);
  const double n = S.l2_norm()[0];
  std::printf("64 Strang steps: norm-1=%.3e energy %.12f -> %.12f rows=%zu\n", n - 1.0, tr.front().energy,
              tr.back().energy, tr.size());
  if (std::fabs(n - 1.0) > 1e-12 || tr.size() != 5) return fail("norm / trajectory");
  std::vector<std::complex<double>> u(4099);
  S.get_state(u.data(), 1, Space::coefficients);
  if (std::fabs(S.l2_distance(u.data(), Space::coefficients)) > 1e-13) return fail("l2_distance");
  std::printf("gpu ok\n");
  return 0;
}
