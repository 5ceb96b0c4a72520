// lattdse::Solver -- the time-stepping hot path on a B200.
//
// Mirrors the tdse/spectral operations of SPEC.md:308-399 / SPEC.md:224-306
// (discretize_initial, strang_step, propagate, l2_norm, energy, analyze,
// synthesize) over a lattice + anti-aliasing norm table + seeded problem.
// All arithmetic runs in the sm_100a pass kernels; this header carries no
// CUDA types. One Solver owns one device, one stream and all its buffers; it
// is not internally synchronised (SURVEY.md §8(b) threading rule).
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "lattice.hpp"
#include "setup.hpp"

namespace lattdse {

enum class Space : int { samples = 0, coefficients = 1 };

struct SolverOptions {
  int device = 0;
  /// rank-1 step algorithm: "circulant" (one length-M convolution per step,
  /// default) or "bluestein" (the literal two length-N DFTs per step).
  std::string method = "circulant";
  /// members stepped together while L2-resident; 0 = automatic.
  std::int64_t group = 0;
  /// force the length-M view M1 x M2 (rank-1; 0 = automatic); with
  /// force_M2a > 0 the rows are split three-level as M2 = M2a x (M2 / M2a)
  std::int64_t force_M1 = 0, force_M2 = 0, force_M2a = 0;
};

struct ProblemSpec {
  double eps = 1.0;
  problems::Potential potential;
  /// one initial condition per ensemble member (batch = size)
  std::vector<problems::Initial> initial;
};

struct TrajectoryRow {
  std::int64_t step;
  double time;
  double norm;
  double energy;
};

struct SolverInfo {
  std::int64_t n_total, batch, M, M1, M2;
  std::int64_t M2a;  // three-level inner split of M2 (0: two-level)
  int rank;
  std::string method;
  double bytes_per_step;        // algorithmic HBM bytes per step (whole batch), see DESIGN.md
  double bytes_per_pass_col, bytes_per_pass_row;
  int launches_per_step;
  std::int64_t group;
  std::int64_t row_chunk;  // three-level: M1 rows per L2-resident row-side chunk (0: whole view)
  int pass4;               // 1: per-step passes have run on the lean plain-layout kernels (fft_pass4.cuh)
};

class Solver {
 public:
  Solver(const Lattice& lat, const AntiAliasSet& aa, const ProblemSpec& prob, const SolverOptions& opt = {});
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  /// Build the propagator phases for a time step.
  void set_dt(double dt);
  double dt() const;
  void set_watchdog(double tol);

  /// g sampled on the lattice for every member; the state is
  /// held in sample space, so this is the discretised initial condition.
  void discretize_initial();

  /// Host <-> device state transfer for members [m0, m0+count).
  void set_state(const std::complex<double>* data, std::int64_t count, Space space, std::int64_t m0 = 0);
  void get_state(std::complex<double>* data, std::int64_t count, Space space, std::int64_t m0 = 0);

  /// nsteps Strang steps on every member.
  void step(std::int64_t nsteps);
  /// m steps with observables every record_every steps.
  /// Raises numerical_invariant when |norm - norm(0)| at a record step exceeds
  /// the watchdog tolerance (set_watchdog; default 1e-9, 0 = off).
  std::vector<TrajectoryRow> propagate(std::int64_t m, std::int64_t record_every, std::int64_t member = 0);

  std::vector<double> l2_norm();   // per member
  std::vector<double> energy();    // per member
  /// ||u - ref|| for member m, ref in the given space.
  double l2_distance(const std::complex<double>* ref, Space space, std::int64_t member = 0);
  /// ||u - g|| for member m against its discretised initial condition,
  /// formed on the device (time-reversibility checks at sizes whose state
  /// does not fit host memory comfortably, config 4).
  double l2_distance_initial(std::int64_t member = 0);

  /// Device time (ms) of nsteps steps bracketed by events on the solver stream.
  double time_steps(std::int64_t nsteps);
  /// Average device time (ms) per launch of the col and row pass kernels over
  /// nsteps instrumented steps.
  void profile_passes(std::int64_t nsteps, double* ms_col, double* ms_row);
  /// Flush L2 by writing a buffer larger than it.
  void flush_l2();
  void synchronize();

  SolverInfo info() const;
  std::int64_t kernel_launches() const;  // pass + aux kernels launched so far

  /// Device pointers of the propagator tables (for the sharded solver):
  /// 0 = K^ (ROW-pass order, M entries), 1 = V (kappa order, N), 2 = V^(1/2) (N).
  const void* device_table(int which) const;
  int device() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> p_;
  friend cbc::Result cbc::construct_device(i64 n, int d_max, int device);  // uses Impl as an FFT engine
};

}  // namespace lattdse
