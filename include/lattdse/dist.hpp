// lattdse::DistSolver -- one rank-1 wave function sharded across G ranks
// (SURVEY.md §8(e), config 4's strategy): the length-M convolution's four-step
// FFT runs its COL passes on column slabs (M1 x M2/G per rank) and its ROW
// passes on row slabs (M1/G x M2 per rank, stored block-major so every
// exchanged block is contiguous on both sides). Between passes the ranks
// exchange G x G blocks of (M1/G) x (M2/G) elements: two all-to-alls per
// Strang step (the circulant step; the literal Bluestein step would need four).
// Beyond one COL x ROW split (config 4) each row is itself an Ma x Mb
// four-step handled locally on the row slab: still two exchanges per step.
//
// Exchange backends:
//  - "local": all G ranks live on one device (virtual ranks); blocks move
//    with device-to-device copies. Exercises every kernel and index map of
//    the sharded path on a single GPU (tests/test_gpu_parity.py).
//  - "nccl": one process per GPU; grouped ncclSend/ncclRecv per exchange
//    (libnccl.so.2 is dlopen'ed; the unique id comes from rank 0).
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <vector>

#include "solver.hpp"

namespace lattdse {

struct DistOptions {
  int world = 2;            // G ranks
  int rank = -1;            // this process's rank; -1 = all ranks virtual on `device`
  int device = 0;
  const void* nccl_id = nullptr;  // 128-byte ncclUniqueId (rank >= 0)
};

class DistSolver {
 public:
  DistSolver(const Lattice& lat, const AntiAliasSet& aa, const ProblemSpec& prob, const DistOptions& opt);
  ~DistSolver();
  DistSolver(const DistSolver&) = delete;
  DistSolver& operator=(const DistSolver&) = delete;

  void set_dt(double dt);
  void discretize_initial();
  /// samples of the whole wave function (kappa order); in NCCL mode only the
  /// entries this rank owns are written/read (others untouched / ignored).
  void set_state(const std::complex<double>* samples);
  void get_state(std::complex<double>* samples);
  void step(std::int64_t nsteps);
  double l2_norm();  // over all ranks
  double time_steps(std::int64_t nsteps);

  std::int64_t M() const;
  std::int64_t M1() const;
  std::int64_t M2() const;
  /// three-level layout (M2 = Ma * Mb); 0 when the rows are one ROW pass
  std::int64_t Ma() const;
  int world() const;
  /// bytes each rank sends per exchange (two exchanges per step)
  double exchange_bytes_per_rank() const;
  /// device bytes one rank held at the peak of the last set_dt (its slabs,
  /// the transient table slabs and the norm index): scales as 1/G
  double table_peak_bytes() const;

  static void nccl_unique_id(void* out128);

 private:
  void set_dt_full_table(double dt);
  struct Impl;
  std::unique_ptr<Impl> p_;
};

}  // namespace lattdse
