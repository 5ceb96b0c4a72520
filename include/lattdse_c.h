/*
 * lattdse C ABI -- the drop-in boundary of the B200 hot path.
 *
 * The reference (arXiv 1808.06357 artifact, /root/reference) is a C++ library
 * whose only implemented module is lattice-core
 * (proj/src/core/lattice.hpp:31-86, errors.hpp:8-34); its solver surface is
 * specified in SPEC.md (cbc :104-161, antialias :163-222, spectral :224-306,
 * tdse :308-399). Every entry point below cites the reference interface it
 * replaces. Plain C types only: no CUDA or torch types cross this boundary.
 *
 * Return codes: 0 = OK; k+1 = lattdse::Errc ordinal k (errors.hpp:8-22):
 *   1 invalid_argument, 2 non_divisible_moduli, 3 non_coprime_component,
 *   4 rank_deficient, 5 point_count_mismatch, 6 overflow_risk,
 *   7 radius_exhausted, 8 spec_mismatch, 9 non_normalizable, 10 config_error,
 *   11 reference_too_coarse, 12 numerical_invariant, 13 io_error,
 *   appended (never renumbered): 14 device_error, 15 unsupported, 16 nccl_error.
 * lattdse_last_error() returns the thread-local message of the last failure.
 *
 * Complex buffers are little-endian interleaved complex128 (re, im), the
 * snapshot format of SPEC.md:299. Host arrays belong to the caller and are
 * copied; device memory and streams belong to the handle. A handle is not
 * internally synchronised; calls are synchronous at return.
 */
#ifndef LATTDSE_C_H
#define LATTDSE_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lattdse_lattice lattdse_lattice;
typedef struct lattdse_solver lattdse_solver;

/* ---- errors (errors.hpp:25-34) ---------------------------------------- */
const char* lattdse_last_error(void);
int lattdse_last_error_code(void);
const char* lattdse_version(void);

/* ---- lattice-core (lattice.hpp:34-72, lattice.cpp:167-364) ------------- */
/* Lattice::create(dim, rank, gen, moduli); gen holds rank columns of length
 * dim, column i at gen[i*dim .. i*dim+dim-1]. */
int lattdse_lattice_create(int dim, int rank, const int64_t* gen, const int64_t* moduli, lattdse_lattice** out);
/* Lattice::rank1(z, n) (lattice.hpp:41; fixed evaluation-order bug of lattice.cpp:237-239) */
int lattdse_lattice_rank1(const int64_t* z, int dim, int64_t n, lattdse_lattice** out);
/* Lattice::grid(moduli) (lattice.hpp:43) */
int lattdse_lattice_grid(const int64_t* moduli, int dim, lattdse_lattice** out);
/* Lattice::from_json (lattice.hpp:70) */
int lattdse_lattice_from_json(const char* text, lattdse_lattice** out);
void lattdse_lattice_destroy(lattdse_lattice* lat);
/* dim(), rank(), n_total(), denom() (lattice.hpp:45-48) */
int lattdse_lattice_info(const lattdse_lattice* lat, int* dim, int* rank, int64_t* n_total, int64_t* denom);
/* moduli() and gen_column(i) (lattice.hpp:49-51) copied out */
int lattdse_lattice_generators(const lattdse_lattice* lat, int64_t* gen, int64_t* moduli);
/* hash() (lattice.hpp:66) */
int lattdse_lattice_hash(const lattdse_lattice* lat, uint64_t* out);
/* to_json() (lattice.hpp:69): writes up to cap bytes incl. NUL; *needed = strlen+1 */
int lattdse_lattice_to_json(const lattdse_lattice* lat, char* buf, size_t cap, size_t* needed);
/* in_dual / residue / flat_residue (lattice.hpp:54-59) */
int lattdse_lattice_in_dual(const lattdse_lattice* lat, const int64_t* h, int* out);
int lattdse_lattice_residue(const lattdse_lattice* lat, const int64_t* h, int64_t* xi, int64_t* flat);
/* point_numerators() rows [first, first+count) (lattice.hpp:61-62) and the
 * point(flat_index) multi-index (lattice.hpp:60) */
int lattdse_lattice_point_numerators(const lattdse_lattice* lat, int64_t first, int64_t count, int64_t* out);
int lattdse_lattice_point_index(const lattdse_lattice* lat, int64_t flat_index, int64_t* index);

/* ---- cbc -------------------------------------------- */
int lattdse_wce_squared(const int64_t* z, int dim, int64_t n, double* out);
/* z_out[d_max], wce_out[d_max] (criterion after each component, may be NULL) */
int lattdse_cbc_construct(int64_t n, int d_max, int64_t* z_out, double* wce_out);
/* The same construction on CUDA device `device` (prime n > 64, n < 2^31):
 * the shortlisting correlation runs through the solver's length-M FFT. */
int lattdse_cbc_construct_device(int64_t n, int d_max, int device, int64_t* z_out, double* wce_out);

/* ---- antialias -------------------------------------- */
/* norm2_out[n_total] = ||h^(chi)||^2; h_out[n_total*dim] (int16) or NULL;
 * cap_radius <= 0 selects SPEC's default 4 n^(1/d) + 16. */
int lattdse_aaset_build(const lattdse_lattice* lat, double cap_radius, uint32_t* norm2_out, int16_t* h_out,
                        uint32_t* max_norm2);
/* The same norm table built on CUDA device `device` (rank-1, N < 2^31;
 * meet-in-the-middle shell walk, csrc/cuda/aaset_dev.cu). norm2_out may be
 * NULL (then only *max_norm2 is reported). */
int lattdse_aaset_norms_device(const lattdse_lattice* lat, int device, double cap_radius, uint32_t* norm2_out,
                               uint32_t* max_norm2);

/* ---- problem families (BASELINE.json configs; SPEC.md:313-317 slots) --- */
typedef struct lattdse_problem {
  double eps;        /* semiclassical scale (paper's gamma~) */
  int dim;
  const double* a;   /* dim:    v = sum a_j (1 - cos 2 pi x_j) + ...     */
  const double* b;   /* dim-1:  ... + sum b_j cos 2 pi (x_j - x_{j+1})   */
  int64_t batch;     /* ensemble members                                  */
  double sigma;
  const double* c;   /* batch*dim  g centres                              */
  const int* p;      /* batch*dim  g momenta                              */
} lattdse_problem;

/* Seeded draw of (a, b) and member (c, p) -- the documented seed schedule
 * (DESIGN.md "Seeds"). a[dim], b[dim-1], c[batch*dim], p[batch*dim]. */
int lattdse_problem_draw(uint64_t seed, int dim, int64_t batch, double c_lo, double c_hi, int p_max, double* a,
                         double* b, double* c, int* p);

/* ---- solver (StrangPropagator/strang_step/propagate) --- */
typedef struct lattdse_solver_opts {
  int device;        /* CUDA device ordinal                                */
  int method;        /* rank-1: 0 circulant (default), 1 literal Bluestein */
  int64_t group;     /* members stepped together (0 = auto, L2-sized)      */
  /* rank-1 transform view (0 = automatic): M = force_M1 x force_M2; with
   * force_M2a > 0 each row splits three-level as force_M2a x (M2/force_M2a) */
  int64_t force_M1, force_M2, force_M2a;
} lattdse_solver_opts;

typedef struct lattdse_solver_info {
  int64_t n_total, batch, M, M1, M2, group;
  int rank, method;
  double bytes_per_step, bytes_per_pass_col, bytes_per_pass_row;
  int launches_per_step;
  int64_t M2a;       /* three-level inner split of M2 (0: two-level) */
  int64_t row_chunk; /* three-level: M1 rows per L2-resident row-side chunk (0: whole view) */
  int pass4;         /* 1: per-step passes have run on the lean plain-layout kernels (fft_pass4.cuh) */
} lattdse_solver_info;

/* Builds the anti-aliasing norm table, potential samples and device state. */
int lattdse_solver_create(const lattdse_lattice* lat, const lattdse_problem* prob, const lattdse_solver_opts* opts,
                          lattdse_solver** out);
/* Same, with a precomputed norm table (e.g. loaded from the aaset JSON). */
int lattdse_solver_create_with_norms(const lattdse_lattice* lat, const uint32_t* norm2, const lattdse_problem* prob,
                                     const lattdse_solver_opts* opts, lattdse_solver** out);
void lattdse_solver_destroy(lattdse_solver* s);
/* StrangPropagator for dt */
int lattdse_solver_set_dt(lattdse_solver* s, double dt);
/* discretize_initial for every member */
int lattdse_solver_discretize_initial(lattdse_solver* s);
/* space: 0 samples (kappa order), 1 coefficients (chi order); members [m0, m0+count) */
int lattdse_solver_set_state(lattdse_solver* s, const double* c128, int64_t count, int space, int64_t m0);
int lattdse_solver_get_state(lattdse_solver* s, double* c128, int64_t count, int space, int64_t m0);
/* nsteps x strang_step on every member */
int lattdse_solver_step(lattdse_solver* s, int64_t nsteps);
/* l2_norm / energy per member; out[batch] */
int lattdse_solver_l2_norm(lattdse_solver* s, double* out);
int lattdse_solver_energy(lattdse_solver* s, double* out);
/* ||u_member - ref|| with ref in `space` */
int lattdse_solver_l2_distance(lattdse_solver* s, const double* c128, int space, int64_t member, double* out);
/* ||u - g|| against the member's discretised initial condition (device-side) */
int lattdse_solver_l2_distance_initial(lattdse_solver* s, int64_t member, double* out);
/* propagate: rows (step, time, norm, energy) for `member`;
 * rows_out holds floor(m/record_every)+2 rows of 4 doubles; *nrows set. */
int lattdse_solver_propagate(lattdse_solver* s, int64_t m, int64_t record_every, int64_t member, double* rows_out,
                             int64_t* nrows);
int lattdse_solver_info_get(lattdse_solver* s, lattdse_solver_info* out);
/* norm-drift watchdog of propagate: numerical_invariant (12) when
 * |norm - norm(0)| > tol at a record step; default 1e-9, 0 disables */
int lattdse_solver_set_watchdog(lattdse_solver* s, double tol);

/* ---- state snapshots (include/lattdse/snapshot.hpp) -----
 * `path` holds members*N little-endian complex128; `path`.json the sidecar
 * (length, ordering, lattice + hash, step, time, dt). probe/read check the
 * sidecar against `lat`: config_error (10) on mismatch, io_error (13) on
 * missing/short files. space: 0 samples (kappa order), 1 coefficients (chi). */
int lattdse_snapshot_write(const lattdse_lattice* lat, const char* path, const double* c128, int64_t members,
                           int space, int64_t step, double time, double dt);
int lattdse_snapshot_probe(const lattdse_lattice* lat, const char* path, int64_t* members, int* space,
                           int64_t* step, double* time, double* dt);
int lattdse_snapshot_read(const lattdse_lattice* lat, const char* path, double* c128, int64_t capacity);

/* ---- measurement hooks (bench.py) -------------------------------------- */
int lattdse_solver_time_steps(lattdse_solver* s, int64_t nsteps, double* ms);
int lattdse_solver_profile_passes(lattdse_solver* s, int64_t nsteps, double* ms_col, double* ms_row);
int lattdse_solver_flush_l2(lattdse_solver* s);
int lattdse_solver_kernel_launches(lattdse_solver* s, int64_t* out);
/* wait for all work queued on the solver stream */
int lattdse_solver_synchronize(lattdse_solver* s);

/* ---- sharded single wave function (SURVEY.md §8(e), config 4 strategy) --
 * world ranks; rank = -1 runs all ranks as virtual ranks on `device` (block
 * exchanges by device copies), rank >= 0 is one process per GPU with NCCL
 * grouped send/recv (nccl_id from lattdse_dist_nccl_unique_id on rank 0).
 * norm2 = NULL: the norm table is built on the device (rank-1 lattices). */
typedef struct lattdse_dist lattdse_dist;
int lattdse_dist_nccl_unique_id(uint8_t* out128);
int lattdse_dist_create(const lattdse_lattice* lat, const uint32_t* norm2, const lattdse_problem* prob, int world,
                        int rank, int device, const uint8_t* nccl_id, lattdse_dist** out);
void lattdse_dist_destroy(lattdse_dist* d);
int lattdse_dist_set_dt(lattdse_dist* d, double dt);
int lattdse_dist_discretize_initial(lattdse_dist* d);
/* full kappa-order sample vectors (N complex128); NCCL ranks touch only theirs */
int lattdse_dist_set_state(lattdse_dist* d, const double* c128);
int lattdse_dist_get_state(lattdse_dist* d, double* c128);
int lattdse_dist_step(lattdse_dist* d, int64_t nsteps);
int lattdse_dist_l2_norm(lattdse_dist* d, double* out);
int lattdse_dist_time_steps(lattdse_dist* d, int64_t nsteps, double* ms);
/* M, M1, M2 of the sharded view; bytes each rank sends per exchange (2/step) */
int lattdse_dist_info(lattdse_dist* d, int64_t* M, int64_t* M1, int64_t* M2, double* exchange_bytes);
/* device bytes one rank held at the peak of the last set_dt (slabs + transient table slabs + norm index) */
int lattdse_dist_table_peak_bytes(lattdse_dist* d, double* bytes);
/* three-level row layout M2 = Ma x Mb of config-4-sized N (Ma = Mb = 0: two-level) */
int lattdse_dist_three_level(lattdse_dist* d, int64_t* Ma, int64_t* Mb);

#ifdef __cplusplus
}
#endif

#endif /* LATTDSE_C_H */
