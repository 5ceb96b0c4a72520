// extern "C" layer over the C++ API: no exception crosses the boundary; each
// failure maps lattdse::Errc ordinal k to return code k+1 and stores a
// thread-local message (include/lattdse_c.h).
#include <complex>
#include <cstring>
#include <new>
#include <string>

#include "lattdse/dist.hpp"
#include "lattdse/lattice.hpp"
#include "lattdse/setup.hpp"
#include "lattdse/snapshot.hpp"
#include "lattdse/solver.hpp"
#include "lattdse_c.h"

struct lattdse_lattice {
  lattdse::Lattice lat;
};
struct lattdse_solver {
  std::unique_ptr<lattdse::Solver> s;
  std::int64_t batch = 1;
};
struct lattdse_dist {
  std::unique_ptr<lattdse::DistSolver> d;
};

namespace {

thread_local std::string g_msg;
thread_local int g_code = 0;

int fail(lattdse::Errc c, const std::string& m) {
  g_code = static_cast<int>(c) + 1;
  g_msg = m;
  return g_code;
}

template <class F> int guard(F&& f) {
  try {
    f();
    g_code = 0;
    return 0;
  } catch (const lattdse::Error& e) {
    return fail(e.code(), e.what());
  } catch (const std::bad_alloc&) {
    return fail(lattdse::Errc::device_error, "out of memory");
  } catch (const std::exception& e) {
    return fail(lattdse::Errc::invalid_argument, e.what());
  }
}

void need(const void* p, const char* what) {
  if (!p) lattdse::raise(lattdse::Errc::invalid_argument, std::string(what) + " must not be NULL");
}

lattdse::ProblemSpec make_problem(const lattdse_problem* p) {
  need(p, "problem");
  if (p->dim < 1) lattdse::raise(lattdse::Errc::invalid_argument, "problem dim must be >= 1");
  if (p->batch < 1) lattdse::raise(lattdse::Errc::invalid_argument, "problem batch must be >= 1");
  need(p->a, "problem.a");
  need(p->c, "problem.c");
  need(p->p, "problem.p");
  if (p->dim > 1) need(p->b, "problem.b");
  lattdse::ProblemSpec ps;
  ps.eps = p->eps;
  ps.potential.a.assign(p->a, p->a + p->dim);
  if (p->dim > 1) ps.potential.b.assign(p->b, p->b + p->dim - 1);
  for (std::int64_t m = 0; m < p->batch; ++m) {
    lattdse::problems::Initial g;
    g.sigma = p->sigma;
    g.c.assign(p->c + m * p->dim, p->c + (m + 1) * p->dim);
    g.p.assign(p->p + m * p->dim, p->p + (m + 1) * p->dim);
    ps.initial.push_back(std::move(g));
  }
  return ps;
}

lattdse::SolverOptions make_opts(const lattdse_solver_opts* o) {
  lattdse::SolverOptions so;
  if (o) {
    so.device = o->device;
    so.method = o->method == 1 ? "bluestein" : "circulant";
    so.group = o->group;
    so.force_M1 = o->force_M1;
    so.force_M2 = o->force_M2;
    so.force_M2a = o->force_M2a;
  }
  return so;
}

}  // namespace

extern "C" {

const char* lattdse_last_error(void) { return g_msg.c_str(); }
int lattdse_last_error_code(void) { return g_code; }
#ifndef LATTDSE_EXPERIMENTAL
#define LATTDSE_EXPERIMENTAL 0
#endif
const char* lattdse_version(void) {
  return LATTDSE_EXPERIMENTAL ? "lattdse-b200 0.2.0 (sm_100a, experimental variants)" : "lattdse-b200 0.2.0 (sm_100a)";
}

int lattdse_lattice_create(int dim, int rank, const int64_t* gen, const int64_t* moduli, lattdse_lattice** out) {
  return guard([&] {
    need(out, "out");
    if (dim < 1 || rank < 1) lattdse::raise(lattdse::Errc::invalid_argument, "lattice requires 1 <= rank <= dim");
    need(gen, "gen");
    need(moduli, "moduli");
    std::vector<std::vector<lattdse::i64>> g(rank, std::vector<lattdse::i64>(dim));
    for (int i = 0; i < rank; ++i)
      for (int j = 0; j < dim; ++j) g[i][j] = gen[i * dim + j];
    std::vector<lattdse::i64> n(moduli, moduli + rank);
    *out = new lattdse_lattice{lattdse::Lattice::create(dim, rank, std::move(g), std::move(n))};
  });
}

int lattdse_lattice_rank1(const int64_t* z, int dim, int64_t n, lattdse_lattice** out) {
  return guard([&] {
    need(out, "out");
    if (dim < 1) lattdse::raise(lattdse::Errc::invalid_argument, "lattice requires 1 <= rank <= dim");
    need(z, "z");
    *out = new lattdse_lattice{lattdse::Lattice::rank1(std::vector<lattdse::i64>(z, z + dim), n)};
  });
}

int lattdse_lattice_grid(const int64_t* moduli, int dim, lattdse_lattice** out) {
  return guard([&] {
    need(out, "out");
    if (dim < 1) lattdse::raise(lattdse::Errc::invalid_argument, "lattice requires 1 <= rank <= dim");
    need(moduli, "moduli");
    *out = new lattdse_lattice{lattdse::Lattice::grid(std::vector<lattdse::i64>(moduli, moduli + dim))};
  });
}

int lattdse_lattice_from_json(const char* text, lattdse_lattice** out) {
  return guard([&] {
    need(out, "out");
    need(text, "text");
    *out = new lattdse_lattice{lattdse::Lattice::from_json(text)};
  });
}

void lattdse_lattice_destroy(lattdse_lattice* lat) { delete lat; }

int lattdse_lattice_info(const lattdse_lattice* lat, int* dim, int* rank, int64_t* n_total, int64_t* denom) {
  return guard([&] {
    need(lat, "lattice");
    if (dim) *dim = lat->lat.dim();
    if (rank) *rank = lat->lat.rank();
    if (n_total) *n_total = lat->lat.n_total();
    if (denom) *denom = lat->lat.denom();
  });
}

int lattdse_lattice_generators(const lattdse_lattice* lat, int64_t* gen, int64_t* moduli) {
  return guard([&] {
    need(lat, "lattice");
    const int d = lat->lat.dim(), r = lat->lat.rank();
    for (int i = 0; i < r; ++i) {
      if (gen) {
        auto col = lat->lat.gen_column(i);
        for (int j = 0; j < d; ++j) gen[i * d + j] = col[j];
      }
      if (moduli) moduli[i] = lat->lat.moduli()[i];
    }
  });
}

int lattdse_lattice_hash(const lattdse_lattice* lat, uint64_t* out) {
  return guard([&] {
    need(lat, "lattice");
    need(out, "out");
    *out = lat->lat.hash();
  });
}

int lattdse_lattice_to_json(const lattdse_lattice* lat, char* buf, size_t cap, size_t* needed) {
  return guard([&] {
    need(lat, "lattice");
    const std::string js = lat->lat.to_json();
    if (needed) *needed = js.size() + 1;
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, js.size());
      std::memcpy(buf, js.data(), n);
      buf[n] = '\0';
    }
  });
}

int lattdse_lattice_in_dual(const lattdse_lattice* lat, const int64_t* h, int* out) {
  return guard([&] {
    need(lat, "lattice");
    need(h, "h");
    need(out, "out");
    *out = lat->lat.in_dual(std::span<const lattdse::i64>(h, lat->lat.dim())) ? 1 : 0;
  });
}

int lattdse_lattice_residue(const lattdse_lattice* lat, const int64_t* h, int64_t* xi, int64_t* flat) {
  return guard([&] {
    need(lat, "lattice");
    need(h, "h");
    std::span<const lattdse::i64> hv(h, lat->lat.dim());
    if (xi) {
      auto r = lat->lat.residue(hv);
      std::copy(r.begin(), r.end(), xi);
    }
    if (flat) *flat = lat->lat.flat_residue(hv);
  });
}

int lattdse_lattice_point_numerators(const lattdse_lattice* lat, int64_t first, int64_t count, int64_t* out) {
  return guard([&] {
    need(lat, "lattice");
    need(out, "out");
    const auto& L = lat->lat;
    if (first < 0 || count < 0 || first + count > L.n_total())
      lattdse::raise(lattdse::Errc::invalid_argument, "point range out of bounds");
    if (first == 0 && count == L.n_total()) {
      auto num = L.point_numerators();
      std::copy(num.begin(), num.end(), out);
      return;
    }
    for (int64_t k = 0; k < count; ++k) {
      auto p = L.point(first + k);
      std::copy(p.num.begin(), p.num.end(), out + k * L.dim());
    }
  });
}

int lattdse_lattice_point_index(const lattdse_lattice* lat, int64_t flat_index, int64_t* index) {
  return guard([&] {
    need(lat, "lattice");
    need(index, "index");
    auto p = lat->lat.point(flat_index);
    std::copy(p.index.begin(), p.index.end(), index);
  });
}

int lattdse_wce_squared(const int64_t* z, int dim, int64_t n, double* out) {
  return guard([&] {
    need(z, "z");
    need(out, "out");
    *out = lattdse::cbc::wce_squared(std::span<const lattdse::i64>(z, dim), n);
  });
}

int lattdse_cbc_construct(int64_t n, int d_max, int64_t* z_out, double* wce_out) {
  return guard([&] {
    need(z_out, "z_out");
    auto r = lattdse::cbc::construct(n, d_max);
    std::copy(r.z.begin(), r.z.end(), z_out);
    if (wce_out) std::copy(r.wce.begin(), r.wce.end(), wce_out);
  });
}

int lattdse_aaset_build(const lattdse_lattice* lat, double cap_radius, uint32_t* norm2_out, int16_t* h_out,
                        uint32_t* max_norm2) {
  return guard([&] {
    need(lat, "lattice");
    auto aa = lattdse::AntiAliasSet::build(lat->lat, h_out != nullptr, cap_radius);
    if (norm2_out) std::copy(aa.norm2.begin(), aa.norm2.end(), norm2_out);
    if (h_out) std::copy(aa.h.begin(), aa.h.end(), h_out);
    if (max_norm2) *max_norm2 = aa.max_norm2;
  });
}

int lattdse_cbc_construct_device(int64_t n, int d_max, int device, int64_t* z_out, double* wce_out) {
  return guard([&] {
    need(z_out, "z_out");
    auto r = lattdse::cbc::construct_device(n, d_max, device);
    std::copy(r.z.begin(), r.z.end(), z_out);
    if (wce_out) std::copy(r.wce.begin(), r.wce.end(), wce_out);
  });
}

int lattdse_aaset_norms_device(const lattdse_lattice* lat, int device, double cap_radius, uint32_t* norm2_out,
                               uint32_t* max_norm2) {
  return guard([&] {
    need(lat, "lattice");
    auto aa = lattdse::AntiAliasSet::build_norms_device(lat->lat, device, cap_radius);
    if (norm2_out) std::copy(aa.norm2.begin(), aa.norm2.end(), norm2_out);
    if (max_norm2) *max_norm2 = aa.max_norm2;
  });
}

int lattdse_problem_draw(uint64_t seed, int dim, int64_t batch, double c_lo, double c_hi, int p_max, double* a,
                         double* b, double* c, int* p) {
  return guard([&] {
    if (dim < 1 || batch < 1) lattdse::raise(lattdse::Errc::invalid_argument, "dim and batch must be >= 1");
    lattdse::problems::SplitMix64 rng(seed);
    auto v = lattdse::problems::draw_potential(rng, dim);
    if (a) std::copy(v.a.begin(), v.a.end(), a);
    if (b) std::copy(v.b.begin(), v.b.end(), b);
    for (int64_t m = 0; m < batch; ++m) {
      lattdse::problems::Initial g;
      if (batch == 1) {
        g = lattdse::problems::draw_initial(rng, dim, c_lo, c_hi, p_max, 0.0);
      } else {
        lattdse::problems::SplitMix64 mr(lattdse::problems::member_seed(seed, m));
        g = lattdse::problems::draw_initial(mr, dim, c_lo, c_hi, p_max, 0.0);
      }
      if (c) std::copy(g.c.begin(), g.c.end(), c + m * dim);
      if (p) std::copy(g.p.begin(), g.p.end(), p + m * dim);
    }
  });
}

int lattdse_solver_create(const lattdse_lattice* lat, const lattdse_problem* prob, const lattdse_solver_opts* opts,
                          lattdse_solver** out) {
  return guard([&] {
    need(lat, "lattice");
    need(out, "out");
    auto ps = make_problem(prob);
    // rank-1: the solver builds the norm table on its device (empty norm2);
    // rank >= 2: the host shell walk
    lattdse::AntiAliasSet aa;
    if (lat->lat.rank() != 1) aa = lattdse::AntiAliasSet::build(lat->lat, false);
    auto* h = new lattdse_solver;
    h->batch = prob->batch;
    try {
      h->s = std::make_unique<lattdse::Solver>(lat->lat, aa, ps, make_opts(opts));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int lattdse_solver_create_with_norms(const lattdse_lattice* lat, const uint32_t* norm2, const lattdse_problem* prob,
                                     const lattdse_solver_opts* opts, lattdse_solver** out) {
  return guard([&] {
    need(lat, "lattice");
    need(norm2, "norm2");
    need(out, "out");
    auto ps = make_problem(prob);
    lattdse::AntiAliasSet aa;
    aa.n_total = lat->lat.n_total();
    aa.dim = lat->lat.dim();
    aa.norm2.assign(norm2, norm2 + aa.n_total);
    for (auto x : aa.norm2) aa.max_norm2 = std::max(aa.max_norm2, x);
    auto* h = new lattdse_solver;
    h->batch = prob->batch;
    try {
      h->s = std::make_unique<lattdse::Solver>(lat->lat, aa, ps, make_opts(opts));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void lattdse_solver_destroy(lattdse_solver* s) { delete s; }

#define LD_NEED_S() \
  need(s, "solver"); \
  need(s->s.get(), "solver")

int lattdse_solver_set_dt(lattdse_solver* s, double dt) {
  return guard([&] {
    LD_NEED_S();
    s->s->set_dt(dt);
  });
}

int lattdse_solver_discretize_initial(lattdse_solver* s) {
  return guard([&] {
    LD_NEED_S();
    s->s->discretize_initial();
  });
}

int lattdse_solver_set_state(lattdse_solver* s, const double* c128, int64_t count, int space, int64_t m0) {
  return guard([&] {
    LD_NEED_S();
    need(c128, "state");
    s->s->set_state(reinterpret_cast<const std::complex<double>*>(c128), count,
                    space ? lattdse::Space::coefficients : lattdse::Space::samples, m0);
  });
}

int lattdse_solver_get_state(lattdse_solver* s, double* c128, int64_t count, int space, int64_t m0) {
  return guard([&] {
    LD_NEED_S();
    need(c128, "state");
    s->s->get_state(reinterpret_cast<std::complex<double>*>(c128), count,
                    space ? lattdse::Space::coefficients : lattdse::Space::samples, m0);
  });
}

int lattdse_solver_step(lattdse_solver* s, int64_t nsteps) {
  return guard([&] {
    LD_NEED_S();
    if (nsteps < 0) lattdse::raise(lattdse::Errc::invalid_argument, "nsteps must be >= 0");
    s->s->step(nsteps);
  });
}

int lattdse_solver_l2_norm(lattdse_solver* s, double* out) {
  return guard([&] {
    LD_NEED_S();
    need(out, "out");
    auto v = s->s->l2_norm();
    std::copy(v.begin(), v.end(), out);
  });
}

int lattdse_solver_energy(lattdse_solver* s, double* out) {
  return guard([&] {
    LD_NEED_S();
    need(out, "out");
    auto v = s->s->energy();
    std::copy(v.begin(), v.end(), out);
  });
}

int lattdse_solver_l2_distance(lattdse_solver* s, const double* c128, int space, int64_t member, double* out) {
  return guard([&] {
    LD_NEED_S();
    need(c128, "ref");
    need(out, "out");
    *out = s->s->l2_distance(reinterpret_cast<const std::complex<double>*>(c128),
                             space ? lattdse::Space::coefficients : lattdse::Space::samples, member);
  });
}

int lattdse_solver_propagate(lattdse_solver* s, int64_t m, int64_t record_every, int64_t member, double* rows_out,
                             int64_t* nrows) {
  return guard([&] {
    LD_NEED_S();
    auto rows = s->s->propagate(m, record_every, member);
    if (nrows) *nrows = static_cast<int64_t>(rows.size());
    if (rows_out)
      for (size_t i = 0; i < rows.size(); ++i) {
        rows_out[4 * i + 0] = static_cast<double>(rows[i].step);
        rows_out[4 * i + 1] = rows[i].time;
        rows_out[4 * i + 2] = rows[i].norm;
        rows_out[4 * i + 3] = rows[i].energy;
      }
  });
}

int lattdse_solver_set_watchdog(lattdse_solver* s, double tol) {
  return guard([&] {
    LD_NEED_S();
    s->s->set_watchdog(tol);
  });
}

int lattdse_snapshot_write(const lattdse_lattice* lat, const char* path, const double* c128, int64_t members,
                           int space, int64_t step, double time, double dt) {
  return guard([&] {
    need(lat, "lattice");
    need(path, "path");
    need(c128, "data");
    lattdse::SnapshotMeta m;
    m.members = members;
    m.space = space;
    m.step = step;
    m.time = time;
    m.dt = dt;
    lattdse::snapshot_write(path, lat->lat, reinterpret_cast<const std::complex<double>*>(c128), m);
  });
}

int lattdse_snapshot_probe(const lattdse_lattice* lat, const char* path, int64_t* members, int* space,
                           int64_t* step, double* time, double* dt) {
  return guard([&] {
    need(lat, "lattice");
    need(path, "path");
    auto m = lattdse::snapshot_probe(path, lat->lat);
    if (members) *members = m.members;
    if (space) *space = m.space;
    if (step) *step = m.step;
    if (time) *time = m.time;
    if (dt) *dt = m.dt;
  });
}

int lattdse_snapshot_read(const lattdse_lattice* lat, const char* path, double* c128, int64_t capacity) {
  return guard([&] {
    need(lat, "lattice");
    need(path, "path");
    need(c128, "data");
    lattdse::snapshot_read(path, lat->lat, reinterpret_cast<std::complex<double>*>(c128), capacity);
  });
}

int lattdse_solver_l2_distance_initial(lattdse_solver* s, int64_t member, double* out) {
  return guard([&] {
    LD_NEED_S();
    need(out, "out");
    *out = s->s->l2_distance_initial(member);
  });
}

int lattdse_solver_info_get(lattdse_solver* s, lattdse_solver_info* out) {
  return guard([&] {
    LD_NEED_S();
    need(out, "out");
    auto i = s->s->info();
    out->n_total = i.n_total;
    out->batch = i.batch;
    out->M = i.M;
    out->M1 = i.M1;
    out->M2 = i.M2;
    out->group = i.group;
    out->rank = i.rank;
    out->method = i.method.rfind("bluestein", 0) == 0 ? 1 : (i.method == "grid" ? 2 : 0);
    out->bytes_per_step = i.bytes_per_step;
    out->bytes_per_pass_col = i.bytes_per_pass_col;
    out->bytes_per_pass_row = i.bytes_per_pass_row;
    out->launches_per_step = i.launches_per_step;
    out->M2a = i.M2a;
    out->row_chunk = i.row_chunk;
    out->pass4 = i.pass4;
  });
}

int lattdse_solver_time_steps(lattdse_solver* s, int64_t nsteps, double* ms) {
  return guard([&] {
    LD_NEED_S();
    need(ms, "ms");
    *ms = s->s->time_steps(nsteps);
  });
}

int lattdse_solver_profile_passes(lattdse_solver* s, int64_t nsteps, double* ms_col, double* ms_row) {
  return guard([&] {
    LD_NEED_S();
    need(ms_col, "ms_col");
    need(ms_row, "ms_row");
    s->s->profile_passes(nsteps, ms_col, ms_row);
  });
}

int lattdse_solver_flush_l2(lattdse_solver* s) {
  return guard([&] {
    LD_NEED_S();
    s->s->flush_l2();
  });
}

int lattdse_solver_kernel_launches(lattdse_solver* s, int64_t* out) {
  return guard([&] {
    LD_NEED_S();
    need(out, "out");
    *out = s->s->kernel_launches();
  });
}

int lattdse_dist_nccl_unique_id(uint8_t* out128) {
  return guard([&] {
    need(out128, "out");
    lattdse::DistSolver::nccl_unique_id(out128);
  });
}

int lattdse_dist_create(const lattdse_lattice* lat, const uint32_t* norm2, const lattdse_problem* prob, int world,
                        int rank, int device, const uint8_t* nccl_id, lattdse_dist** out) {
  return guard([&] {
    need(lat, "lattice");
    need(out, "out");
    auto ps = make_problem(prob);
    lattdse::AntiAliasSet aa;
    if (norm2) {
      aa.n_total = lat->lat.n_total();
      aa.dim = lat->lat.dim();
      aa.norm2.assign(norm2, norm2 + aa.n_total);
      for (auto x : aa.norm2) aa.max_norm2 = std::max(aa.max_norm2, x);
    }  // else: empty table -- the table-building solver builds the norms on its device (rank-1)
    lattdse::DistOptions o;
    o.world = world;
    o.rank = rank;
    o.device = device;
    o.nccl_id = nccl_id;
    auto* h = new lattdse_dist;
    try {
      h->d = std::make_unique<lattdse::DistSolver>(lat->lat, aa, ps, o);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void lattdse_dist_destroy(lattdse_dist* d) { delete d; }

#define LD_NEED_D() \
  need(d, "dist");  \
  need(d->d.get(), "dist")

int lattdse_dist_set_dt(lattdse_dist* d, double dt) {
  return guard([&] {
    LD_NEED_D();
    d->d->set_dt(dt);
  });
}
int lattdse_dist_discretize_initial(lattdse_dist* d) {
  return guard([&] {
    LD_NEED_D();
    d->d->discretize_initial();
  });
}
int lattdse_dist_set_state(lattdse_dist* d, const double* c128) {
  return guard([&] {
    LD_NEED_D();
    need(c128, "state");
    d->d->set_state(reinterpret_cast<const std::complex<double>*>(c128));
  });
}
int lattdse_dist_get_state(lattdse_dist* d, double* c128) {
  return guard([&] {
    LD_NEED_D();
    need(c128, "state");
    d->d->get_state(reinterpret_cast<std::complex<double>*>(c128));
  });
}
int lattdse_dist_step(lattdse_dist* d, int64_t nsteps) {
  return guard([&] {
    LD_NEED_D();
    d->d->step(nsteps);
  });
}
int lattdse_dist_l2_norm(lattdse_dist* d, double* out) {
  return guard([&] {
    LD_NEED_D();
    need(out, "out");
    *out = d->d->l2_norm();
  });
}
int lattdse_dist_time_steps(lattdse_dist* d, int64_t nsteps, double* ms) {
  return guard([&] {
    LD_NEED_D();
    need(ms, "ms");
    *ms = d->d->time_steps(nsteps);
  });
}
int lattdse_dist_info(lattdse_dist* d, int64_t* M, int64_t* M1, int64_t* M2, double* exchange_bytes) {
  return guard([&] {
    LD_NEED_D();
    if (M) *M = d->d->M();
    if (M1) *M1 = d->d->M1();
    if (M2) *M2 = d->d->M2();
    if (exchange_bytes) *exchange_bytes = d->d->exchange_bytes_per_rank();
  });
}

int lattdse_dist_table_peak_bytes(lattdse_dist* d, double* bytes) {
  return guard([&] {
    LD_NEED_D();
    need(bytes, "bytes");
    *bytes = d->d->table_peak_bytes();
  });
}

int lattdse_dist_three_level(lattdse_dist* d, int64_t* Ma, int64_t* Mb) {
  return guard([&] {
    LD_NEED_D();
    need(Ma, "Ma");
    need(Mb, "Mb");
    *Ma = d->d->Ma();
    *Mb = *Ma > 0 ? d->d->M2() / *Ma : 0;
  });
}

int lattdse_solver_synchronize(lattdse_solver* s) {
  return guard([&] {
    LD_NEED_S();
    s->s->synchronize();
  });
}

}  // extern "C"
