// TEST INFRASTRUCTURE ONLY -- C shim over the reference's own lattice-core
// (/root/reference/proj/src/core/lattice.{hpp,cpp}), compiled in place by
// oracle/build_ref.sh into oracle/_ref/libref_lattice.so. Used solely to
// generate the golden fixtures in tests/golden/ (make_lattice_golden.py).
// Calls Lattice::create (the reference's rank1() always throws under GCC,
// lattice.cpp:237-239).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "lattice.hpp"

using lattdse::Lattice;

extern "C" {

int ref_lattice_create(int dim, int rank, const int64_t* gen, const int64_t* moduli, void** out, char* err,
                       int errcap) {
  try {
    std::vector<std::vector<lattdse::i64>> g(rank, std::vector<lattdse::i64>(dim));
    for (int i = 0; i < rank; ++i)
      for (int j = 0; j < dim; ++j) g[i][j] = gen[i * dim + j];
    std::vector<lattdse::i64> n(moduli, moduli + rank);
    *out = new Lattice(Lattice::create(dim, rank, g, n));
    return 0;
  } catch (const lattdse::Error& e) {
    std::strncpy(err, e.what(), errcap - 1);
    err[errcap - 1] = 0;
    return static_cast<int>(e.code()) + 1;
  }
}

int ref_lattice_rank1_raw(const int64_t* z, int dim, int64_t n, char* err, int errcap) {
  try {
    Lattice::rank1(std::vector<lattdse::i64>(z, z + dim), n);
    return 0;
  } catch (const lattdse::Error& e) {
    std::strncpy(err, e.what(), errcap - 1);
    err[errcap - 1] = 0;
    return static_cast<int>(e.code()) + 1;
  }
}

void ref_lattice_destroy(void* p) { delete static_cast<Lattice*>(p); }
uint64_t ref_lattice_hash(void* p) { return static_cast<Lattice*>(p)->hash(); }
int64_t ref_lattice_denom(void* p) { return static_cast<Lattice*>(p)->denom(); }

int ref_lattice_to_json(void* p, char* buf, int cap) {
  std::string s = static_cast<Lattice*>(p)->to_json();
  std::strncpy(buf, s.c_str(), cap - 1);
  buf[cap - 1] = 0;
  return static_cast<int>(s.size());
}

void ref_lattice_points(void* p, int64_t* out) {
  auto v = static_cast<Lattice*>(p)->point_numerators();
  std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
}

void ref_lattice_residue(void* p, const int64_t* h, int64_t* xi, int64_t* flat, int* dual) {
  auto* L = static_cast<Lattice*>(p);
  std::span<const lattdse::i64> hv(h, L->dim());
  auto r = L->residue(hv);
  std::memcpy(xi, r.data(), r.size() * sizeof(int64_t));
  *flat = L->flat_residue(hv);
  *dual = L->in_dual(hv) ? 1 : 0;
}

int ref_lattice_from_json(const char* text, void** out, char* err, int errcap) {
  try {
    *out = new Lattice(Lattice::from_json(text));
    return 0;
  } catch (const lattdse::Error& e) {
    std::strncpy(err, e.what(), errcap - 1);
    err[errcap - 1] = 0;
    return static_cast<int>(e.code()) + 1;
  }
}
}
