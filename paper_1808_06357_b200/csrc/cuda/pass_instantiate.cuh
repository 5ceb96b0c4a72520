// Instantiates and registers the pass kernels of one line length L.
#pragma once

#include "fft_pass.cuh"
#include "pass_registry.hpp"

namespace lattdse::dev {

// Launch geometry per (axis, L):
//  ROW lines are contiguous: one line per CTA for L >= 256, else several.
//  COL lines are strided: B adjacent columns per CTA so every row segment a
//  CTA touches is B*16 bytes (>= one 32-byte sector).
template <int AXIS, int L> struct Geometry {
  static constexpr int B = AXIS == lattdse_dev::AX_ROW ? (L >= 256 ? 1 : 256 / L)
                                                       : (L >= 1024 ? 2 : (L >= 256 ? 4 : 8));
  static constexpr int raw = B * L / 8;
  static constexpr int NT = raw <= 32 ? 32 : (raw >= 256 ? 256 : ((raw + 31) / 32) * 32);
};

template <int AXIS, int L, int PROG, int SIGN> void reg_one() {
  using G = Geometry<AXIS, L>;
  PassKernel k;
  k.fn = reinterpret_cast<const void*>(&lattdse_dev::fft_pass_kernel<AXIS, L, G::B, G::NT, PROG, SIGN>);
  k.B = G::B;
  k.NT = G::NT;
  k.smem = lattdse_dev::SmemGeom<L, G::B>::bytes;
  register_pass_kernel(AXIS, L, PROG, SIGN, k);
}

template <int AXIS, int L> void reg_axis() {
  using namespace lattdse_dev;
  reg_one<AXIS, L, PROG_DOUBLE, -1>();
  reg_one<AXIS, L, PROG_DOUBLE, +1>();
  reg_one<AXIS, L, PROG_LOADDIAG, -1>();
  reg_one<AXIS, L, PROG_LOADDIAG, +1>();
  reg_one<AXIS, L, PROG_STOREDIAG, -1>();
  reg_one<AXIS, L, PROG_STOREDIAG, +1>();
}

}  // namespace lattdse::dev

#define LATTDSE_INSTANTIATE_L(L)                                  \
  namespace {                                                     \
  struct Reg##L {                                                 \
    Reg##L() {                                                    \
      lattdse::dev::reg_axis<lattdse_dev::AX_ROW, L>();           \
      lattdse::dev::reg_axis<lattdse_dev::AX_COL, L>();           \
    }                                                             \
  } reg_instance_##L;                                             \
  }                                                               \
  extern "C" int lattdse_pass_L##L##_linked() { return L; }
