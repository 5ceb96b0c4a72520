// Instantiates and registers the pass kernels of one line length L.
#pragma once

#include "fft_pass.cuh"
#include "fft_pass3.cuh"
#include "pass_registry.hpp"

#ifndef LATTDSE_BUILD_PASS3
#define LATTDSE_BUILD_PASS3 1  // persistent TMA-fed per-step passes (fft_pass3.cuh)
#endif
#ifndef LATTDSE_COL_B1_MIN
#define LATTDSE_COL_B1_MIN 8192  // columns this long: one column per CTA
#endif

namespace lattdse::dev {

// Launch geometry per (axis, L):
//  ROW lines are contiguous: one line per CTA for L >= 256, else several.
//  COL lines are strided: B adjacent columns per CTA so every row segment a
//  CTA touches is B*16 bytes (>= one 32-byte sector).
// NT covers the busiest stage (B * L / R_min tasks) so no thread loops.
//  COL lines of 4096 (config 2): two columns per CTA (32-byte row segments)
//  at two tasks per thread, one CTA per SM with ~250 registers and no spills
//  (measured 314 us vs 393 us for one column per CTA, profiles/README.md).
template <int AXIS, int L> struct Geometry {
  static constexpr bool wide_col = AXIS == lattdse_dev::AX_COL && L >= 4096 && L < LATTDSE_COL_B1_MIN;
  // COL 512 (the power-of-two view 512 x 4096 of config 1): four columns
  // (64-byte row segments) at 256 threads, measured 32.1 us vs 79 us for two
  // columns at 512 threads (profiles/README.md)
  static constexpr bool col512 = AXIS == lattdse_dev::AX_COL && L == 512;
  static constexpr int B = AXIS == lattdse_dev::AX_ROW ? (L >= 256 ? 1 : 256 / L)
                                                       : (L >= LATTDSE_COL_B1_MIN ? 1 : (L >= 512 && !col512 ? 2 : (L >= 128 ? 4 : 8)));
  static constexpr int raw = B * lattdse_dev::Plan<L>::max_tasks();
  static constexpr int NT = (wide_col || col512) ? 256 : (raw <= 32 ? 32 : (raw >= 512 ? 512 : ((raw + 31) / 32) * 32));
  // pass3 (persistent, TMA-fed): CTAs per SM by shared memory, and the
  // register cap that keeps that many resident
  using G3 = lattdse_dev::Pass3Geom<AXIS, L, B>;
  static constexpr int smem3 = G3::bytes;
  static constexpr int ctas3 = (228 * 1024) / (smem3 + 1024);
  // resident CTAs: as many as shared memory allows, at most what ~96
  // registers per thread allow (the v1 kernels' budget; more registers cost
  // warps, measured profiles/r2c: 166 regs -> 0.69x the warps on ROW 486)
  static constexpr int by_regs = 65536 / (NT * 96) > 0 ? 65536 / (NT * 96) : 1;
  static constexpr int mb3 = ctas3 < 1 ? 1 : (ctas3 < by_regs ? ctas3 : by_regs);
};

template <int AXIS, int L, int PROG, int SIGN> void reg_one() {
  using G = Geometry<AXIS, L>;
  PassKernel k;
  k.fn = reinterpret_cast<const void*>(&lattdse_dev::fft_pass_kernel<AXIS, L, G::B, G::NT, PROG, SIGN>);
  k.B = G::B;
  k.NT = G::NT;
  k.smem = lattdse_dev::SmemGeom<L, G::B>::bytes;
  k.nst = lattdse_dev::Plan<L>::nst;
  for (int s = 0; s < k.nst && s < 16; ++s) k.radix[s] = lattdse_dev::Plan<L>::radix(s);
  if constexpr (PROG == lattdse_dev::PROG_DOUBLE) {
    k.fn_mb[1] = k.fn;
    k.fn_mb[2] = reinterpret_cast<const void*>(&lattdse_dev::fft_pass_kernel<AXIS, L, G::B, G::NT, PROG, SIGN, 2>);
    k.fn_mb[3] = reinterpret_cast<const void*>(&lattdse_dev::fft_pass_kernel<AXIS, L, G::B, G::NT, PROG, SIGN, 3>);
    k.fn_mb[4] = nullptr;  // measured never best (spills); not instantiated to keep the library small
    // measured on C1 (profiles/README.md): 3 resident CTAs/SM balance register
    // caps (small L1-resident spills) against occupancy for 5-10 warp CTAs
    // ROW: 3 CTAs/SM; COL (four-step twiddle math in the fused stages) keeps
    // more registers at 2 CTAs/SM
    // ROW lines of 4096 (radix-16 stages) spill heavily under the 3-CTA cap
    k.default_mb = G::wide_col ? 1 : (G::NT > 320 ? 2 : (AXIS == lattdse_dev::AX_ROW && L < 4096 ? 3 : 2));
  }
  if constexpr (LATTDSE_BUILD_PASS3 && PROG == lattdse_dev::PROG_DOUBLE && G::smem3 <= 227 * 1024) {
    k.fn3 = reinterpret_cast<const void*>(&lattdse_dev::fft_pass3_kernel<AXIS, L, G::B, G::NT, SIGN, G::mb3>);
    k.smem3 = G::smem3;
    k.boxr3 = G::G3::boxr;
  }
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
