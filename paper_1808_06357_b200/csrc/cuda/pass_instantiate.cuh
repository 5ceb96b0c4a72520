// Instantiates and registers the pass kernels of one line length L.
#pragma once

#include "fft_pass.cuh"
#include "fft_pass4.cuh"
#include "pass_registry.hpp"

#ifndef LATTDSE_BUILD_PASS4
#define LATTDSE_BUILD_PASS4 1  // lean per-step passes of the plain layouts (fft_pass4.cuh)
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
};

// pass4 launch geometry per (axis, L), from the sweeps of fft_pass4_devtest
// (profiles/r2/p4_sweep*.txt; us per launch, config-3 shapes over 64 members
// unless noted):
//  ROW: one line per CTA (two below 512, more for short lines); two stage
//       buffers (one barrier per stage) for plans with a radix above 12
//       while both fit 72 KB, in place otherwise;
//  COL: more, smaller CTAs beat wider tiles -- L <= 648: four adjacent
//       columns (64-byte row segments) in place, COL 486 four CTAs of 224
//       threads 348 vs two CTAs of eight columns 366 vs v1 441; longer
//       columns two per CTA (also 4096: 262 vs 338 for one column), with
//       two stage buffers while they fit 90 KB (config 1, COL 1296: 35.0 vs
//       39.0 in place vs v1 39.7);
//  NT covers the busiest stage unless a narrower CTA running that stage in
//  two rounds wastes fewer thread slots; resident CTAs per SM as ~96 (two
//  buffers) or ~72 (in place) registers per thread and the shared memory
//  allow (ROW 1080: 5 CTAs of 128 threads 271, 6 CTAs at 80 registers 293).
// Plans whose first or last radix is a multiple of 4 run with swizzled
// slots (P4Seq::swz; ROW 4096 163 vs 259 unswizzled vs v1 216, COL 4096 two
// columns 262 vs v1 303 on config 2, ROW 2048 139 vs v1 219); the few such
// plans the swizzle cannot keep affine (512, 1024: a radix-2 / 4 end stage
// behind radix 16) stay on the v1 kernels.
// WIDE: the eight-column variant of short COL lines (L <= 648), used when the
// rows of the view lie megabytes apart (config 4's first-level pass: row
// stride 70 MB, every 64-byte segment its own DRAM page; 128-byte segments
// 32.1 vs 35.2 ms per launch), while config 3 (row stride 17 KB) keeps four
// columns (equal in the sustained bench, 5% faster at boost clocks)
template <int AXIS, int L, bool WIDE = false> struct Geometry4 {
  using P = lattdse_dev::Plan<L>;
  static constexpr bool row = AXIS == lattdse_dev::AX_ROW;
  static constexpr bool ok = P::nst >= 2 && L >= 64 && lattdse_dev::P4Seq<L>::swz_ok() && (!WIDE || (!row && L <= 648));
  static constexpr int B = row ? (L >= 512 ? 1 : (L >= 256 ? 2 : 256 / L * 2)) : (L <= 648 ? (WIDE ? 8 : 4) : 2);
  // threads: the multiple of 32 with the fewest thread slots over the stage
  // sequence (a stage of t tasks runs ceil(t / NT) rounds of NT threads,
  // each task R elements of work; the fused mid stage runs once with two
  // transforms' worth, the others once per direction), at most two rounds
  // per stage and those charged 25% extra (two tasks' registers live at
  // once); ties to the larger CTA
  static constexpr long long waste(int nt) {
    long long w = 0;
    for (int s = 0; s < P::nst; ++s) {
      const int R = P::radix(s), t = B * (L / R), rounds = (t + nt - 1) / nt;
      if (rounds > 2) return -1;
      w += (long long)rounds * nt * R * (rounds > 1 ? 5 : 4);
    }
    return w;
  }
  static constexpr int pick_nt() {
    int best = 512;
    long long bw = -1;
    for (int nt = 64; nt <= 512; nt += 32) {
      const long long w = waste(nt);
      if (w >= 0 && (bw < 0 || w <= bw)) {
        bw = w;
        best = nt;
      }
    }
    return best;
  }
  static constexpr int NT = pick_nt();
  // registers per thread the kernel is capped to (resident CTAs by registers):
  // radix-16 end stages 128, else 96 with two stage buffers or a radix >= 15
  // anywhere, 72 in place with small radices
  static constexpr bool big = P::radix(0) >= 16 || P::radix(P::nst - 1) >= 16;
  static constexpr int max_radix() {
    int m = 0;
    for (int s = 0; s < P::nst; ++s) m = P::radix(s) > m ? P::radix(s) : m;
    return m;
  }
  static constexpr int ip_budget = big ? 128 : (max_radix() >= 15 ? 96 : (row ? 80 : 72));
  static constexpr int fit(int bytes) { return (227 * 1024) / (bytes + 1024) > 0 ? (227 * 1024) / (bytes + 1024) : 1; }
  static constexpr int regs_ctas(int budget) { return 65536 / (NT * budget) > 0 ? 65536 / (NT * budget) : 1; }
  static constexpr int bytes_pp = lattdse_dev::P4Geom<AXIS, L, B, 1, true>::bytes;
  static constexpr int bytes_ip = lattdse_dev::P4Geom<AXIS, L, B, 1, false>::bytes;
  // two stage buffers (one barrier per stage) when they do not cost resident
  // CTAs: ROW while both fit 72 KB and shared memory still holds as many
  // CTAs as the registers allow (ROW 2048: in place at 4 CTAs 139 us, two
  // buffers at 3 CTAs 180 us over 4 x 2048 lines); COL above 648 while both
  // fit 90 KB (config 1, COL 1296: 35.0 vs 39.0 us), short COL lines in place
  // (ROW lines of small radices run in place as well: 1080 at 6 CTAs of 80
  // registers 262.7 us, two buffers at 5 CTAs of 94 registers 270.6 us)
  static constexpr bool PP = row ? (max_radix() > 12 && bytes_pp <= 72 * 1024 && fit(bytes_pp) >= regs_ctas(big ? 128 : 96))
                                 : (L > 648 && bytes_pp <= 90 * 1024);
  static constexpr int smem = PP ? bytes_pp : bytes_ip;
  static constexpr int by_regs = regs_ctas(PP ? (big ? 128 : 96) : ip_budget);
  static constexpr int by_smem = fit(smem);
  static constexpr int MB = by_regs < by_smem ? by_regs : by_smem;
  static_assert(smem <= 227 * 1024, "pass4 tile exceeds shared memory");
};

template <int AXIS, int L, int PROG, int SIGN> void reg_one() {
  using G = Geometry<AXIS, L>;
  PassKernel k;
  k.B = G::B;
  k.NT = G::NT;
  k.smem = lattdse_dev::SmemGeom<L, G::B>::bytes;
  k.nst = lattdse_dev::Plan<L>::nst;
  for (int s = 0; s < k.nst && s < 16; ++s) k.radix[s] = lattdse_dev::Plan<L>::radix(s);
  if constexpr (PROG == lattdse_dev::PROG_DOUBLE) {
    // resident CTAs per SM the double program is compiled for (its register
    // cap), measured on C1 / C2 (profiles/README.md): ROW 3 (small L1-resident
    // spills against occupancy for 5-10 warp CTAs); COL (four-step twiddle
    // math in the fused stages) and CTAs above 320 threads 2; ROW lines of
    // 4096 (radix-16 stages) spill heavily under the 3-CTA cap: 2; the wide
    // 4096-long COL tile 1. Only this variant is instantiated (the 1 / 2 / 3
    // sweep of round 1 tripled the library for a debugging knob).
    constexpr int mb = G::wide_col ? 1 : (G::NT > 320 ? 2 : (AXIS == lattdse_dev::AX_ROW && L < 4096 ? 3 : 2));
    k.fn = reinterpret_cast<const void*>(&lattdse_dev::fft_pass_kernel<AXIS, L, G::B, G::NT, PROG, SIGN, mb>);
    k.fn_mb[mb] = k.fn;
    k.default_mb = mb;
  } else {
    k.fn = reinterpret_cast<const void*>(&lattdse_dev::fft_pass_kernel<AXIS, L, G::B, G::NT, PROG, SIGN>);
  }
  if constexpr (LATTDSE_BUILD_PASS4 && PROG == lattdse_dev::PROG_DOUBLE && Geometry4<AXIS, L>::ok) {
    using G4 = Geometry4<AXIS, L>;
    using namespace lattdse_dev;
    if constexpr (AXIS == AX_ROW) {
      k.fn4[0] = reinterpret_cast<const void*>(&fft_pass4_kernel<AXIS, L, G4::B, 1, G4::PP, G4::NT, SIGN, false, DG_CPLX, G4::MB>);
    } else {
      k.fn4[0] = reinterpret_cast<const void*>(&fft_pass4_kernel<AXIS, L, G4::B, 1, G4::PP, G4::NT, SIGN, true, DG_CPLX, G4::MB>);
      k.fn4[1] = reinterpret_cast<const void*>(&fft_pass4_kernel<AXIS, L, G4::B, 1, G4::PP, G4::NT, SIGN, false, DG_LUT16, G4::MB>);
    }
    k.B4 = G4::B;
    k.NT4 = G4::NT;
    k.smem4 = G4::smem;
    if constexpr (Geometry4<AXIS, L, true>::ok) {
      using GW = Geometry4<AXIS, L, true>;
      k.fn4w = reinterpret_cast<const void*>(&fft_pass4_kernel<AXIS, L, GW::B, 1, GW::PP, GW::NT, SIGN, true, DG_CPLX, GW::MB>);
      k.B4w = GW::B;
      k.NT4w = GW::NT;
      k.smem4w = GW::smem;
    }
  }
  // the three-level inner passes (single transform, four-step twiddles on one
  // side): forward + output twiddles, or input twiddles + inverse
  if constexpr (LATTDSE_BUILD_PASS4 && AXIS == lattdse_dev::AX_COL && Geometry4<AXIS, L>::ok &&
                ((PROG == lattdse_dev::PROG_LOADDIAG && SIGN == -1) || (PROG == lattdse_dev::PROG_STOREDIAG && SIGN == +1))) {
    using G4 = Geometry4<AXIS, L>;
    k.fn4[0] = reinterpret_cast<const void*>(
        &lattdse_dev::fft_pass4s_kernel<L, G4::B, G4::PP, G4::NT, SIGN, PROG == lattdse_dev::PROG_STOREDIAG, G4::MB>);
    k.B4 = G4::B;
    k.NT4 = G4::NT;
    k.smem4 = G4::smem;
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
