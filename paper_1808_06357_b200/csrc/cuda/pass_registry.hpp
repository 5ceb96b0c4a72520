// Registry of compiled pass-kernel instantiations, keyed by
// (axis, line length L, program, sign of the first transform).
// Each csrc/cuda/inst/pass_L*.cu registers one L for both axes and all six
// programs at static-initialisation time.
#pragma once

#include <vector>

namespace lattdse::dev {


struct PassKernel {
  const void* fn = nullptr;  // __global__ fft_pass_kernel<...>
  int B = 0;                 // lines per CTA
  int NT = 0;                // threads per CTA
  int smem = 0;              // dynamic shared memory bytes
  bool attr_set = false;     // cudaFuncAttributeMaxDynamicSharedMemorySize applied
  // pass4: lean per-step variant of the PROG_DOUBLE programs on the plain
  // layouts (fft_pass4.cuh). fn4[0]: complex diagonal (COL: with four-step
  // twiddles; ROW: without); fn4[1]: COL, u16 norm index + LUT, no twiddles
  // (the rank-2 grid's kinetic pass)
  const void* fn4[2] = {};
  int B4 = 0, NT4 = 0, smem4 = 0;
  bool attr4_set = false;
  // short COL lines: the eight-column variant of fn4[0] for views whose rows
  // lie far apart (pass_instantiate.cuh Geometry4 WIDE)
  const void* fn4w = nullptr;
  int B4w = 0, NT4w = 0, smem4w = 0;
  // PROG_DOUBLE instantiated with __launch_bounds__(NT, minBlocks) for
  // minBlocks = 1..4 (register cap vs occupancy); index 0 unused
  const void* fn_mb[5] = {};
  int default_mb = 1;
  int nst = 0;
  int radix[16] = {};        // Plan<L> radices, stage order
};


PassKernel* find_pass_kernel(int axis, int L, int prog, int sign);
void register_pass_kernel(int axis, int L, int prog, int sign, const PassKernel& k);
std::vector<int> pass_lengths(int axis);

// measured pass costs, ps per element per pass (solver.cu): two-level COL /
// ROW passes, three-level first-level COL pass and row side (La x Lb)
double cost_col(int L);
double cost_row(int L);
double cost_col3(int L);
double cost_row3(int La, int Lb);
double cost_pair_ensemble(int L1, int L2);

}  // namespace lattdse::dev
