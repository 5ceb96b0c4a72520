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
};

PassKernel* find_pass_kernel(int axis, int L, int prog, int sign);
void register_pass_kernel(int axis, int L, int prog, int sign, const PassKernel& k);
std::vector<int> pass_lengths(int axis);

}  // namespace lattdse::dev
