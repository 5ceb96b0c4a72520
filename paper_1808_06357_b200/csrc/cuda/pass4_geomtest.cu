// Prints the compile-time launch geometry of the lean pass kernels
// (pass_instantiate.cuh Geometry4, fft_pass4.cuh P4Seq) for the line lengths
// the five configs use; tests/test_abi.py pins the measured choices.
// Host-only: no kernel is instantiated (LATTDSE_BUILD_PASS4=0).
#include <cstdio>

#include "pass_instantiate.cuh"

namespace lattdse::dev {
void register_pass_kernel(int, int, int, int, const PassKernel&) {}
}  // namespace lattdse::dev

template <int L> void show() {
  using namespace lattdse::dev;
  using namespace lattdse_dev;
  using R = Geometry4<AX_ROW, L>;
  using C = Geometry4<AX_COL, L>;
  using W = Geometry4<AX_COL, L, true>;
  std::printf("L=%d plan", L);
  for (int s = 0; s < Plan<L>::nst; ++s) std::printf(" %d", Plan<L>::radix(s));
  std::printf(" ok=%d swz=%d | ROW B=%d pp=%d NT=%d MB=%d smem=%d | COL B=%d pp=%d NT=%d MB=%d smem=%d | WIDE ok=%d B=%d NT=%d MB=%d\n",
              (int)R::ok, (int)P4Seq<L>::swz, R::B, (int)R::PP, R::NT, R::MB, R::smem, C::B, (int)C::PP, C::NT, C::MB,
              C::smem, (int)W::ok, W::B, W::NT, W::MB);
  // skew / swizzle tables stay inside the tile the geometry allocates
  static_assert(P4Geom<AX_ROW, L, R::B, 1, R::PP>::LS >= P4Seq<L>::extent(), "line stride covers the skewed extent");
  static_assert(R::smem <= 227 * 1024 && C::smem <= 227 * 1024, "tiles fit shared memory");
}

int main() {
  show<486>();
  show<1080>();
  show<1296>();
  show<1620>();
  show<2048>();
  show<2160>();
  show<4096>();
  show<512>();
  show<1024>();
  return 0;
}
