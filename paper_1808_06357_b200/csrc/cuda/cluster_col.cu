// Instantiations and launcher of the cluster COL pass (cluster_col.inl):
// config 2's 4096-long columns (rank-2 grid, PROG_DOUBLE).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <vector>

#include "cluster_col.hpp"
#include "cluster_col.inl"

namespace lattdse::dev {
using namespace lattdse_dev;

namespace {
template <int LLOC, int C, int B, int NT, int SIGN, int MINB>
cudaError_t launch_one(PassArgs a, const double2* tables, long long ncols, long long nbatch, cudaStream_t s) {
  auto fn = cluster_col_kernel<LLOC, C, B, NT, SIGN, MINB>;
  const int smem = ClusterGeom<LLOC, C, B>::bytes;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  a.tw_lo = tables;                 // exp(-2 pi i t / L), t < L
  a.fft_tw = tables + LLOC * C;     // Plan<LLOC> stage twiddles
  fn<<<dim3((unsigned)(C * (ncols / B)), (unsigned)nbatch), NT, smem, s>>>(a);
  return cudaGetLastError();
}

// read at solver creation (the solver keeps the chosen Lloc)
int variant() {
  const char* e = std::getenv("LATTDSE_CLUSTER_COL");
  return e ? std::atoi(e) : 0;  // cluster size (8 or 4); off by default (slower, profiles/README.md)
}
int minb() {
  const char* e = std::getenv("LATTDSE_CLUSTER_MINB");
  return e ? std::atoi(e) : 2;
}
}  // namespace

int cluster_col_lloc(int L, long long ncols) {
  const int c = variant();
  if (L != 4096 || (c != 8 && c != 4 && c != 2)) return 0;
  const int B = c;  // B = C columns per cluster (8: 128-byte, 4: 64-byte, 2: 32-byte row segments)
  if (ncols % B != 0) return 0;
  return L / c;
}

std::vector<double2> cluster_col_tables(int L, int lloc) {
  std::vector<double2> t(L);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int k = 0; k < L; ++k) {
    const long double ang = -2.0L * pi * (long double)k / (long double)L;
    t[k] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  int radix[16], nst = 0;
  if (lloc == 512) {
    for (int s = 0; s < Plan<512>::nst; ++s) radix[nst++] = Plan<512>::radix(s);
  } else if (lloc == 1024) {
    for (int s = 0; s < Plan<1024>::nst; ++s) radix[nst++] = Plan<1024>::radix(s);
  } else if (lloc == 2048) {
    for (int s = 0; s < Plan<2048>::nst; ++s) radix[nst++] = Plan<2048>::radix(s);
  }
  const int n = std::max(1, build_stage_twiddles(radix, nst, nullptr));
  std::vector<double2> st(n, make_double2(1.0, 0.0));
  build_stage_twiddles(radix, nst, st.data());
  t.insert(t.end(), st.begin(), st.end());
  return t;
}

cudaError_t launch_cluster_col(int L, int lloc, int sign, const PassArgs& a, const double2* tables, long long ncols,
                               long long nbatch, cudaStream_t s) {
  if (lloc * (L / lloc) != L || ncols % (L / lloc) != 0) return cudaErrorInvalidValue;
  const bool m3 = minb() == 3;
  if (lloc == 512) {
    if (sign < 0)
      return m3 ? launch_one<512, 8, 8, 256, -1, 3>(a, tables, ncols, nbatch, s)
                : launch_one<512, 8, 8, 256, -1, 2>(a, tables, ncols, nbatch, s);
    return m3 ? launch_one<512, 8, 8, 256, +1, 3>(a, tables, ncols, nbatch, s)
              : launch_one<512, 8, 8, 256, +1, 2>(a, tables, ncols, nbatch, s);
  }
  if (lloc == 1024) {
    if (sign < 0)
      return m3 ? launch_one<1024, 4, 4, 256, -1, 3>(a, tables, ncols, nbatch, s)
                : launch_one<1024, 4, 4, 256, -1, 2>(a, tables, ncols, nbatch, s);
    return m3 ? launch_one<1024, 4, 4, 256, +1, 3>(a, tables, ncols, nbatch, s)
              : launch_one<1024, 4, 4, 256, +1, 2>(a, tables, ncols, nbatch, s);
  }
  if (lloc == 2048) {
    if (sign < 0)
      return m3 ? launch_one<2048, 2, 2, 256, -1, 3>(a, tables, ncols, nbatch, s)
                : launch_one<2048, 2, 2, 256, -1, 2>(a, tables, ncols, nbatch, s);
    return m3 ? launch_one<2048, 2, 2, 256, +1, 3>(a, tables, ncols, nbatch, s)
              : launch_one<2048, 2, 2, 256, +1, 2>(a, tables, ncols, nbatch, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lattdse::dev
