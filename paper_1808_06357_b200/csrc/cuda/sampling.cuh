// Rank-1 problem sampling on the device (problems.cpp restated): the
// numerators (kappa z_j) mod N are exact 64-bit integers; trigonometric
// arguments are formed from them reduced mod N. Shared by the
// single-device solver (solver.cu) and the sharded one (solver_dist.cu), so
// both sample bit-identical values.
#pragma once

#include <cuda_runtime.h>

namespace lattdse_dev {

constexpr int kMaxDimDev = 64;  // device-sampled rank-1 problems: d <= 64

struct R1Points {
  long long N;
  int d;
  long long z[kMaxDimDev];
};
__device__ __forceinline__ long long r1_num(const R1Points& P, long long k, int j) {
  return (long long)(((unsigned long long)k * (unsigned long long)P.z[j]) % (unsigned long long)P.N);
}
__device__ __forceinline__ double cos2pi_frac_dev(long long a, long long L) {
  long long r = a % L;
  if (r < 0) r += L;
  return cospi(2.0 * (double)r / (double)L);
}
// v(x) = sum_j a_j (1 - cos 2 pi x_j) + sum_{j<d} b_j cos 2 pi (x_j - x_{j+1})  (problems.cpp eval_v)
__device__ __forceinline__ double sample_v_point(const R1Points& P, long long k, const double* __restrict__ a,
                                                 const double* __restrict__ b) {
  double acc = 0.0;
  for (int j = 0; j < P.d; ++j) acc += a[j] * (1.0 - cos2pi_frac_dev(r1_num(P, k, j), P.N));
  for (int j = 0; j + 1 < P.d; ++j) acc += b[j] * cos2pi_frac_dev(r1_num(P, k, j) - r1_num(P, k, j + 1), P.N);
  return acc;
}
// unnormalised g at point kappa = k (problems.cpp eval_g_unnormalized)
__device__ __forceinline__ double2 sample_g_point(const R1Points& P, long long k, const double* __restrict__ c,
                                                  const int* __restrict__ p, double inv2s2) {
  double expo = 0.0;
  long long phase = 0;
  for (int j = 0; j < P.d; ++j) {
    const long long nj = r1_num(P, k, j);
    const double s = sinpi((double)nj / (double)P.N - c[j]);
    expo -= s * s * inv2s2;
    phase += (long long)p[j] * nj;
  }
  long long ph = phase % P.N;
  if (ph < 0) ph += P.N;
  double sn, cs;
  sincospi(2.0 * (double)ph / (double)P.N, &sn, &cs);
  const double amp = exp(expo);
  return make_double2(amp * cs, amp * sn);
}

}  // namespace lattdse_dev
