// Device orchestration of the Strang hot path on one B200.
//
// State between calls: samples u(p_kappa) in kappa order, one N-vector per
// ensemble member. A step(n) call runs entirely on the
// device stream with no host synchronisation until it returns:
//
//   rank-1, method "circulant" (default): F^-1 D F is the circulant matrix of
//     k = F^-1(D)/N, applied as a length-M cyclic convolution (M >= 2N-1,
//     M = M1*M2) through a four-step FFT, so one step is
//        ROW pass  : FFT_M2 . (x K^) . IFFT_M2
//        COL pass  : IFFT_M1 . (mask j<N, x V) . FFT_M1   (with 4-step twiddles)
//     and the two potential half steps of consecutive steps are fused into V.
//   rank-1, method "bluestein": the literal two length-N DFTs per step
//     (Algorithm 1), each a Bluestein convolution: 4 passes.
//   rank-2 grid: ROW pass IFFT.(xV).FFT along n2, COL pass FFT.(xD/N).IFFT
//     along n1.
//
// Ensemble members are stepped in groups sized to stay L2-resident for the
// whole step(n) call (each member's work buffer is reused across steps).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>

#include "fft_pass.cuh"
#include "sampling.cuh"
#include "lattdse/solver.hpp"
#include "aaset_dev.hpp"
#include "pass_registry.hpp"
#ifndef LATTDSE_EXPERIMENTAL
#define LATTDSE_EXPERIMENTAL 0  // measured-slower variants (cluster COL, Good-Thomas, row chunks): make EXPERIMENTAL=1
#endif
#if LATTDSE_EXPERIMENTAL
#include "cluster_col.hpp"
#endif

using namespace lattdse_dev;

namespace lattdse {

#define LD_CK(x)                                                                                      \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) raise(Errc::device_error, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------- registry
namespace dev {
namespace {
struct Registry {
  std::mutex mu;
  std::map<std::tuple<int, int, int, int>, PassKernel> k;
};
Registry& registry() {
  static Registry r;
  return r;
}
}  // namespace

PassKernel* find_pass_kernel(int axis, int L, int prog, int sign) {
  auto& r = registry();
  std::lock_guard<std::mutex> g(r.mu);
  auto it = r.k.find({axis, L, prog, sign});
  return it == r.k.end() ? nullptr : &it->second;
}
void register_pass_kernel(int axis, int L, int prog, int sign, const PassKernel& k) {
  auto& r = registry();
  std::lock_guard<std::mutex> g(r.mu);
  r.k[{axis, L, prog, sign}] = k;
}
std::vector<int> pass_lengths(int axis) {
  auto& r = registry();
  std::lock_guard<std::mutex> g(r.mu);
  std::vector<int> out;
  for (auto& [key, v] : r.k)
    if (std::get<0>(key) == axis && std::get<2>(key) == PROG_DOUBLE && std::get<3>(key) == -1)
      out.push_back(std::get<1>(key));
  return out;
}
}  // namespace dev

// --------------------------------------------------------- aux kernels
namespace {


__global__ void k_phase(const double* __restrict__ v, long long n, double coef, double2* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double s, c;
    sincos(coef * v[i], &s, &c);
    out[i] = make_double2(c, s);
  }
}

// c_j = exp(-pi i j^2 / N), j^2 reduced mod 2N exactly; also conj(c) and c/N.
__global__ void k_chirp(long long N, double2* __restrict__ c, double2* __restrict__ cc, double2* __restrict__ cn) {
  const double invN = 1.0 / (double)N;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    unsigned long long q = (unsigned long long)(((unsigned __int128)j * (unsigned __int128)j) % (unsigned __int128)(2 * N));
    double sgn = 1.0;
    if (q >= (unsigned long long)N) {  // exp(-pi i (q)/N) = -exp(-pi i (q-N)/N)
      q -= (unsigned long long)N;
      sgn = -1.0;
    }
    double s, co;
    sincospi((double)q / (double)N, &s, &co);
    double2 v = make_double2(sgn * co, -sgn * s);
    if (c) c[j] = v;
    if (cc) cc[j] = make_double2(v.x, -v.y);
    if (cn) cn[j] = make_double2(v.x * invN, v.y * invN);
  }
}

// Embed a length-N sequence into a length-M cyclic kernel, scaled:
//  periodic: K[t] = k[t mod N] for t in (-N, N)   (circulant kernel)
//  even:     K[t] = k[|t|]      for t in (-N, N)   (Bluestein chirp)
__global__ void k_wrap(const double2* __restrict__ k, long long N, long long M, double scale, int even,
                       double2* __restrict__ K) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < M; t += (long long)gridDim.x * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (t < N)
      v = k[t];
    else if (t > M - N)
      v = even ? k[M - t] : k[t - (M - N)];
    K[t] = make_double2(v.x * scale, v.y * scale);
  }
}

// Good-Thomas position p = n1*M2 + n2 holds natural n = (M2 n1 + M1 n2) mod M.
__device__ __forceinline__ long long pfa_nat(long long p, long long M1, long long M2, long long M) {
  const long long n1 = p / M2, n2 = p - n1 * M2;
  long long n = M2 * n1 + M1 * n2;
  return n >= M ? n - M : n;
}
__global__ void k_perm_c(const double2* __restrict__ v, long long N, long long M1, long long M2,
                         double2* __restrict__ out) {
  const long long M = M1 * M2;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < M; p += (long long)gridDim.x * blockDim.x) {
    const long long n = pfa_nat(p, M1, M2, M);
    out[p] = n < N ? v[n] : make_double2(0.0, 0.0);
  }
}
__global__ void k_perm_u16(const unsigned short* __restrict__ v, long long N, long long M1, long long M2,
                           unsigned short sentinel, unsigned short* __restrict__ out) {
  const long long M = M1 * M2;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < M; p += (long long)gridDim.x * blockDim.x) {
    const long long n = pfa_nat(p, M1, M2, M);
    out[p] = n < N ? v[n] : sentinel;
  }
}

__global__ void k_lut_gather(const unsigned short* __restrict__ idx, const double2* __restrict__ lut, long long n,
                             double2* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = lut[idx[i]];
}

__global__ void k_mul(const double2* __restrict__ a, const double2* __restrict__ b, long long n, double2* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = c_mul(a[i], b[i]);
}

// ---- rank-1 problem sampling on the device (sampling.cuh)
__global__ void k_sample_v(const R1Points P, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ out) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < P.N; k += (long long)gridDim.x * blockDim.x)
    out[k] = sample_v_point(P, k, a, b);
}
// unnormalised g (problems.cpp eval_g_unnormalized)
__global__ void k_sample_g(const R1Points P, const double* __restrict__ c, const int* __restrict__ p, double inv2s2,
                           double2* __restrict__ out) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < P.N; k += (long long)gridDim.x * blockDim.x)
    out[k] = sample_g_point(P, k, c, p, inv2s2);
}
__global__ void k_scale(double2* __restrict__ x, long long n, double s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = make_double2(x[i].x * s, x[i].y * s);
}

// ---- device CBC (cbc::construct_device): kernels over k in [0, n)
// omega(j) = 2 pi^2 B2(j/n) = num * C, num = 6j(j-n) + n^2 exact (|.| <= n^2 < 2^62),
// C = pi^2 / (3 n^2) as a double-double from the host's long double: the
// product is formed to ~100 bits and rounded once, so omega matches the
// host's cbc::omega (long double product, then double) but for rare
// double-rounding ties.
struct OmC {
  long long n;
  double hi, lo;
};
__device__ __forceinline__ double omega_dev(long long j, const OmC& oc) {
  const long long n = oc.n;
  const long long num = 6 * j * (j - n) + n * n;
  const double nh = (double)num;
  const double nl = (double)(num - (long long)nh);
  const double ph = nh * oc.hi;
  const double pl = fma(nh, oc.hi, -ph) + (nh * oc.lo + nl * oc.hi);
  return ph + pl;
}
__device__ __forceinline__ long long mulmod_dev(long long a, long long b, long long n) {
  return (long long)(((unsigned long long)a * (unsigned long long)b) % (unsigned long long)n);  // a, b < n < 2^31
}
// P[k] *= 1 + omega(k c mod n); c = 0: P[k] = 1
__global__ void k_cbc_apply(double* __restrict__ P, long long n, long long c, const OmC oc) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    P[k] = c ? P[k] * (1.0 + omega_dev(mulmod_dev(k, c, n), oc)) : 1.0;
}
// g^a mod n for a in [0, L), 256 consecutive exponents per thread
__global__ void k_gpow(long long g, long long n, long long L, unsigned* __restrict__ out) {
  const long long chunk = 256;
  for (long long a0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * chunk; a0 < L;
       a0 += (long long)gridDim.x * blockDim.x * chunk) {
    long long x = 1, b = g, e = a0;
    while (e) {
      if (e & 1) x = mulmod_dev(x, b, n);
      b = mulmod_dev(b, b, n);
      e >>= 1;
    }
    const long long a1 = a0 + chunk < L ? a0 + chunk : L;
    for (long long a = a0; a < a1; ++a) {
      out[a] = (unsigned)x;
      x = mulmod_dev(x, g, n);
    }
  }
}
// X[t] = P(g^t) (t < L), W[t] = omega(g^(t mod L)) (t < 2L-1), zero beyond
__global__ void k_cbc_fill(const double* __restrict__ P, const unsigned* __restrict__ gp, long long n, long long L,
                           long long M, const OmC oc, double2* __restrict__ X, double2* __restrict__ W) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < M; t += (long long)gridDim.x * blockDim.x) {
    X[t] = make_double2(t < L ? P[gp[t]] : 0.0, 0.0);
    W[t] = make_double2(t < 2 * L - 1 ? omega_dev(gp[t < L ? t : t - L], oc) : 0.0, 0.0);
  }
}
__global__ void k_conj_mul(double2* __restrict__ X, const double2* __restrict__ W, long long M) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < M; t += (long long)gridDim.x * blockDim.x) {
    const double2 a = X[t], b = W[t];
    X[t] = make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
  }
}
// approx criterion of candidate g^e: (base + corr(e)) / n - 1, corr = Re(X[e]) / M
__device__ __forceinline__ double cbc_approx(const double2* X, long long e, double base, double invM, double n) {
  return (base + X[e].x * invM) / n - 1.0;
}
__global__ void k_cbc_min(const double2* __restrict__ X, long long L, double base, double invM, double n,
                          double* __restrict__ partial) {
  __shared__ double red[32];
  double m = INFINITY;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < L; e += (long long)gridDim.x * blockDim.x)
    m = fmin(m, cbc_approx(X, e, base, invM, n));
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) partial[blockIdx.x] = m;
  }
}
__global__ void k_cbc_count(const double2* __restrict__ X, long long L, double base, double invM, double n,
                            double thresh, unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < L; e += (long long)gridDim.x * blockDim.x)
    c += cbc_approx(X, e, base, invM, n) <= thresh;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}
__global__ void k_cbc_collect(const double2* __restrict__ X, long long L, double base, double invM, double n,
                              double thresh, const unsigned* __restrict__ gp, unsigned* __restrict__ out,
                              unsigned* __restrict__ count, unsigned cap) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < L; e += (long long)gridDim.x * blockDim.x)
    if (cbc_approx(X, e, base, invM, n) <= thresh) {
      const unsigned i = atomicAdd(count, 1u);
      if (i < cap) out[i] = gp[e];
    }
}
// Per-block double-double partial sums of P[k] (1 + omega(k c mod n)) - 1
// (c = 0: P[k] - 1, c < 0: P[k]^2). The criterion is (1/n) sum - 1 ~ 1e-5,
// the sum itself ~ n: subtracting the 1 per term and carrying the rounding
// error of every product and addition keeps ~30 significant digits, more
// than the host's long-double sequential sum (cbc.cpp score_naive).
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  const double s = a.hi + b.hi;
  const double bb = s - a.hi;
  const double e = (a.hi - (s - bb)) + (b.hi - bb);
  const double lo = e + a.lo + b.lo;
  const double hi = s + lo;
  return {hi, lo - (hi - s)};
}
__device__ __forceinline__ DD dd_term(double P, double om) {
  // P (1 + om) - 1 exactly to double-double: 1 + om = s + e, P s = h + l
  const double s = 1.0 + om;
  const double e = om - (s - 1.0);
  const double h = P * s;
  const double l = fma(P, s, -h);
  DD t = dd_add({h, l}, {P * e, 0.0});
  return dd_add(t, {-1.0, 0.0});
}
__global__ void k_cbc_score(const double* __restrict__ P, long long n, long long c, const OmC oc,
                            double* __restrict__ partial) {
  __shared__ DD red[32];
  DD acc{0.0, 0.0};
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const double p = P[k];
    DD t;
    if (c > 0) t = dd_term(p, omega_dev(mulmod_dev(k, c, n), oc));
    else if (c == 0) t = dd_add({p, 0.0}, {-1.0, 0.0});
    else t = {p * p, fma(p, p, -p * p)};
    acc = dd_add(acc, t);
  }
  for (int o = 16; o > 0; o >>= 1) {
    DD x{__shfl_xor_sync(0xffffffffu, acc.hi, o), __shfl_xor_sync(0xffffffffu, acc.lo, o)};
    acc = dd_add(acc, x);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : DD{0.0, 0.0};
    for (int o = 16; o > 0; o >>= 1) {
      DD x{__shfl_xor_sync(0xffffffffu, acc.hi, o), __shfl_xor_sync(0xffffffffu, acc.lo, o)};
      acc = dd_add(acc, x);
    }
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = acc.hi;
      partial[2 * blockIdx.x + 1] = acc.lo;
    }
  }
}

// Per-block partial sums of w_i * |x_i|^2 (w from a real table, an index
// table scaled, or 1), batch along blockIdx.y.
__global__ void k_wsumsq(const double2* __restrict__ x, long long n, long long bstride, const double* __restrict__ w,
                         const unsigned short* __restrict__ widx, double wscale, const double2* __restrict__ y,
                         double* __restrict__ partial) {
  __shared__ double red[32];
  const double2* xb = x + blockIdx.y * bstride;
  const double2* yb = y ? y + blockIdx.y * bstride : nullptr;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double2 v = xb[i];
    if (yb) v = c_sub(v, yb[i]);
    double m = v.x * v.x + v.y * v.y;
    if (w) m *= w[i];
    if (widx) m *= wscale * (double)widx[i];
    acc += m;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = acc;
  }
}

template <class T> struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (p && n == count) return;
    release();
    if (count == 0) return;
    LD_CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
};

const long double kPiL = 3.141592653589793238462643383279502884L;

std::vector<double2> root_table(long long n, long long count, long long stride) {
  std::vector<double2> t(count);
  for (long long i = 0; i < count; ++i) {
    long long q = (i * stride) % n;
    long double a = -2.0L * kPiL * (long double)q / (long double)n;
    t[i] = make_double2((double)cosl(a), (double)sinl(a));
  }
  return t;
}

}  // namespace

// ---- measured pass costs (ps per element per pass) for the geometry choice
namespace dev {
// C1 sweep (M = 2099520) where measured, else the C3 sweep (M = 524880, 8
// members) scaled by 1.15 to C1's occupancy; unmeasured lengths get a
// neutral estimate (profiles/README.md)
double cost_col(int L) {
  switch (L) {
    case 486: return 19.4; case 729: return 21.4; case 1296: return 22.7; case 1215: return 22.7;
    case 972: return 22.5; case 648: return 23.5; case 1458: return 25.4; case 810: return 25.5;
    case 432: return 26.1; case 1944: return 26.4; case 1620: return 26.6; case 1728: return 27.5;
    case 1080: return 27.6; case 540: return 31.4; case 405: return 33.9; case 720: return 37.3;
    case 1440: return 38.8; default: return 30.0;
  }
}
double cost_row(int L) {
  switch (L) {
    case 486: return 14.8; case 729: return 15.3; case 972: return 15.3; case 1620: return 16.7;
    case 1296: return 18.0; case 648: return 18.2; case 1728: return 18.2; case 1215: return 18.8;
    case 2160: return 18.8; case 1080: return 19.6; case 540: return 21.5; case 810: return 22.0;
    case 720: return 22.1; case 1440: return 20.8; case 1458: return 22.7; case 1944: return 23.6;
    case 405: return 24.8; case 432: return 25.0; default: return 22.0;
  }
}
// measured at config-4 size (tools/c4_geom_sweep.sh, profiles/README.md):
// first-level COL pass, and the row side (inner COL forward + ROW + inner
// COL inverse); the inner COL passes run twice per step as single
// transforms (~0.6 of a fused double pass each). Re-measured (r1e) after
// the persisting-L2 carve-out was dropped for tables beyond it: COL lengths
// below 512 run four columns per CTA (64-byte row segments), which the
// HBM-streaming first-level pass rewards (486: 17.4 vs 810: 29.9 ps).
double cost_col3(int L) {
  switch (L) {
    case 486: return 17.4; case 324: return 19.9; case 432: return 20.7; case 243: return 22.9;
    case 648: return 26.7; case 972: return 26.7; case 405: return 27.1; case 1296: return 27.9;
    case 1458: return 28.1; case 1620: return 29.0; case 810: return 29.9; case 540: return 33.1;
    case 720: return 33.7; default: return 1.5 * cost_col(L);
  }
}
// ensembles of >= 64 members stepped in one group (config 3, M = 524880):
// measured ps per element per Strang step of the (COL L1, ROW L2) pair
// (tools/c3_group_sweep.sh, profiles/README.md); -1 = not measured
double cost_pair_ensemble(int L1, int L2) {
  const long long k = (long long)L1 * 10000 + L2;
  switch (k) {
    // r2 (profiles/r2g): 1080 runs the (9, 8, 15) plan, best as a ROW pass
    case 4861080: return 25.1; case 10800486: return 30.5; case 7290720: return 34.2;
    case 9720540: return 34.8;
    default: return -1.0;
  }
}
double cost_row3(int La, int Lb) {
  const long long k = (long long)La * 10000 + Lb;
  switch (k) {
    case 6484096: return 40.6; case 6482048: return 40.6; case 21602048: return 42.0; case 17281728: return 42.1;
    case 21604096: return 42.7; case 20482160: return 43.4; case 12962048: return 45.2; case 16202048: return 45.9;
    case 12964096: return 45.9; case 16204096: return 46.7; case 19442048: return 47.4; case 14582048: return 49.7;
    case 12154096: return 52.0; case 12151215: return 53.6; case 10802048: return 53.8; case 10804096: return 54.5;
    case 40962160: return 60.8; case 8102048: return 63.0; case 8104096: return 63.3;
    default: return 1.5 * (1.2 * cost_col(La) + cost_row(Lb));
  }
}
}  // namespace dev

// fused observables of an exit pass (PassArgs::obs): partial-sum buffer and
// the weight of the second sum (potential table or scaled norm index)
struct ObsSpec {
  double* out = nullptr;
  const double* w = nullptr;
  const unsigned short* widx = nullptr;
  double wscale = 0.0;
  void apply(PassArgs& a) const {
    a.obs = out;
    a.obs_w = w;
    a.obs_widx = widx;
    a.obs_wscale = wscale;
  }
};

// ------------------------------------------------------------- Impl
struct Solver::Impl {
  // problem
  int rank = 1, dim = 1;
  // rank-r grid (r >= 2): tensor n1 x ... x nr, row-major.
  // n1: first modulus (COL pass over the n1 x (N / n1) view), nrow: last
  // modulus (ROW pass over N / nrow contiguous lines); the moduli between
  // them are transformed by single-transform COL passes inside every block of
  // `outer` leading indices (batch = member * outer + block, `inner` columns)
  long long N = 0, n1 = 0, nrow = 0;
  struct InnerAxis {
    long long len, inner, outer;
    DBuf<double2> tw, tw2;
  };
  std::vector<InnerAxis> axes;
  long long batch = 1, group = 1;
  double eps = 1, dt_ = 0;
  double watchdog_tol = 1e-9;  // propagate: max |norm - norm(0)| (0 = off)
  bool have_dt = false;
  std::string method;
  ProblemSpec prob;
  Lattice lat;
  std::uint32_t max_norm2 = 0;

  // transform geometry
  long long M = 0, M1 = 0, M2 = 0;  // work = M1 rows x M2 cols
  // three-level (rank-1, M beyond one COL x ROW split): each length-M2 row is
  // itself an Ma x Mb four-step (COL pass of length Ma inside the row, ROW
  // pass of length Mb); three = false: the ROW pass covers M2 directly
  bool three = false;
  long long Ma = 0, Mb = 0;
  long long row_chunk = 0;  // three-level: M1 rows per L2-resident row-side chunk (0: whole view)
  int tw_shift = 0;
  bool pfa = false;                 // Good-Thomas layout (rank-1), else four-step
  long long forced_M1 = 0, forced_M2 = 0, forced_M2a = 0;

  // device
  int device = 0;
  cudaStream_t stream = nullptr;
  DBuf<double2> work, samples, coef, tmp;
  DBuf<double> v;                 // potential at the points
  DBuf<unsigned short> nidx;      // ||h_chi||^2 per chi
  DBuf<double2> V, Vh, Ventry, Vexit, kin_lut, kin_full, Vperm;
  DBuf<unsigned short> nidx_perm;  // Good-Thomas: norm index in position order (sentinel = zero phase)
  DBuf<double2> Khat, B1hat, B2hat, chirp, chirp_c, chirp_n;
  DBuf<double2> tw_col, tw_row, tw_col2, tw_row2, tw_mid, tw_mid2, tw_lo, tw_hi, scal;
  DBuf<double2> cc_tab;  // rank-2 cluster COL pass tables (cluster_col.hpp), empty when unused
  int cc_lloc = 0;        // its rows per CTA (0: plain COL pass; opt-in LATTDSE_CLUSTER_COL)
  DBuf<double> partial;
  DBuf<char> flush;
  bool bluestein_tables = false;
  long long launches = 0;
  bool sync_check = std::getenv("LATTDSE_SYNC_CHECK") != nullptr;  // debug: sync after every launch
  // lean per-step passes of the plain layouts (fft_pass4.cuh); LATTDSE_PASS4=0
  // keeps every pass on the generic kernels (A/B runs, sanitizer coverage)
  bool use_pass4 = !(std::getenv("LATTDSE_PASS4") && std::atoi(std::getenv("LATTDSE_PASS4")) == 0);
  int pass4_pf = std::getenv("LATTDSE_PASS4_PF") ? std::atoi(std::getenv("LATTDSE_PASS4_PF")) : 0;  // L2 prefetch distance, tiles
  long long launches4 = 0;
  int num_sms = 148;
  // CUDA graphs of kGraphSteps (and 16, 8, 4) identical middle steps, per (group start, size)
  static constexpr int kGraphSteps = 32;
  std::map<std::tuple<long long, long long, long long>, cudaGraphExec_t> graphs;  // (group start, size, steps)
  bool use_graphs = std::getenv("LATTDSE_NO_GRAPHS") == nullptr;
  // programmatic dependent launch between consecutive passes (opt-in LATTDSE_PDL=1:
  // measured neutral on C1/C3, +1% on C2; profiles/README.md)
  bool use_pdl = std::getenv("LATTDSE_PDL") && std::atoi(std::getenv("LATTDSE_PDL")) != 0;
  void drop_graphs() {
    for (auto& [k, g] : graphs) cudaGraphExecDestroy(g);
    graphs.clear();
  }
  long long persist_bytes = 0;   // L2 persisting carve-out granted (0: off)
  // which pass's table is pinned: 1 ROW (K^ / B^), 2 COL (V), 3 both
  int persist_mode = std::getenv("LATTDSE_L2_PERSIST") ? std::atoi(std::getenv("LATTDSE_L2_PERSIST")) : 1;
  size_t persist_window = 0;     // max access-policy window

  explicit Impl(const Lattice& l) : lat(l) {}

  DBuf<double> obs_part, obs_kin;  // exit-pass partials of the samples / of the analysis (kinetic part)
  double* rec_host = nullptr;      // pinned record buffer of propagate (block partials per record)
  size_t rec_host_n = 0;
  std::vector<cudaEvent_t> rec_ev;
  // CTAs per batch member of the exit pass that produces samples (rank 1:
  // COL STOREDIAG over M2 columns; rank 2: ROW STOREDIAG over n1 rows) or
  // coefficients (rank 2 analysis: COL STOREDIAG over n2 columns)
  long long exit_blocks(bool coeffs) const {
    if (rank >= 2) {
      dev::PassKernel* k = coeffs ? dev::find_pass_kernel(AX_COL, (int)n1, PROG_STOREDIAG, -1)
                                  : dev::find_pass_kernel(AX_ROW, (int)nrow, PROG_STOREDIAG, +1);
      const long long lines = coeffs ? N / n1 : N / nrow;
      return k ? (lines + k->B - 1) / k->B : 0;
    }
    dev::PassKernel* k = dev::find_pass_kernel(AX_COL, (int)M1, PROG_STOREDIAG, +1);
    return k ? (M2 + k->B - 1) / k->B : 0;
  }
  // ---- launch helpers
  void launch_pass(int axis, int L, int prog, int sign, PassArgs a, long long nlines, long long nbatch) {
    dev::PassKernel* k = dev::find_pass_kernel(axis, L, prog, sign);
    if (!k) raise(Errc::unsupported, "no pass kernel compiled for axis " + std::to_string(axis) + " L=" + std::to_string(L));
    a.nlines = (int)nlines;
    if (use_pass4 && prog == PROG_DOUBLE && nbatch <= 65535) {
      const int v4 = pass4_variant(axis, L, k, a, nlines);
      if (v4 >= 0) return launch_pass4(axis, L, prog, k, v4, a, nlines, nbatch);
    }
    if (use_pass4 && prog != PROG_DOUBLE && nbatch <= 65535 && pass4_single_ok(axis, L, prog, k, a, nlines))
      return launch_pass4(axis, L, prog, k, 0, a, nlines, nbatch);
    const void* fn = k->fn;
    if (prog == PROG_DOUBLE) {
      const int mb = k->default_mb;
      if (mb >= 1 && mb <= 4 && k->fn_mb[mb]) fn = k->fn_mb[mb];
    }
    int smem = k->smem;
    dim3 grid;
    {
      if (!k->attr_set) {
        for (int m = 0; m <= 4; ++m) {
          const void* f = m == 0 ? k->fn : k->fn_mb[m];
          if (f) LD_CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        }
        k->attr_set = true;
      }
      if (nbatch > 65535) {  // grid.y limit: launch in batch chunks (tables are per position, shared)
        for (long long b0 = 0; b0 < nbatch; b0 += 65535) {
          PassArgs c = a;
          c.in = a.in + b0 * a.in_bstride;
          c.out = a.out + b0 * a.out_bstride;
          if (c.obs) c.obs = a.obs + 2 * b0 * ((nlines + k->B - 1) / k->B);
          launch_pass(axis, L, prog, sign, c, nlines, std::min<long long>(65535, nbatch - b0));
        }
        return;
      }
      grid = dim3((unsigned)((nlines + k->B - 1) / k->B), (unsigned)nbatch);
    }
    void* args[] = {&a};
    const bool persist_this = persist_bytes > 0 && prog == PROG_DOUBLE && a.diag_kind == DG_CPLX &&
                              ((axis == AX_ROW && (persist_mode & 1)) || (axis == AX_COL && (persist_mode & 2)));
    const bool pdl_this = use_pdl;
    if (persist_this || pdl_this) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(k->NT);
      cfg.dynamicSmemBytes = (size_t)smem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[2];
      int na = 0;
      if (persist_this) {
        // keep the per-step diagonal table (K^ / V) L2-resident across steps:
        // it is read once per step and would otherwise be evicted by the
        // streaming work buffer (profiles/README.md, steady-state DRAM bytes)
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = (void*)a.diag;
        attr[na].val.accessPolicyWindow.num_bytes = std::min<size_t>(persist_window, (size_t)table_bytes(a));
        attr[na].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
      }
      if (pdl_this) {
        // the pass waits (griddepcontrol.wait) for its predecessor's results;
        // its CTAs may be scheduled while the predecessor's tail drains
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
      }
      cfg.attrs = attr;
      cfg.numAttrs = na;
      LD_CK(cudaLaunchKernelExC(&cfg, fn, args));
    } else {
      LD_CK(cudaLaunchKernel(fn, grid, dim3(k->NT), args, (size_t)smem, stream));
    }
    ++launches;
    if (sync_check) {
      cudaError_t e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess)
        raise(Errc::device_error, "pass axis=" + std::to_string(axis) + " L=" + std::to_string(L) + " prog=" +
                                      std::to_string(prog) + " sign=" + std::to_string(sign) + " v1" +
                                      ": " + cudaGetErrorString(e));
    }
  }
  // pass4 serves the per-step double programs of the plain layouts: full
  // tiles, no load / store masks, the twiddle and diagonal kinds its two
  // instantiations cover (fft_pass4.cuh); everything else stays on v1.
  // Returns the fn4 index or -1.
  int pass4_variant(int axis, int L, const dev::PassKernel* k, const PassArgs& a, long long nlines) const {
    if (!k->fn4[0] || a.pfa || a.rb_w > 0 || a.ncols_g > 0 || a.tw_mul > 1 || a.obs) return -1;
    if (nlines % k->B4 != 0) return -1;
    const long long span = axis == AX_COL ? (long long)L * a.ncols : nlines * (long long)L;
    if (axis == AX_COL && nlines != a.ncols) return -1;
    if (a.nvalid_in < span || a.nvalid_out < span) return -1;
    if (a.in_bstride != 0 && a.in_bstride < span) return -1;
    if (axis == AX_ROW) return (a.diag_kind == DG_CPLX && !a.pre_tw && !a.post_tw) ? 0 : -1;
    if (a.diag_kind == DG_CPLX && a.pre_tw && a.post_tw) return 0;
    if (a.diag_kind == DG_LUT16 && !a.pre_tw && !a.post_tw && k->fn4[1]) return 1;
    return -1;
  }
  // the lean single-transform kernel (fft_pass4s_kernel): plain COL layout,
  // no diagonal, four-step twiddles on the output (forward) or input
  // (inverse) side only -- the inner passes of the three-level layout
  bool pass4_single_ok(int axis, int L, int prog, const dev::PassKernel* k, const PassArgs& a, long long nlines) const {
    if (axis != AX_COL || !k->fn4[0] || a.diag_kind != DG_NONE || a.pfa || a.rb_w > 0 || a.ncols_g > 0 ||
        a.col_off != 0 || a.obs)
      return false;
    if (nlines % k->B4 != 0 || nlines != a.ncols) return false;
    const long long span = (long long)L * a.ncols;
    if (a.nvalid_in < span || a.nvalid_out < span || a.in_bstride < span || a.out_bstride < span) return false;
    return prog == PROG_LOADDIAG ? (a.post_tw && !a.pre_tw) : (a.pre_tw && !a.post_tw);
  }
  void launch_pass4(int axis, int L, int prog, dev::PassKernel* k, int v4, PassArgs a, long long nlines, long long nbatch) {
    if (!k->attr4_set) {
      for (const void* f : k->fn4)
        if (f) LD_CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem4));
      if (k->fn4w) LD_CK(cudaFuncSetAttribute(k->fn4w, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem4w));
      k->attr4_set = true;
    }
    a.nlines = (int)nlines;
    const long long nmid = std::max<long long>(0, a.nvalid_mid);
    a.mid_rb = (int)std::min<long long>(nmid / a.ncols, 0x7fffffff);
    a.mid_cb = (int)(nmid % a.ncols);
    a.pf = pass4_pf;
    int B4 = k->B4, NT4 = k->NT4, smem4 = k->smem4;
    const void* fn = k->fn4[v4];
    // rows of the view a megabyte or more apart: eight columns per CTA
    if (prog == PROG_DOUBLE && v4 == 0 && axis == AX_COL && k->fn4w && (long long)a.ncols * 16 >= (1LL << 20) &&
        nlines % k->B4w == 0) {
      fn = k->fn4w;
      B4 = k->B4w;
      NT4 = k->NT4w;
      smem4 = k->smem4w;
    }
    const dim3 grid((unsigned)(nlines / B4), (unsigned)nbatch);
    void* args[] = {&a};
    const bool persist_this = persist_bytes > 0 && a.diag_kind == DG_CPLX &&
                              ((axis == AX_ROW && (persist_mode & 1)) || (axis == AX_COL && (persist_mode & 2)));
    if (persist_this) {
      // keep the per-step diagonal table L2-resident (see launch_pass)
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(NT4);
      cfg.dynamicSmemBytes = (size_t)smem4;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
      attr[0].val.accessPolicyWindow.base_ptr = (void*)a.diag;
      attr[0].val.accessPolicyWindow.num_bytes = std::min<size_t>(persist_window, (size_t)table_bytes(a));
      attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
      attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      LD_CK(cudaLaunchKernelExC(&cfg, fn, args));
    } else {
      LD_CK(cudaLaunchKernel(fn, grid, dim3(NT4), args, (size_t)smem4, stream));
    }
    ++launches;
    ++launches4;
    if (sync_check) {
      cudaError_t e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess)
        raise(Errc::device_error, "pass4 axis=" + std::to_string(axis) + " L=" + std::to_string(L) + ": " +
                                      cudaGetErrorString(e));
    }
  }
  // bytes of the complex diagonal table a DOUBLE pass reads (position order)
  long long table_bytes(const PassArgs& a) const {
    return 16LL * (rank == 1 && a.diag == Khat.p ? M : (rank == 1 && a.diag == B1hat.p) || (rank == 1 && a.diag == B2hat.p) ? M
                                                                                                                     : (pfa && a.diag == Vperm.p ? M : N));
  }
  int grid1d(long long n) const { return (int)std::min<long long>((n + 255) / 256, 148 * 16); }
  void aux_done(const char* what = "aux") {
    LD_CK(cudaGetLastError());
    ++launches;
    if (sync_check) {
      cudaError_t e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) raise(Errc::device_error, std::string(what) + ": " + cudaGetErrorString(e));
    }
  }

  PassArgs base_args(int axis) const {
    PassArgs a{};
    a.tw_shift = tw_shift;
    a.tw_lo = tw_lo.p;
    a.tw_hi = tw_hi.p;
    a.fft_tw = axis == AX_COL ? tw_col.p : tw_row.p;
    a.fft_tw2 = axis == AX_COL ? tw_col2.p : tw_row2.p;
    a.ncols = (int)M2;
    a.pfa = pfa ? 1 : 0;
    a.pM1 = (int)M1;
    a.pM2 = (int)M2;
    a.pM = M;
    a.tw_mul = 1;
    return a;
  }
  static void set_diag(PassArgs& a, const double2* d) {
    a.diag_kind = d ? DG_CPLX : DG_NONE;
    a.diag = d;
  }

  // ---- rank-1 four-step passes (COL length M1, ROW length M2)
  // entry: compact[j<N] x diag -> FFT_M1 -> twiddle -> work
  void r1_col_entry(const double2* in, long long in_stride, const double2* diag, double2* w, long long nb) {
    PassArgs a = base_args(AX_COL);
    a.in = in;
    a.out = w;
    a.in_bstride = in_stride;
    a.out_bstride = M;
    a.nvalid_in = N;
    a.nvalid_mid = a.nvalid_out = M;
    a.post_tw = pfa ? 0 : 1;
    set_diag(a, diag);
    launch_pass(AX_COL, (int)M1, PROG_LOADDIAG, -1, a, M2, nb);
  }
  // x V at the mid: four-step -> natural V masked at N; Good-Thomas -> the
  // position-ordered V_perm with the mask folded in (zeros)
  void r1_col_mid(double2* w, const double2* diag, long long nb) {
    PassArgs a = base_args(AX_COL);
    a.in = w;
    a.out = w;
    a.in_bstride = a.out_bstride = M;
    a.nvalid_in = a.nvalid_out = M;
    a.nvalid_mid = pfa ? M : N;
    a.pre_tw = a.post_tw = pfa ? 0 : 1;
    set_diag(a, pfa ? Vperm.p : diag);
    launch_pass(AX_COL, (int)M1, PROG_DOUBLE, +1, a, M2, nb);
  }
  void r1_col_mid_lut(double2* w, long long nb) {  // x D/N through the norm index
    PassArgs a = base_args(AX_COL);
    a.in = w;
    a.out = w;
    a.in_bstride = a.out_bstride = M;
    a.nvalid_in = a.nvalid_out = M;
    a.nvalid_mid = pfa ? M : N;
    a.pre_tw = a.post_tw = pfa ? 0 : 1;
    a.diag_kind = DG_LUT16;
    a.diag_idx = pfa ? nidx_perm.p : nidx.p;
    a.lut = kin_lut.p;
    launch_pass(AX_COL, (int)M1, PROG_DOUBLE, +1, a, M2, nb);
  }
  void r1_col_exit(double2* w, const double2* diag, double2* out, long long out_stride, long long nb,
                   const ObsSpec& ob = ObsSpec{}) {
    PassArgs a = base_args(AX_COL);
    ob.apply(a);
    a.in = w;
    a.out = out;
    a.in_bstride = M;
    a.out_bstride = out_stride;
    a.nvalid_in = a.nvalid_mid = M;
    a.nvalid_out = N;
    a.pre_tw = pfa ? 0 : 1;
    set_diag(a, diag);
    launch_pass(AX_COL, (int)M1, PROG_STOREDIAG, +1, a, M2, nb);
  }
  // ROW pass over the rows of the view: length M2 (two-level) or Mb (three-level)
  void r1_row_pass(int prog, int sign, double2* w, const double2* table, long long nb) {
    PassArgs a = base_args(AX_ROW);
    a.in = w;
    a.out = w;
    a.in_bstride = a.out_bstride = M;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = M;
    set_diag(a, table);
    const long long L = three ? Mb : M2;
    launch_pass(AX_ROW, (int)L, prog, sign, a, M / L, nb);
  }
  // three-level: COL pass of length Ma inside every row (an Ma x Mb matrix;
  // batch index = member * M1 + row), with the row's own four-step twiddles
  // W_M2^(ka*nb) = W_M^(M1*ka*nb)
  PassArgs mid_args(double2* w) const {
    PassArgs a = base_args(AX_COL);
    a.fft_tw = tw_mid.p;
    a.fft_tw2 = tw_mid2.p;
    a.ncols = (int)Mb;
    a.tw_mul = M1;
    a.in = w;
    a.out = w;
    a.in_bstride = a.out_bstride = M2;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = M2;
    return a;
  }
  void r1_mid_fwd(double2* w, long long nb) {  // FFT_Ma, then x W_M2^(ka*nb)
    PassArgs a = mid_args(w);
    a.post_tw = 1;
    launch_pass(AX_COL, (int)Ma, PROG_LOADDIAG, -1, a, Mb, M1 * nb);
  }
  void r1_mid_inv(double2* w, long long nb) {  // x conj W_M2^(ka*nb), then IFFT_Ma
    PassArgs a = mid_args(w);
    a.pre_tw = 1;
    launch_pass(AX_COL, (int)Ma, PROG_STOREDIAG, +1, a, Mb, M1 * nb);
  }
  // per row of the view: FFT_M2 . (x table) . IFFT_M2 (table in the layout
  // r1_row_fwd produces)
  void r1_row_mid(double2* w, const double2* table, long long nb) {
    if (three && row_chunk > 0) return r1_row_mid_chunked(w, table, nb);
    if (three) r1_mid_fwd(w, nb);
    r1_row_pass(PROG_DOUBLE, -1, w, table, nb);
    if (three) r1_mid_inv(w, nb);
  }
  // three-level, opt-in: the row side's three passes on row_chunk rows of
  // the M1 x M2 view at a time, so the chunk (row_chunk * 16 M2 bytes) can
  // stay L2-resident between the inner COL forward, the ROW pass and the
  // inner COL inverse (the state crosses HBM once on this side instead of
  // three times; measured slower at config 4, see the option above)
  void r1_row_mid_chunked(double2* w, const double2* table, long long nb) {
    for (long long m = 0; m < nb; ++m)
      for (long long r0 = 0; r0 < M1; r0 += row_chunk) {
        const long long k = std::min<long long>(row_chunk, M1 - r0);
        double2* wc = w + m * M + r0 * M2;
        PassArgs f = mid_args(wc);
        f.post_tw = 1;
        launch_pass(AX_COL, (int)Ma, PROG_LOADDIAG, -1, f, Mb, k);
        PassArgs a = base_args(AX_ROW);
        a.in = a.out = wc;
        a.in_bstride = a.out_bstride = M;
        a.nvalid_in = a.nvalid_mid = a.nvalid_out = k * M2;
        set_diag(a, table + r0 * M2);
        launch_pass(AX_ROW, (int)Mb, PROG_DOUBLE, -1, a, k * M2 / Mb, 1);
        PassArgs b = mid_args(wc);
        b.pre_tw = 1;
        launch_pass(AX_COL, (int)Ma, PROG_STOREDIAG, +1, b, Mb, k);
      }
  }
  void r1_row_fwd(double2* w) {
    if (three) r1_mid_fwd(w, 1);
    r1_row_pass(PROG_LOADDIAG, -1, w, nullptr, 1);
  }
  // unnormalised IFFT_M from the layout r1_fft_table_full produces back to
  // natural order, in place (four-step layouts only)
  void r1_ifft_full(double2* w) {
    r1_row_pass(PROG_STOREDIAG, +1, w, nullptr, 1);
    if (three) r1_mid_inv(w, 1);
    PassArgs a = base_args(AX_COL);
    a.in = w;
    a.out = w;
    a.in_bstride = a.out_bstride = M;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = M;
    a.pre_tw = 1;
    launch_pass(AX_COL, (int)M1, PROG_STOREDIAG, +1, a, M2, 1);
  }
  // ---- rank-r grid passes (ROW length nrow over N / nrow rows; COL length n1 over N / n1 columns)
  void g_row(int prog, int sign, const double2* in, double2* out, const double2* diag, long long nb,
             const ObsSpec& ob = ObsSpec{}) {
    PassArgs a = base_args(AX_ROW);
    ob.apply(a);
    a.in = in;
    a.out = out;
    a.in_bstride = a.out_bstride = N;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = N;
    set_diag(a, diag);
    launch_pass(AX_ROW, (int)nrow, prog, sign, a, N / nrow, nb);
  }
  void g_col(int prog, int sign, const double2* in, double2* out, int dkind, long long nb,
             const ObsSpec& ob = ObsSpec{}) {
    PassArgs a = base_args(AX_COL);
    ob.apply(a);
    a.in = in;
    a.out = out;
    a.in_bstride = a.out_bstride = N;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = N;
    a.diag_kind = dkind;
    a.diag_idx = nidx.p;
    a.lut = dkind == DG_SCALAR ? scal.p : kin_lut.p;
#if LATTDSE_EXPERIMENTAL
    if (prog == PROG_DOUBLE && cc_lloc > 0 && (dkind == DG_LUT16 || dkind == DG_NONE)) {
      // long columns (config 2): one cluster of CTAs per column block, the
      // column split across the cluster's shared memories (cluster_col.inl)
      a.nlines = (int)(N / n1);
      for (long long b0 = 0; b0 < nb; b0 += 65535) {
        PassArgs c = a;
        c.in = a.in + b0 * a.in_bstride;
        c.out = a.out + b0 * a.out_bstride;
        LD_CK(dev::launch_cluster_col((int)n1, cc_lloc, sign, c, cc_tab.p, N / n1, std::min<long long>(65535, nb - b0), stream));
        ++launches;
        if (sync_check) LD_CK(cudaStreamSynchronize(stream));
      }
      return;
    }
#endif
    launch_pass(AX_COL, (int)n1, prog, sign, a, N / n1, nb);
  }
  // the moduli between the first and the last (rank >= 3): one plain
  // transform of length n_a along axis a of every member, in place
  void g_axis(InnerAxis& ax, int sign, double2* w, long long nb) {
    PassArgs a = base_args(AX_COL);
    a.fft_tw = ax.tw.p;
    a.fft_tw2 = ax.tw2.p;
    a.ncols = (int)ax.inner;
    a.in = w;
    a.out = w;
    a.in_bstride = a.out_bstride = ax.len * ax.inner;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = ax.len * ax.inner;
    a.diag_kind = DG_NONE;
    launch_pass(AX_COL, (int)ax.len, sign < 0 ? PROG_LOADDIAG : PROG_STOREDIAG, sign, a, ax.inner, nb * ax.outer);
  }
  void g_axes(int sign, double2* w, long long nb) {
    for (auto& ax : axes) g_axis(ax, sign, w, nb);
  }

  // ---- rank-1 problem sampling on the device
  R1Points r1_points() const {
    R1Points P{};
    P.N = N;
    P.d = dim;
    const auto steps = lat.numerator_steps();
    for (int j = 0; j < dim; ++j) P.z[j] = steps[0][j];
    return P;
  }
  template <class T> void upload_small(DBuf<T>& b, const std::vector<T>& h) {
    b.alloc(std::max<size_t>(1, h.size()));
    if (!h.empty()) LD_CK(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, stream));
  }
  void sample_v_dev() {
    DBuf<double> da, db;
    upload_small(da, prob.potential.a);
    upload_small(db, prob.potential.b);
    v.alloc(N);
    k_sample_v<<<grid1d(N), 256, 0, stream>>>(r1_points(), da.p, db.p, v.p);
    aux_done("k_sample_v");
    LD_CK(cudaStreamSynchronize(stream));  // da/db are freed at scope exit
  }
  // normalised g of member m into samples (problems.cpp sample_g restated)
  void sample_g_dev(long long m, double2* dst = nullptr) {
    problems::Initial& g = prob.initial[m];
    DBuf<double> dc;
    DBuf<int> dp;
    upload_small(dc, g.c);
    upload_small(dp, g.p);
    double2* out = dst ? dst : samples.p + m * N;
    k_sample_g<<<grid1d(N), 256, 0, stream>>>(r1_points(), dc.p, dp.p, 1.0 / (2.0 * g.sigma * g.sigma), out);
    aux_done("k_sample_g");
    const double tot = reduce(out, N, 1, N, nullptr, nullptr, 0.0, nullptr)[0];
    if (!(tot > 0)) raise(Errc::non_normalizable, "initial condition vanishes on the lattice");
    g.C = 1.0 / std::sqrt(tot / (double)N);
    k_scale<<<grid1d(N), 256, 0, stream>>>(out, N, g.C);
    aux_done("k_scale");
    LD_CK(cudaStreamSynchronize(stream));
  }

  // ---- setup
  void choose_geometry() {
    if (rank >= 2) {
      M1 = n1;
      M2 = N / n1;  // columns of the n1 x (N / n1) view the COL pass runs over
      M = N;
      bool ok = dev::find_pass_kernel(AX_ROW, (int)nrow, PROG_DOUBLE, -1) && dev::find_pass_kernel(AX_COL, (int)n1, PROG_DOUBLE, -1);
      for (auto& ax : axes) ok = ok && dev::find_pass_kernel(AX_COL, (int)ax.len, PROG_LOADDIAG, -1);
      if (!ok) {
        std::string dims;
        for (long long m : lat.moduli()) dims += (dims.empty() ? "" : "x") + std::to_string(m);
        raise(Errc::unsupported, "rank-" + std::to_string(rank) + " grid " + dims + " has no compiled pass kernels");
      }
      return;
    }
    const long long need = 2 * N - 1;
    auto have3 = [&](long long g1, long long ga, long long gb) {
      return g1 > 0 && ga > 0 && gb > 0 && g1 <= 4096 && ga <= 4096 && gb <= 4096 &&
             dev::find_pass_kernel(AX_COL, (int)g1, PROG_DOUBLE, -1) &&
             dev::find_pass_kernel(AX_COL, (int)ga, PROG_LOADDIAG, -1) &&
             dev::find_pass_kernel(AX_ROW, (int)gb, PROG_DOUBLE, -1);
    };
    auto set3 = [&](long long g1, long long ga, long long gb) {
      three = true;
      pfa = false;
      M1 = g1;
      Ma = ga;
      Mb = gb;
      M2 = ga * gb;
      M = M1 * M2;
    };
    if (forced_M1 > 0 && forced_M2 > 0 && forced_M2a > 0) {
      if (forced_M2 % forced_M2a != 0 || forced_M1 * forced_M2 < need || !have3(forced_M1, forced_M2a, forced_M2 / forced_M2a))
        raise(Errc::unsupported, "forced three-level geometry " + std::to_string(forced_M1) + "x" +
                                     std::to_string(forced_M2a) + "x" + std::to_string(forced_M2 / std::max<long long>(1, forced_M2a)) +
                                     " is not compiled or too small for N=" + std::to_string(N));
      set3(forced_M1, forced_M2a, forced_M2 / forced_M2a);
      return;
    }
    if (forced_M1 > 0 && forced_M2 > 0) {
      if (forced_M1 * forced_M2 < need || !dev::find_pass_kernel(AX_COL, (int)forced_M1, PROG_DOUBLE, -1) ||
          !dev::find_pass_kernel(AX_ROW, (int)forced_M2, PROG_DOUBLE, -1))
        raise(Errc::unsupported, "forced geometry " + std::to_string(forced_M1) + "x" + std::to_string(forced_M2) +
                                     " is not compiled or too small for N=" + std::to_string(N));
      M1 = forced_M1;
      M2 = forced_M2;
      M = M1 * M2;
      pfa = false;
      return;
    }
    if (const char* g = std::getenv("LATTDSE_GEOM")) {  // "M1xM2" / "M1xMaxMb" override (experiments)
      long long g1 = 0, ga = 0, gb = 0;
      if (std::sscanf(g, "%lldx%lldx%lld", &g1, &ga, &gb) == 3 && g1 * ga * gb >= need && have3(g1, ga, gb)) {
        set3(g1, ga, gb);
        return;
      }
      long long g2 = 0;
      if (std::sscanf(g, "%lldx%lld", &g1, &g2) == 2 && g1 * g2 >= need && dev::find_pass_kernel(AX_COL, (int)g1, PROG_DOUBLE, -1) &&
          dev::find_pass_kernel(AX_ROW, (int)g2, PROG_DOUBLE, -1)) {
        M1 = g1;
        M2 = g2;
        M = g1 * g2;
        pfa = LATTDSE_EXPERIMENTAL && std::getenv("LATTDSE_PFA") != nullptr && std::gcd(g1, g2) == 1;
        return;
      }
    }
    // Among the splits with the smallest M (within 0.5%), take the one with
    // the lowest measured pass cost (dev::cost_* below)
    auto col_cost = dev::cost_col;
    auto row_cost = dev::cost_row;
    long long mmin = -1;
    for (int L1 : dev::pass_lengths(AX_COL))
      for (int L2 : dev::pass_lengths(AX_ROW)) {
        const long long m = (long long)L1 * L2;
        if (m >= need && (mmin < 0 || m < mmin)) mmin = m;
      }
    if (mmin < 0) {
      // three-level: smallest M = L1 * La * Lb >= 2N-1 (within 0.5%), then the
      // lowest estimated cost; the inner COL passes run twice per step as
      // single transforms (~0.6 of a fused double pass each)
      long long m3 = -1;
      for (int L1 : dev::pass_lengths(AX_COL))
        for (int La : dev::pass_lengths(AX_COL))
          for (int Lb : dev::pass_lengths(AX_ROW)) {
            const long long m = (long long)L1 * La * Lb;
            if (m >= need && (m3 < 0 || m < m3) && have3(L1, La, Lb)) m3 = m;
          }
      if (m3 < 0) raise(Errc::unsupported, "N=" + std::to_string(N) + " exceeds the three-level four-step range");
      auto col3 = dev::cost_col3;
      auto row3 = dev::cost_row3;
      long long c1 = 0, ca = 0, cb = 0;
      double bc = 0;
      for (int L1 : dev::pass_lengths(AX_COL))
        for (int La : dev::pass_lengths(AX_COL))
          for (int Lb : dev::pass_lengths(AX_ROW)) {
            const long long m = (long long)L1 * La * Lb;
            if (m < need || (double)m > 1.005 * (double)m3 || !have3(L1, La, Lb)) continue;
            const double cost = (double)m * (col3(L1) + row3(La, Lb));
            if (c1 == 0 || cost < bc) { c1 = L1; ca = La; cb = Lb; bc = cost; }
          }
      set3(c1, ca, cb);
      return;
    }
    long long best = -1, b1 = 0, b2 = 0, bestp = -1, p1 = 0, p2 = 0;
    double bcost = 0, pcost = 0;
    for (int L1 : dev::pass_lengths(AX_COL))
      for (int L2 : dev::pass_lengths(AX_ROW)) {
        const long long m = (long long)L1 * L2;
        if (m < need || (double)m > 1.005 * (double)mmin) continue;
        // ensembles: measured pair costs where known (config 3's length)
        const double pe = batch >= 64 ? dev::cost_pair_ensemble(L1, L2) : -1.0;
        const double cost = (double)m * (pe > 0 ? pe : col_cost(L1) + row_cost(L2));
        if (best < 0 || cost < bcost) { best = m; b1 = L1; b2 = L2; bcost = cost; }
        if (std::gcd(L1, L2) == 1 && (bestp < 0 || cost < pcost)) { bestp = m; p1 = L1; p2 = L2; pcost = cost; }
      }
    const bool allow_pfa = LATTDSE_EXPERIMENTAL && std::getenv("LATTDSE_PFA") != nullptr;  // opt-in: DESIGN.md
    if (allow_pfa && bestp > 0) {
      pfa = true;
      M = bestp;
      M1 = p1;
      M2 = p2;
    } else {
      pfa = false;
      M = best;
      M1 = b1;
      M2 = b2;
    }
  }

  void upload_twiddles() {
    auto up = [&](DBuf<double2>& b, const std::vector<double2>& h) {
      b.alloc(h.size());
      LD_CK(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice, stream));
    };
    auto stage_tw = [&](int axis, long long L, bool rev) {
      const dev::PassKernel* k = dev::find_pass_kernel(axis, (int)L, PROG_DOUBLE, -1);
      if (!k) raise(Errc::unsupported, "no pass kernel for L=" + std::to_string(L));
      int radix[16];
      for (int s = 0; s < k->nst; ++s) radix[s] = k->radix[rev ? k->nst - 1 - s : s];
      const int n = std::max(1, build_stage_twiddles(radix, k->nst, nullptr));
      std::vector<double2> t(n, make_double2(1.0, 0.0));
      build_stage_twiddles(radix, k->nst, t.data());
      return t;
    };
    up(tw_col, stage_tw(AX_COL, M1, false));
    const long long Lrow = rank >= 2 ? nrow : (three ? Mb : M2);
    up(tw_row, stage_tw(AX_ROW, Lrow, false));
    up(tw_col2, stage_tw(AX_COL, M1, true));
    up(tw_row2, stage_tw(AX_ROW, Lrow, true));
    for (auto& ax : axes) {
      up(ax.tw, stage_tw(AX_COL, ax.len, false));
      up(ax.tw2, stage_tw(AX_COL, ax.len, true));
    }
    if (three) {
      up(tw_mid, stage_tw(AX_COL, Ma, false));
      up(tw_mid2, stage_tw(AX_COL, Ma, true));
    }
    tw_shift = 0;
    while ((1LL << (2 * tw_shift)) < M) ++tw_shift;
    const long long nlo = 1LL << tw_shift, nhi = (M + nlo - 1) / nlo;
    up(tw_lo, root_table(M, nlo, 1));
    up(tw_hi, root_table(M, nhi, nlo));
    std::vector<double2> s = {make_double2(1.0 / (double)N, 0.0)};
    up(scal, s);
#if LATTDSE_EXPERIMENTAL
    if (rank == 2) cc_lloc = dev::cluster_col_lloc((int)n1, N / n1);
    if (cc_lloc > 0) up(cc_tab, dev::cluster_col_tables((int)n1, cc_lloc));
#endif
    LD_CK(cudaStreamSynchronize(stream));
  }

  // Bluestein tables of the length-N DFTs (analyze / synthesize): chirp
  // c_j = exp(-pi i j^2 / N) and B^ = FFT_M(wrapped chirp)/M. Built on
  // first use, each direction separately; `scratch` (M entries) is any
  // buffer free during the build. Lean mode (huge N) frees them after use.
  bool lean = false;
  bool synth_tables = false, analysis_tables = false;
  void build_synth_tables(double2* scratch) {  // synthesize: chirp_c in/out, B2^ = FFT(wrap c)/M
    if (synth_tables || rank != 1) return;
    chirp_c.alloc(N);
    k_chirp<<<grid1d(N), 256, 0, stream>>>(N, scratch, chirp_c.p, nullptr);  // c into scratch[0, N)
    aux_done("k_chirp");
    B2hat.alloc(M);
    // wrap c (scratch[0,N)) into B2hat's storage, then FFT out of place into scratch? the
    // forward table transform needs src != dst: wrap into B2hat, FFT B2hat -> scratch, swap
    k_wrap<<<grid1d(M), 256, 0, stream>>>(scratch, N, M, 1.0 / (double)M, 1, B2hat.p);
    aux_done("k_wrap");
    r1_fft_table_full(B2hat.p, scratch);
    LD_CK(cudaMemcpyAsync(B2hat.p, scratch, sizeof(double2) * M, cudaMemcpyDeviceToDevice, stream));
    LD_CK(cudaStreamSynchronize(stream));
    synth_tables = true;
  }
  void build_analysis_tables(double2* scratch) {  // analyze: chirp in, chirp/N out, B1^ = FFT(wrap conj c)/M
    if (analysis_tables || rank != 1) return;
    chirp.alloc(N);
    chirp_n.alloc(N);
    k_chirp<<<grid1d(N), 256, 0, stream>>>(N, chirp.p, scratch, chirp_n.p);  // conj c into scratch[0, N)
    aux_done("k_chirp");
    B1hat.alloc(M);
    k_wrap<<<grid1d(M), 256, 0, stream>>>(scratch, N, M, 1.0 / (double)M, 1, B1hat.p);
    aux_done("k_wrap");
    r1_fft_table_full(B1hat.p, scratch);
    LD_CK(cudaMemcpyAsync(B1hat.p, scratch, sizeof(double2) * M, cudaMemcpyDeviceToDevice, stream));
    LD_CK(cudaStreamSynchronize(stream));
    analysis_tables = true;
  }
  void drop_synth_tables() {
    chirp_c.release();
    B2hat.release();
    synth_tables = false;
  }
  void drop_analysis_tables() {
    chirp.release();
    chirp_n.release();
    B1hat.release();
    analysis_tables = false;
  }
  // K^ = FFT_M(K) with K in natural order in `src` (M entries), written in the
  // ROW pass's position layout to `w`. src != w: the Good-Thomas gather reads
  // natural positions owned by other CTAs, so it cannot run in place.
  void r1_fft_table_full(const double2* src, double2* w) {
    PassArgs a = base_args(AX_COL);
    a.in = src;
    a.out = w;
    a.in_bstride = a.out_bstride = M;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = M;
    a.post_tw = pfa ? 0 : 1;
    launch_pass(AX_COL, (int)M1, PROG_LOADDIAG, -1, a, M2, 1);
    r1_row_fwd(w);
  }

  // samples (N, one member) -> coefficients (N) and back, on the device
  // kin_obs: the exit pass also writes (sum |c|^2, sum kin ||h||^2 |c|^2)
  // partials of the coefficients into obs_part (fused kinetic energy)
  void analyze_dev(const double2* s, double2* c, double2* w, bool kin_obs = false) {
    ObsSpec o;
    if (kin_obs) {
      obs_kin.alloc((size_t)(2 * exit_blocks(true)));
      o.out = obs_kin.p;
      o.widx = nidx.p;
      o.wscale = 0.5 * eps * 4.0 * M_PI * M_PI;
    }
    if (rank == 1) {
      build_analysis_tables(w);
      r1_col_entry(s, N, chirp.p, w, 1);
      r1_row_mid(w, B1hat.p, 1);
      r1_col_exit(w, chirp_n.p, c, N, 1, o);
    } else {
      g_row(PROG_LOADDIAG, -1, s, w, nullptr, 1);
      g_axes(-1, w, 1);
      g_col(PROG_STOREDIAG, -1, w, c, DG_SCALAR, 1, o);
    }
  }
  void synthesize_dev(const double2* c, double2* s, double2* w) {
    if (rank == 1) {
      build_synth_tables(w);
      r1_col_entry(c, N, chirp_c.p, w, 1);
      r1_row_mid(w, B2hat.p, 1);
      r1_col_exit(w, chirp_c.p, s, N, 1);
    } else {
      g_col(PROG_LOADDIAG, +1, c, w, DG_NONE, 1);
      g_axes(+1, w, 1);
      g_row(PROG_STOREDIAG, +1, w, s, nullptr, 1);
    }
  }

  void build_propagator(double dt) {
    drop_graphs();
    // potential phases: V = exp(-i dt v / eps), Vh = exp(-i dt v / (2 eps));
    // lean mode (circulant) builds them after K^ so the peak stays below HBM
    auto phases = [&] {
      V.alloc(N);
      Vh.alloc(N);
      k_phase<<<grid1d(N), 256, 0, stream>>>(v.p, N, -dt / eps, V.p);
      aux_done("k_phase");
      k_phase<<<grid1d(N), 256, 0, stream>>>(v.p, N, -dt / (2.0 * eps), Vh.p);
      aux_done("k_phase");
    };
    const bool phases_last = lean && rank == 1 && method == "circulant" && !pfa;
    if (phases_last) {
      V.release();
      Vh.release();
    } else {
      phases();
    }
    // kinetic LUT exp(-i eps dt 2 pi^2 s)/N for s = 0..max ||h||^2
    std::vector<double2> lut(max_norm2 + 2, make_double2(0.0, 0.0));  // [max+1] = 0: masked slots
    for (std::uint32_t s = 0; s <= max_norm2; ++s) {
      long double a = -(long double)eps * (long double)dt * 2.0L * kPiL * kPiL * (long double)s;
      long double r = fmodl(a, 2.0L * kPiL);
      lut[s] = make_double2((double)(cosl(r) / (long double)N), (double)(sinl(r) / (long double)N));
    }
    kin_lut.alloc(lut.size());
    LD_CK(cudaMemcpyAsync(kin_lut.p, lut.data(), lut.size() * sizeof(double2), cudaMemcpyHostToDevice, stream));
    LD_CK(cudaStreamSynchronize(stream));  // lut is a host temporary

    if (rank == 1 && pfa) {
      Vperm.alloc(M);
      k_perm_c<<<grid1d(M), 256, 0, stream>>>(V.p, N, M1, M2, Vperm.p);
      aux_done("k_perm_c");
      if (method == "bluestein" && !nidx_perm.p) {
        nidx_perm.alloc(M);
        k_perm_u16<<<grid1d(M), 256, 0, stream>>>(nidx.p, N, M1, M2, (unsigned short)(max_norm2 + 1), nidx_perm.p);
        aux_done("k_perm_u16");
      }
    }
    if (rank == 1 && method == "circulant") {
      // k = F^-1(D)/N: synthesize the D/N phases (Bluestein on the device),
      // wrap periodically into length M, K^ = FFT_M(K)/M. K^'s own storage
      // holds the length-N input (front) and output (back) of the synthesis
      // (only ever one of them live), the work buffer is the scratch: no
      // allocation beyond K^ and the synthesis tables (config 4 fits one GPU).
      Khat.alloc(M);
      double2* kin = Khat.p;
      double2* kt = Khat.p + (M - N);
      k_lut_gather<<<grid1d(N), 256, 0, stream>>>(nidx.p, kin_lut.p, N, kin);
      aux_done("k_lut_gather");
      synthesize_dev(kin, kt, work.p);
      k_wrap<<<grid1d(M), 256, 0, stream>>>(kt, N, M, 1.0 / (double)M, 0, work.p);
      aux_done("k_wrap");
      r1_fft_table_full(work.p, Khat.p);
      LD_CK(cudaStreamSynchronize(stream));
      if (lean) drop_synth_tables();
      Ventry.release();
      Vexit.release();
      if (phases_last) phases();
    } else if (rank == 1) {
      build_analysis_tables(work.p);
      build_synth_tables(work.p);
      Ventry.alloc(N);
      Vexit.alloc(N);
      k_mul<<<grid1d(N), 256, 0, stream>>>(Vh.p, chirp.p, N, Ventry.p);
      aux_done("k_mul");
      k_mul<<<grid1d(N), 256, 0, stream>>>(Vh.p, chirp_c.p, N, Vexit.p);
      aux_done("k_mul");
    }
    LD_CK(cudaStreamSynchronize(stream));
    dt_ = dt;
    have_dt = true;
  }

  // ---- stepping (asynchronous on `stream`); optional per-pass events
  struct PassTimer {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> col, row;
  };
  template <class F> void timed(PassTimer* pt, bool is_col, F&& f) {
    if (!pt) {
      f();
      return;
    }
    cudaEvent_t a, b;
    LD_CK(cudaEventCreate(&a));
    LD_CK(cudaEventCreate(&b));
    LD_CK(cudaEventRecord(a, stream));
    f();
    LD_CK(cudaEventRecord(b, stream));
    (is_col ? pt->col : pt->row).push_back({a, b});
  }

  // observe: the exit pass of every group also writes the fused observable
  // partials (sum |u|^2, sum v |u|^2) of each member into obs_part
  void enqueue_steps(long long nsteps, PassTimer* pt = nullptr, bool observe = false) {
    const long long nblk_obs = observe ? exit_blocks(false) : 0;
    if (observe) obs_part.alloc((size_t)(2 * nblk_obs * batch));
    auto obs_for = [&](long long g0) {
      ObsSpec o;
      if (observe) {
        o.out = obs_part.p + 2 * nblk_obs * g0;
        o.w = v.p;
      }
      return o;
    };
    if (!have_dt) raise(Errc::config_error, "set_dt must be called before stepping");
    if (nsteps <= 0) return;
    for (long long g0 = 0; g0 < batch; g0 += group) {
      const long long gb = std::min(group, batch - g0);
      double2* s = samples.p + g0 * N;
      double2* w = work.p;
      if (rank >= 2) {
        // F = F_1 ... F_r axis by axis; the kinetic diagonal sits between the
        // forward and inverse transforms of the first axis, the potential
        // between those of the last; the axes between them (rank >= 3) are
        // plain transforms on either side of the first-axis pass
        timed(pt, false, [&] { g_row(PROG_LOADDIAG, -1, s, w, Vh.p, gb); });
        for (long long k = 0; k < nsteps; ++k) {
          if (!axes.empty()) timed(pt, true, [&] { g_axes(-1, w, gb); });
          timed(pt, true, [&] { g_col(PROG_DOUBLE, -1, w, w, DG_LUT16, gb); });
          if (!axes.empty()) timed(pt, true, [&] { g_axes(+1, w, gb); });
          if (k + 1 < nsteps)
            timed(pt, false, [&] { g_row(PROG_DOUBLE, +1, w, w, V.p, gb); });
          else
            timed(pt, false, [&] { g_row(PROG_STOREDIAG, +1, w, s, Vh.p, gb, obs_for(g0)); });
        }
      } else if (method == "circulant") {
        timed(pt, true, [&] { r1_col_entry(s, N, Vh.p, w, gb); });
        long long k = 0;
        // middle steps (ROW, COL) in graph chunks: identical launches, so the
        // GPU runs them back to back without host launch latency
        if (!pt && use_graphs && !sync_check && row_chunk == 0) {
          // nsteps - 1 middle steps as graphs of 32, then 16, 8, 4 (a
          // propagation that records every 64 steps would otherwise run
          // half of them as loose launches with host gaps between)
          const int per = three ? 4 : 2;
          for (long long len = kGraphSteps; len >= 4; len >>= 1) {
            while (nsteps - 1 - k >= len) {
              cudaGraphExec_t& ge = graphs[{g0, gb, len}];
              if (!ge) {
                cudaGraph_t g;
                LD_CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
                for (long long i = 0; i < len; ++i) {
                  r1_row_mid(w, Khat.p, gb);
                  r1_col_mid(w, V.p, gb);
                }
                LD_CK(cudaStreamEndCapture(stream, &g));
                LD_CK(cudaGraphInstantiate(&ge, g, 0));
                cudaGraphDestroy(g);
                launches -= per * len;  // counted per replay below
              }
              LD_CK(cudaGraphLaunch(ge, stream));
              launches += per * len;
              k += len;
            }
          }
        }
        for (; k < nsteps; ++k) {
          timed(pt, false, [&] { r1_row_mid(w, Khat.p, gb); });
          if (k + 1 < nsteps)
            timed(pt, true, [&] { r1_col_mid(w, V.p, gb); });
          else
            timed(pt, true, [&] { r1_col_exit(w, Vh.p, s, N, gb, obs_for(g0)); });
        }
      } else {  // literal Bluestein: two length-N DFTs per step
        timed(pt, true, [&] { r1_col_entry(s, N, Ventry.p, w, gb); });
        for (long long k = 0; k < nsteps; ++k) {
          timed(pt, false, [&] { r1_row_mid(w, B1hat.p, gb); });
          timed(pt, true, [&] { r1_col_mid_lut(w, gb); });
          timed(pt, false, [&] { r1_row_mid(w, B2hat.p, gb); });
          if (k + 1 < nsteps)
            timed(pt, true, [&] { r1_col_mid(w, V.p, gb); });
          else
            timed(pt, true, [&] { r1_col_exit(w, Vexit.p, s, N, gb, obs_for(g0)); });
        }
      }
    }
  }

  std::vector<double> reduce(const double2* x, long long n, long long nb, long long bstride, const double* w,
                             const unsigned short* widx, double wscale, const double2* y) {
    const int blocks = (int)std::min<long long>((n + 255) / 256, 592);
    partial.alloc((size_t)blocks * nb);
    k_wsumsq<<<dim3(blocks, (unsigned)nb), 256, 0, stream>>>(x, n, bstride, w, widx, wscale, y, partial.p);
    aux_done("k_wsumsq");
    std::vector<double> h((size_t)blocks * nb);
    LD_CK(cudaMemcpyAsync(h.data(), partial.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
    LD_CK(cudaStreamSynchronize(stream));
    std::vector<double> out(nb);
    for (long long b = 0; b < nb; ++b) {
      long double s = 0;
      for (int i = 0; i < blocks; ++i) s += h[b * blocks + i];
      out[b] = (double)s;
    }
    return out;
  }

  // (||u||, E) of ONE member: norm and potential part from
  // the samples, kinetic part from one analysis of that member only
  std::pair<double, double> observables(long long m) {
    LD_CK(cudaSetDevice(device));
    const double2* sm = samples.p + m * N;
    const double sq = reduce(sm, N, 1, N, nullptr, nullptr, 0, nullptr)[0];
    const double pot = reduce(sm, N, 1, N, v.p, nullptr, 0, nullptr)[0];
    coef.alloc(N);
    analyze_dev(sm, coef.p, work.p);
    const double kin = reduce(coef.p, N, 1, N, nullptr, nidx.p, 0.5 * eps * 4.0 * M_PI * M_PI, nullptr)[0];
    return {std::sqrt(sq / (double)N), kin + pot / (eps * (double)N)};
  }
};

// ------------------------------------------------------------ Solver
Solver::Solver(const Lattice& lat, const AntiAliasSet& aa, const ProblemSpec& prob, const SolverOptions& opt)
    : p_(std::make_unique<Impl>(lat)) {
  Impl& s = *p_;
  s.rank = lat.rank();
  s.dim = lat.dim();
  s.N = lat.n_total();
  if (s.rank >= 2) {
    const auto& n = lat.moduli();
    s.n1 = n.front();
    s.nrow = n.back();
    long long outer = s.n1;
    for (int a = 1; a + 1 < s.rank; ++a) {
      long long inner = 1;
      for (int t = a + 1; t < s.rank; ++t) inner *= n[t];
      s.axes.emplace_back();
      s.axes.back().len = n[a];
      s.axes.back().inner = inner;
      s.axes.back().outer = outer;
      outer *= n[a];
    }
  }
  const bool norms_on_device = aa.norm2.empty();  // build the norm table on this device (rank-1)
  if (norms_on_device && s.rank != 1) raise(Errc::unsupported, "device-built norm tables need a rank-1 lattice");
  if (!norms_on_device && aa.n_total != s.N) raise(Errc::spec_mismatch, "anti-aliasing set does not match the lattice");
  if (aa.max_norm2 > 65534) raise(Errc::unsupported, "||h||^2 above 65535 does not fit the uint16 norm index");
  if (prob.initial.empty()) raise(Errc::invalid_argument, "problem needs at least one initial condition");
  if (!(prob.eps > 0)) raise(Errc::invalid_argument, "eps must be > 0");
  if ((int)prob.potential.a.size() != s.dim || (int)prob.potential.b.size() != std::max(0, s.dim - 1))
    raise(Errc::invalid_argument, "potential coefficients do not match the dimension");
  s.prob = prob;
  s.eps = prob.eps;
  s.batch = (long long)prob.initial.size();
  s.method = s.rank >= 2 ? "grid" : opt.method;
  if (s.rank == 1 && s.method != "circulant" && s.method != "bluestein")
    raise(Errc::invalid_argument, "method must be 'circulant' or 'bluestein'");
  s.max_norm2 = aa.max_norm2;  // device-built tables: set below
  s.device = opt.device;
  s.forced_M1 = opt.force_M1;
  s.forced_M2 = opt.force_M2;
  s.forced_M2a = opt.force_M2a;
  LD_CK(cudaSetDevice(s.device));
  LD_CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  LD_CK(cudaDeviceGetAttribute(&s.num_sms, cudaDevAttrMultiProcessorCount, s.device));
  s.choose_geometry();
  {
    // lean mode: every table resident at once would not fit (config 4:
    // N ~ 2^30, M ~ 2^31): build K^ in its own storage, then V/V^(1/2), and
    // drop the Bluestein tables after use (DESIGN.md memory budget)
    size_t free_b = 0, total_b = 0;
    LD_CK(cudaMemGetInfo(&free_b, &total_b));
    const double full = 16.0 * ((double)s.M * 4 + (double)s.N * 6) + 10.0 * (double)s.N + 16.0 * (double)s.N * (double)s.batch;
    s.lean = full > 0.8 * (double)free_b;
  }
  if (s.persist_mode > 0 && s.rank == 1) {
    int maxp = 0, maxw = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, s.device);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, s.device);
    const long long want = 16LL * ((s.persist_mode & 1) ? s.M : 0) + 16LL * ((s.persist_mode & 2) ? s.M : 0);
    // a table far larger than the carve-out (config 4) would only pin its
    // first window's worth and shrink the L2 the chunked row side streams in
    const long long grant = want > 2LL * maxp ? 0 : std::min<long long>(want, maxp);
    cudaCtxResetPersistingL2Cache();  // drop persisting lines left by earlier work on this device
    if (grant > 0 && maxw > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)grant) == cudaSuccess) {
      s.persist_bytes = grant;
      s.persist_window = (size_t)maxw;
    }
    cudaGetLastError();
    if (std::getenv("LATTDSE_VERBOSE"))
      std::fprintf(stderr, "lattdse: L2 persisting max %d window %d granted %lld\n", maxp, maxw, s.persist_bytes);
  }

  // L2-resident ensemble groups: work buffers of the group + shared tables
  // within ~70% of L2.
  const long long env_group = std::getenv("LATTDSE_GROUP") ? std::atoll(std::getenv("LATTDSE_GROUP")) : 0;  // experiments
  if (opt.group > 0 || env_group > 0) {
    s.group = std::min<long long>(opt.group > 0 ? opt.group : env_group, s.batch);
  } else {
    // every member in one group when the work buffers fit a quarter of the
    // free HBM: wider launches beat L2-resident groups (config 3: 7533 us per
    // step with all 512 members vs 8232 us with the L2-sized group of 9,
    // profiles/README.md) because the passes are not HBM-bound
    size_t free_b = 0, total_b = 0;
    LD_CK(cudaMemGetInfo(&free_b, &total_b));
    long long g = (long long)std::floor(0.25 * (double)free_b / (16.0 * (double)s.M));
    s.group = std::max<long long>(1, std::min<long long>(g, s.batch));
    s.group = std::min<long long>(s.group, 65535);
  }

  if (LATTDSE_EXPERIMENTAL && s.three && s.rank == 1) {
    // opt-in (LATTDSE_ROW_CHUNK = M1 rows per chunk): the three-level row
    // side on L2-sized row chunks. Measured slower on config 4 (row side 105
    // vs 97 ms/step, profiles/README.md): the streaming passes are not
    // HBM-bound, so the saved HBM round trips do not pay for 2430 short
    // launches per step.
    const char* e = std::getenv("LATTDSE_ROW_CHUNK");
    const long long forced = e ? std::atoll(e) : 0;
    if (forced > 0) s.row_chunk = std::min<long long>(forced, s.M1);
  }

  s.upload_twiddles();
  s.work.alloc((size_t)s.M * s.group);
  s.samples.alloc((size_t)s.N * s.batch);
  LD_CK(cudaMemsetAsync(s.samples.p, 0, sizeof(double2) * s.N * s.batch, s.stream));

  // potential values (rank-1: sampled on the device) and the norm index
  std::vector<double> vv;
  if (s.rank == 1 && s.dim <= kMaxDimDev) {
    s.sample_v_dev();
  } else {
    vv = problems::sample_v(lat, prob.potential);
    s.v.alloc(s.N);
    LD_CK(cudaMemcpyAsync(s.v.p, vv.data(), sizeof(double) * s.N, cudaMemcpyHostToDevice, s.stream));
  }
  s.nidx.alloc(s.N);
  std::vector<unsigned short> ni;
  if (norms_on_device) {
    s.max_norm2 = dev::aaset_norms_device(lat, s.nidx.p, s.stream);
  } else {
    ni.resize(s.N);
    for (long long c = 0; c < s.N; ++c) ni[c] = (unsigned short)aa.norm2[c];
    LD_CK(cudaMemcpyAsync(s.nidx.p, ni.data(), sizeof(unsigned short) * s.N, cudaMemcpyHostToDevice, s.stream));
  }
  LD_CK(cudaStreamSynchronize(s.stream));
}

Solver::~Solver() {
  if (p_ && p_->stream) {
    cudaStreamSynchronize(p_->stream);
    p_->drop_graphs();
    for (auto e : p_->rec_ev) cudaEventDestroy(e);
    if (p_->rec_host) cudaFreeHost(p_->rec_host);
    if (p_->persist_bytes > 0) cudaCtxResetPersistingL2Cache();
    cudaStreamDestroy(p_->stream);
  }
}

void Solver::set_dt(double dt) {
  if (!(dt != 0.0) || !std::isfinite(dt)) raise(Errc::invalid_argument, "dt must be finite and nonzero");
  LD_CK(cudaSetDevice(p_->device));
  p_->build_propagator(dt);
}

double Solver::dt() const { return p_->dt_; }

void Solver::set_watchdog(double tol) {
  if (!(tol >= 0)) raise(Errc::invalid_argument, "watchdog tolerance must be >= 0");
  p_->watchdog_tol = tol;
}

void Solver::discretize_initial() {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  for (long long m = 0; m < s.batch; ++m) {
    if (s.rank == 1 && s.dim <= kMaxDimDev) {
      s.sample_g_dev(m);
      continue;
    }
    problems::Initial g = s.prob.initial[m];
    auto gv = problems::sample_g(s.lat, g);
    LD_CK(cudaMemcpy(s.samples.p + m * s.N, gv.data(), sizeof(double2) * s.N, cudaMemcpyHostToDevice));
  }
}

void Solver::set_state(const std::complex<double>* data, std::int64_t count, Space space, std::int64_t m0) {
  Impl& s = *p_;
  if (m0 < 0 || count < 0 || m0 + count > s.batch) raise(Errc::invalid_argument, "set_state: member range out of bounds");
  LD_CK(cudaSetDevice(s.device));
  if (space == Space::samples) {
    LD_CK(cudaMemcpyAsync(s.samples.p + m0 * s.N, data, sizeof(double2) * s.N * count, cudaMemcpyHostToDevice, s.stream));
  } else {
    s.coef.alloc(s.N);
    for (std::int64_t m = 0; m < count; ++m) {
      LD_CK(cudaMemcpyAsync(s.coef.p, data + m * s.N, sizeof(double2) * s.N, cudaMemcpyHostToDevice, s.stream));
      s.synthesize_dev(s.coef.p, s.samples.p + (m0 + m) * s.N, s.work.p);
    }
  }
  LD_CK(cudaStreamSynchronize(s.stream));
}

void Solver::get_state(std::complex<double>* data, std::int64_t count, Space space, std::int64_t m0) {
  Impl& s = *p_;
  if (m0 < 0 || count < 0 || m0 + count > s.batch) raise(Errc::invalid_argument, "get_state: member range out of bounds");
  LD_CK(cudaSetDevice(s.device));
  if (space == Space::samples) {
    LD_CK(cudaMemcpyAsync(data, s.samples.p + m0 * s.N, sizeof(double2) * s.N * count, cudaMemcpyDeviceToHost, s.stream));
  } else {
    s.coef.alloc(s.N);
    for (std::int64_t m = 0; m < count; ++m) {
      s.analyze_dev(s.samples.p + (m0 + m) * s.N, s.coef.p, s.work.p);
      LD_CK(cudaMemcpyAsync(data + m * s.N, s.coef.p, sizeof(double2) * s.N, cudaMemcpyDeviceToHost, s.stream));
    }
  }
  LD_CK(cudaStreamSynchronize(s.stream));
}

void Solver::step(std::int64_t nsteps) {
  LD_CK(cudaSetDevice(p_->device));
  p_->enqueue_steps(nsteps);
  LD_CK(cudaStreamSynchronize(p_->stream));
  LD_CK(cudaGetLastError());
}

std::vector<double> Solver::l2_norm() {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  auto ss = s.reduce(s.samples.p, s.N, s.batch, s.N, nullptr, nullptr, 0, nullptr);
  for (auto& x : ss) x = std::sqrt(x / (double)s.N);
  return ss;
}

std::vector<double> Solver::energy() {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  std::vector<double> out(s.batch);
  s.coef.alloc(s.N);
  const double kin = 0.5 * s.eps * 4.0 * M_PI * M_PI;
  for (long long m = 0; m < s.batch; ++m) {
    const double2* sm = s.samples.p + m * s.N;
    auto pot = s.reduce(sm, s.N, 1, s.N, s.v.p, nullptr, 0, nullptr);
    s.analyze_dev(sm, s.coef.p, s.work.p);
    auto kn = s.reduce(s.coef.p, s.N, 1, s.N, nullptr, s.nidx.p, kin, nullptr);
    out[m] = kn[0] + pot[0] / (s.eps * (double)s.N);
  }
  return out;
}

double Solver::l2_distance_initial(std::int64_t member) {
  Impl& s = *p_;
  if (member < 0 || member >= s.batch) raise(Errc::invalid_argument, "l2_distance_initial: member out of range");
  LD_CK(cudaSetDevice(s.device));
  s.tmp.alloc(s.N);
  if (s.rank == 1 && s.dim <= kMaxDimDev) {
    s.sample_g_dev(member, s.tmp.p);
  } else {
    problems::Initial g = s.prob.initial[member];
    auto gv = problems::sample_g(s.lat, g);
    LD_CK(cudaMemcpy(s.tmp.p, gv.data(), sizeof(double2) * s.N, cudaMemcpyHostToDevice));
  }
  auto d = s.reduce(s.samples.p + member * s.N, s.N, 1, s.N, nullptr, nullptr, 0, s.tmp.p);
  s.tmp.release();
  return std::sqrt(d[0] / (double)s.N);
}

double Solver::l2_distance(const std::complex<double>* ref, Space space, std::int64_t member) {
  Impl& s = *p_;
  if (member < 0 || member >= s.batch) raise(Errc::invalid_argument, "l2_distance: member out of range");
  LD_CK(cudaSetDevice(s.device));
  s.tmp.alloc(s.N);
  LD_CK(cudaMemcpyAsync(s.tmp.p, ref, sizeof(double2) * s.N, cudaMemcpyHostToDevice, s.stream));
  if (space == Space::coefficients) {
    s.coef.alloc(s.N);
    LD_CK(cudaMemcpyAsync(s.coef.p, s.tmp.p, sizeof(double2) * s.N, cudaMemcpyDeviceToDevice, s.stream));
    s.synthesize_dev(s.coef.p, s.tmp.p, s.work.p);
  }
  auto d = s.reduce(s.samples.p + member * s.N, s.N, 1, s.N, nullptr, nullptr, 0, s.tmp.p);
  return std::sqrt(d[0] / (double)s.N);
}

std::vector<TrajectoryRow> Solver::propagate(std::int64_t m, std::int64_t record_every, std::int64_t member) {
  if (m < 0) raise(Errc::invalid_argument, "propagate: m must be >= 0");
  if (member < 0 || member >= p_->batch)
    raise(Errc::invalid_argument, "propagate: member " + std::to_string(member) + " outside [0, " +
                                      std::to_string(p_->batch) + ")");
  if (record_every <= 0) record_every = m > 0 ? m : 1;
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  std::vector<TrajectoryRow> rows;
  {
    const auto ob = s.observables(member);  // initial state (set_state / discretize_initial)
    rows.push_back({0, 0.0, ob.first, ob.second});
  }
  const double norm0 = rows[0].norm;
  const double invN = 1.0 / (double)s.N;
  // Observables fused into the passes: the exit pass
  // that writes the samples also sums |u|^2 and v |u|^2 per member; the
  // kinetic part comes out of the analysis exit pass of this member. Records
  // are asynchronous: the block partials go to pinned host memory behind the
  // passes and the host finishes record r-1 (long double sums, watchdog)
  // while record r's steps are already queued, so the GPU never waits for
  // the host between records.
  const long long nblk_s = s.exit_blocks(false), nblk_k = s.exit_blocks(true);
  const std::int64_t nrec = m > 0 ? (m + record_every - 1) / record_every : 0;
  const size_t per = (size_t)(2 * (nblk_s + nblk_k));
  // pinned record buffer and events live with the solver (pinned allocation
  // costs milliseconds: it would dominate a short propagation)
  if (s.rec_host_n < per * (size_t)nrec) {
    if (s.rec_host) cudaFreeHost(s.rec_host);
    s.rec_host = nullptr;
    s.rec_host_n = 0;
    LD_CK(cudaMallocHost(&s.rec_host, per * (size_t)nrec * sizeof(double)));
    s.rec_host_n = per * (size_t)nrec;
  }
  double* host = s.rec_host;
  while (s.rec_ev.size() < (size_t)nrec) {
    cudaEvent_t e;
    LD_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s.rec_ev.push_back(e);
  }
  std::vector<cudaEvent_t>& ev = s.rec_ev;
  s.coef.alloc(s.N);
  std::vector<std::int64_t> at((size_t)nrec);
  auto finish = [&](std::int64_t r) {
    LD_CK(cudaEventSynchronize(ev[(size_t)r]));
    const double* h = host + per * (size_t)r;
    long double sq = 0, pot = 0, kin = 0;
    for (long long i = 0; i < nblk_s; ++i) {
      sq += h[2 * i];
      pot += h[2 * i + 1];
    }
    for (long long i = 0; i < nblk_k; ++i) kin += h[2 * nblk_s + 2 * i + 1];
    const std::int64_t k = at[(size_t)r];
    rows.push_back({k, (double)k * s.dt_, std::sqrt((double)sq * invN), (double)kin + (double)pot * invN / s.eps});
    // norm-drift watchdog (numerical_invariant, CLI exit code 3)
    const double drift = std::fabs(rows.back().norm - norm0);
    if (p_->watchdog_tol > 0 && !(drift <= p_->watchdog_tol)) {
      cudaStreamSynchronize(s.stream);  // queued steps finish before the buffers go away
      raise(Errc::numerical_invariant, "norm drift " + std::to_string(drift) + " at step " + std::to_string(k) +
                                           " exceeds " + std::to_string(p_->watchdog_tol));
    }
  };
  std::int64_t r = 0;
  for (std::int64_t k = 0; k < m; ++r) {
    const std::int64_t n = std::min(record_every, m - k);
    s.enqueue_steps(n, nullptr, true);
    double* h = host + per * (size_t)r;
    LD_CK(cudaMemcpyAsync(h, s.obs_part.p + 2 * nblk_s * member, (size_t)(2 * nblk_s) * sizeof(double),
                          cudaMemcpyDeviceToHost, s.stream));
    s.analyze_dev(s.samples.p + member * s.N, s.coef.p, s.work.p, true);
    LD_CK(cudaMemcpyAsync(h + 2 * nblk_s, s.obs_kin.p, (size_t)(2 * nblk_k) * sizeof(double), cudaMemcpyDeviceToHost,
                          s.stream));
    LD_CK(cudaEventRecord(ev[(size_t)r], s.stream));
    LD_CK(cudaGetLastError());
    k += n;
    at[(size_t)r] = k;
    if (r > 0) finish(r - 1);
  }
  if (nrec > 0) finish(nrec - 1);
  return rows;
}

double Solver::time_steps(std::int64_t nsteps) {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  cudaEvent_t a, b;
  LD_CK(cudaEventCreate(&a));
  LD_CK(cudaEventCreate(&b));
  LD_CK(cudaEventRecord(a, s.stream));
  s.enqueue_steps(nsteps);
  LD_CK(cudaEventRecord(b, s.stream));
  LD_CK(cudaEventSynchronize(b));
  float ms = 0;
  LD_CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  LD_CK(cudaGetLastError());
  return ms;
}

void Solver::profile_passes(std::int64_t nsteps, double* ms_col, double* ms_row) {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  Impl::PassTimer pt;
  s.enqueue_steps(nsteps, &pt);
  LD_CK(cudaStreamSynchronize(s.stream));
  auto avg = [](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
    double tot = 0;
    for (auto& [a, b] : v) {
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      tot += ms;
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    return v.empty() ? 0.0 : tot / (double)v.size();
  };
  *ms_col = avg(pt.col);
  *ms_row = avg(pt.row);
}

void Solver::flush_l2() {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  const size_t bytes = 512ull << 20;
  if (!s.flush.p) s.flush.alloc(bytes);
  LD_CK(cudaMemsetAsync(s.flush.p, (int)(s.launches & 0xff), bytes, s.stream));
  LD_CK(cudaStreamSynchronize(s.stream));
}

void Solver::synchronize() {
  LD_CK(cudaSetDevice(p_->device));
  LD_CK(cudaStreamSynchronize(p_->stream));
}

SolverInfo Solver::info() const {
  const Impl& s = *p_;
  SolverInfo i{};
  i.n_total = s.N;
  i.batch = s.batch;
  i.M = s.M;
  i.M1 = s.M1;
  i.M2 = s.M2;
  i.M2a = s.three ? s.Ma : 0;
  i.row_chunk = s.three ? s.row_chunk : 0;
  i.rank = s.rank;
  i.method = s.method + (s.rank == 1 ? (s.pfa ? "/good-thomas" : "/four-step") : "");
  i.group = s.group;
  i.pass4 = s.launches4 > 0 ? 1 : 0;  // the lean per-step kernels have run (plain layouts)
  // algorithmic bytes: every member's state read + written once per pass;
  // the diagonal tables are shared by the members of a group, so a launch
  // (one group) reads each table once
  const double M = (double)s.M, N = (double)s.N, B = (double)s.batch;
  const double G = (double)s.group, groups = std::ceil(B / G);
  if (s.rank >= 2) {
    const double na = (double)s.axes.size();  // rank >= 3: a plain pass per inner axis on each side
    i.bytes_per_pass_row = B * 32.0 * N + groups * 16.0 * N;                    // state R+W + V
    i.bytes_per_pass_col = (1.0 + 2.0 * na) * B * 32.0 * N + groups * 2.0 * N;  // state R+W (+ inner axes) + D index
    i.bytes_per_step = i.bytes_per_pass_row + i.bytes_per_pass_col;
    i.launches_per_step = 2 + 2 * (int)s.axes.size();
  } else if (s.method == "circulant") {
    // state R+W + V: four-step reads the N valid V entries, Good-Thomas the
    // position-ordered V_perm (M entries, mask folded in)
    i.bytes_per_pass_col = B * 32.0 * M + groups * 16.0 * (s.pfa ? M : N);
    // state R+W + K^ once per group; three-level: the "row" side is three
    // passes (inner COL forward, ROW with K^, inner COL inverse), which cross
    // HBM once in total when they run on L2-resident row chunks
    const bool chunked = s.three && s.row_chunk > 0;
    i.bytes_per_pass_row = ((s.three && !chunked) ? 3.0 : 1.0) * B * 32.0 * M + groups * 16.0 * M;
    i.bytes_per_step = i.bytes_per_pass_col + i.bytes_per_pass_row;
    const long long nchunks = chunked ? (s.M1 + s.row_chunk - 1) / s.row_chunk : 1;
    i.launches_per_step = (int)((chunked ? 1 + 3 * nchunks * s.group : (s.three ? 4 : 2)) * (long long)groups);
  } else {
    i.bytes_per_pass_col = B * 32.0 * M + groups * 9.0 * N;  // avg of (V 16N) and (D idx 2N)
    i.bytes_per_pass_row = B * 32.0 * M + groups * 16.0 * M;
    i.bytes_per_step = 2.0 * (i.bytes_per_pass_col + i.bytes_per_pass_row);
    i.launches_per_step = 4 * (int)groups;
  }
  return i;
}

std::int64_t Solver::kernel_launches() const { return p_->launches; }

const void* Solver::device_table(int which) const {
  switch (which) {
    case 0: return p_->Khat.p;
    case 1: return p_->V.p;
    case 2: return p_->Vh.p;
    default: return nullptr;
  }
}

int Solver::device() const { return p_->device; }

// ------------------------------------------------------- device CBC
namespace cbc {

namespace {
bool prime_n(i64 n) {
  if (n < 2) return false;
  for (i64 p : {2, 3, 5, 7, 11, 13})
    if (n % p == 0) return n == p;
  for (i64 f = 17; f * f <= n; f += 2)
    if (n % f == 0) return false;
  return true;
}
i64 powmod_h(i64 b, i64 e, i64 m) {
  __int128 r = 1, x = b % m;
  while (e) {
    if (e & 1) r = r * x % m;
    x = x * x % m;
    e >>= 1;
  }
  return (i64)r;
}
i64 primitive_root_h(i64 p) {
  std::vector<i64> fac;
  i64 m = p - 1;
  for (i64 f = 2; f * f <= m; ++f)
    if (m % f == 0) {
      fac.push_back(f);
      while (m % f == 0) m /= f;
    }
  if (m > 1) fac.push_back(m);
  for (i64 g = 2; g < p; ++g) {
    bool ok = true;
    for (i64 f : fac)
      if (powmod_h(g, (p - 1) / f, p) == 1) {
        ok = false;
        break;
      }
    if (ok) return g;
  }
  return 1;
}
}  // namespace

Result construct_device(i64 n, int d_max, int device) {
  if (d_max < 1) raise(Errc::invalid_argument, "cbc: d_max must be >= 1");
  if (!prime_n(n) || n <= 64) raise(Errc::unsupported, "device CBC: prime n > 64 only (use cbc::construct)");
  if (n >= (1LL << 31)) raise(Errc::unsupported, "device CBC: n must be < 2^31");
  // the solver's transform machinery as a length-M FFT engine, M >= 2n-1 >= 2L-1
  Lattice lat1 = Lattice::rank1({1}, n);
  Solver::Impl E(lat1);
  E.rank = 1;
  E.dim = 1;
  E.N = n;
  E.method = "circulant";
  E.device = device;
  LD_CK(cudaSetDevice(device));
  LD_CK(cudaStreamCreateWithFlags(&E.stream, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{E.stream};
  LD_CK(cudaDeviceGetAttribute(&E.num_sms, cudaDevAttrMultiProcessorCount, device));
  E.choose_geometry();
  E.pfa = false;
  E.upload_twiddles();
  const long long L = n - 1, M = E.M;
  OmC oc;
  {
    const long double C = 9.869604401089358618834490999876151135L / (3.0L * (long double)n * (long double)n);
    oc.n = n;
    oc.hi = (double)C;
    oc.lo = (double)(C - (long double)oc.hi);
  }
  DBuf<double> P, part;
  DBuf<unsigned> gp, cand, cnt;
  DBuf<double2> X, W;
  P.alloc(n);
  Result res;
  const int blocks = 148 * 8;
  part.alloc(2 * blocks);
  // sum_k P[k] (1 + omega(k c mod n)) - n (c > 0); sum_k P[k] - n (c = 0); sum_k P[k]^2 (c < 0)
  auto raw_sum = [&](long long c) {
    k_cbc_score<<<blocks, 256, 0, E.stream>>>(P.p, n, c, oc, part.p);
    E.aux_done("k_cbc_score");
    std::vector<double> h(2 * blocks);
    LD_CK(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * 2 * blocks, cudaMemcpyDeviceToHost, E.stream));
    LD_CK(cudaStreamSynchronize(E.stream));
    long double t = 0;
    for (int b = 0; b < blocks; ++b) t += (long double)h[2 * b] + (long double)h[2 * b + 1];
    return t;
  };
  // criterion (1/n) sum_k P[k](1 + omega(k c)) - 1 = (sum_k [P(1+omega) - 1]) / n
  auto score = [&](long long c) { return (double)(raw_sum(c) / (long double)n); };
  const bool verbose = std::getenv("LATTDSE_CBC_VERBOSE") != nullptr;
  // z_1 = 1: criterion with P = 1, then P = 1 + omega(k)
  k_cbc_apply<<<E.grid1d(n), 256, 0, E.stream>>>(P.p, n, 0, oc);
  E.aux_done("k_cbc_apply");
  res.z.push_back(1);
  res.wce.push_back(score(1));
  k_cbc_apply<<<E.grid1d(n), 256, 0, E.stream>>>(P.p, n, 1, oc);
  E.aux_done("k_cbc_apply");
  if (d_max > 1) {
    const i64 g = primitive_root_h(n);
    gp.alloc(L);
    k_gpow<<<E.grid1d((L + 255) / 256), 256, 0, E.stream>>>(g, n, L, gp.p);
    E.aux_done("k_gpow");
    X.alloc(M);
    W.alloc(M);
    const unsigned cap = 2048;
    cand.alloc(cap);
    cnt.alloc(1);
    DBuf<unsigned long long> cnt64;
    cnt64.alloc(1);
    for (int s = 2; s <= d_max; ++s) {
      k_cbc_fill<<<E.grid1d(M), 256, 0, E.stream>>>(P.p, gp.p, n, L, M, oc, X.p, W.p);
      E.aux_done("k_cbc_fill");
      E.r1_fft_table_full(X.p, X.p);  // in place: four-step layout
      E.r1_fft_table_full(W.p, W.p);
      k_conj_mul<<<E.grid1d(M), 256, 0, E.stream>>>(X.p, W.p, M);
      E.aux_done("k_conj_mul");
      E.r1_ifft_full(X.p);  // X[e] = M * corr(e), e < L
      // base = sum_k P[k] + P[0] omega(0)
      double p0 = 0;
      LD_CK(cudaMemcpyAsync(&p0, P.p, sizeof(double), cudaMemcpyDeviceToHost, E.stream));
      const long double sumP = raw_sum(0) + (long double)n;
      const double om0 = cbc::omega(0, n);
      const double base = (double)(sumP + (long double)p0 * om0);
      // FFT correlation error bound ~ eps log2(M) ||p|| ||w|| (||w||^2 = sum omega^2
      // = n (2 pi^2)^2 / 180 for B2): widen the shortlist window past it
      const double pnorm = std::sqrt((double)raw_sum(-1));
      const double wnorm = std::sqrt((double)n * 4.0 * 97.40909103400244 / 180.0);
      const double fft_err = 4.0 * 1.1e-16 * std::log2((double)M) * pnorm * wnorm / (double)n;
      k_cbc_min<<<blocks, 256, 0, E.stream>>>(X.p, L, base, 1.0 / (double)M, (double)n, part.p);
      E.aux_done("k_cbc_min");
      std::vector<double> h(blocks);
      LD_CK(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * blocks, cudaMemcpyDeviceToHost, E.stream));
      LD_CK(cudaStreamSynchronize(E.stream));
      double best = INFINITY;
      for (double x : h) best = std::min(best, x);
      const double window = std::max(std::max(1e-9 * std::fabs(best), 1e-13), fft_err);
      double thresh = best + window;
      // Shortlists beyond `cap` (n ~ 2^30: the FFT correlation's rounding
      // floor exceeds the spread of the leading criteria) keep the `cap`
      // smallest approximations: bisect the threshold on the count.
      auto count_le = [&](double t) {
        LD_CK(cudaMemsetAsync(cnt64.p, 0, sizeof(unsigned long long), E.stream));
        k_cbc_count<<<blocks, 256, 0, E.stream>>>(X.p, L, base, 1.0 / (double)M, (double)n, t, cnt64.p);
        E.aux_done("k_cbc_count");
        unsigned long long c = 0;
        LD_CK(cudaMemcpyAsync(&c, cnt64.p, sizeof(c), cudaMemcpyDeviceToHost, E.stream));
        LD_CK(cudaStreamSynchronize(E.stream));
        return c;
      };
      bool truncated = false;
      if (count_le(thresh) > cap) {
        truncated = true;
        double lo = best, hi = thresh;
        for (int it = 0; it < 200 && lo < hi; ++it) {
          const double mid = lo + 0.5 * (hi - lo);
          if (mid <= lo || mid >= hi) break;
          if (count_le(mid) > cap) hi = mid;
          else lo = mid;
        }
        thresh = lo;
      }
      LD_CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned), E.stream));
      k_cbc_collect<<<blocks, 256, 0, E.stream>>>(X.p, L, base, 1.0 / (double)M, (double)n, thresh, gp.p, cand.p,
                                                  cnt.p, cap);
      E.aux_done("k_cbc_collect");
      unsigned nc = 0;
      LD_CK(cudaMemcpyAsync(&nc, cnt.p, sizeof(unsigned), cudaMemcpyDeviceToHost, E.stream));
      LD_CK(cudaStreamSynchronize(E.stream));
      if (nc == 0) raise(Errc::device_error, "device CBC: empty shortlist");
      if (nc > cap) raise(Errc::unsupported, "device CBC: shortlist above " + std::to_string(cap) + " candidates");
      std::vector<unsigned> cs(nc);
      LD_CK(cudaMemcpyAsync(cs.data(), cand.p, sizeof(unsigned) * nc, cudaMemcpyDeviceToHost, E.stream));
      LD_CK(cudaStreamSynchronize(E.stream));
      std::sort(cs.begin(), cs.end());
      std::vector<std::pair<double, i64>> scored;
      for (unsigned c : cs) scored.push_back({score((long long)c), (i64)c});
      // smallest value; values within kTieRel of it tie -> smallest candidate (cbc.cpp pick)
      double bv = scored.front().first;
      for (auto& sc : scored) bv = std::min(bv, sc.first);
      const double tol = kTieRel * std::fabs(bv);
      i64 zs = -1;
      double val = 0;
      for (auto& sc : scored)
        if (sc.first <= bv + tol && (zs < 0 || sc.second < zs)) {
          zs = sc.second;
          val = sc.first;
        }
      if (verbose)
        std::fprintf(stderr, "cbc_dev s=%d best~%.17g window=%.3g (fft_err %.3g) shortlist=%u%s z=%lld wce=%.17g\n", s,
                     best, window, fft_err, nc, truncated ? " (truncated)" : "", (long long)zs, val);
      res.z.push_back(zs);
      res.wce.push_back(val);
      k_cbc_apply<<<E.grid1d(n), 256, 0, E.stream>>>(P.p, n, zs, oc);
      E.aux_done("k_cbc_apply");
    }
  }
  LD_CK(cudaStreamSynchronize(E.stream));
  return res;
}

}  // namespace cbc

}  // namespace lattdse
