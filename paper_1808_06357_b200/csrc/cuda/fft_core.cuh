// In-register small DFTs and the shared-memory Stockham stage used by the
// fused Strang pass kernels (fft_pass.cuh).
//
// Everything here is __host__ __device__ so the exact same index algebra is
// exercised by the CPU emulation test (tests/test_fft_core_emulation.py runs
// the nvcc-built host harness csrc/cuda/fft_core_hosttest.cu).
//
// Conventions: complex fp64 is double2 (x = re, y = im). A transform of sign
// SIGN computes X[k] = sum_n x[n] exp(SIGN * 2*pi*i*n*k/R); SIGN=-1 is the
// forward DFT of SPEC.md:243-251 (analyze), SIGN=+1 the unnormalised inverse
// (synthesize).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <utility>

#include "dft_consts.h"

#if defined(__CUDACC__)
#define LD_HD __host__ __device__ __forceinline__
#else
#define LD_HD inline
#endif

namespace lattdse_dev {

// ---------------------------------------------------------------- complex ops
LD_HD double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
LD_HD double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
LD_HD double2 c_mul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
LD_HD double2 c_mulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
LD_HD double2 c_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// a * (i*S), S = +-1
template <int S> LD_HD double2 c_muli(double2 a) {
  return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// ------------------------------------------------------- compile-time loops
template <class F, int... Is>
LD_HD void sfor_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F> LD_HD void sfor(F&& f) {
  sfor_impl(f, std::make_integer_sequence<int, N>{});
}

// multiply by the compile-time root exp(SIGN*2*pi*i*M/R)
template <int R, int M, int SIGN> LD_HD double2 tw_const(double2 a) {
  constexpr int m = ((M % R) + R) % R;
  if constexpr (m == 0) {
    return a;
  } else if constexpr (2 * m == R) {
    return make_double2(-a.x, -a.y);
  } else if constexpr (4 * m == R) {
    return c_muli<SIGN>(a);
  } else if constexpr (4 * m == 3 * R) {
    return c_muli<-SIGN>(a);
  } else {
    constexpr double c = TwC<R, m>::c;
    constexpr double s = SIGN * TwC<R, m>::s;
    return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
  }
}

// ----------------------------------------------------------- small DFTs
template <int R, int SIGN> struct DFT;

template <int SIGN> struct DFT<1, SIGN> {
  LD_HD static void run(double2*) {}
};

template <int SIGN> struct DFT<2, SIGN> {
  LD_HD static void run(double2* x) {
    double2 t = x[0];
    x[0] = c_add(t, x[1]);
    x[1] = c_sub(t, x[1]);
  }
};

template <int SIGN> struct DFT<3, SIGN> {
  LD_HD static void run(double2* x) {
    constexpr double h = TwC<3, 1>::s;  // sqrt(3)/2
    double2 s = c_add(x[1], x[2]);
    double2 d = c_sub(x[1], x[2]);
    double2 m = make_double2(fma(-0.5, s.x, x[0].x), fma(-0.5, s.y, x[0].y));
    x[0] = c_add(x[0], s);
    double2 u = c_muli<SIGN>(c_scale(d, h));  // i*SIGN*h*(x1-x2)
    x[1] = c_add(m, u);
    x[2] = c_sub(m, u);
  }
};

template <int SIGN> struct DFT<4, SIGN> {
  LD_HD static void run(double2* x) {
    double2 a = c_add(x[0], x[2]);
    double2 b = c_sub(x[0], x[2]);
    double2 c = c_add(x[1], x[3]);
    double2 d = c_muli<SIGN>(c_sub(x[1], x[3]));
    x[0] = c_add(a, c);
    x[2] = c_sub(a, c);
    x[1] = c_add(b, d);
    x[3] = c_sub(b, d);
  }
};

template <int SIGN> struct DFT<5, SIGN> {
  LD_HD static void run(double2* x) {
    constexpr double c1 = TwC<5, 1>::c, c2 = TwC<5, 2>::c;
    constexpr double s1 = TwC<5, 1>::s, s2 = TwC<5, 2>::s;
    double2 t1 = c_add(x[1], x[4]), t2 = c_add(x[2], x[3]);
    double2 t3 = c_sub(x[1], x[4]), t4 = c_sub(x[2], x[3]);
    double2 x0 = x[0];
    x[0] = c_add(x0, c_add(t1, t2));
    double2 a1 = make_double2(fma(c2, t2.x, fma(c1, t1.x, x0.x)), fma(c2, t2.y, fma(c1, t1.y, x0.y)));
    double2 a2 = make_double2(fma(c1, t2.x, fma(c2, t1.x, x0.x)), fma(c1, t2.y, fma(c2, t1.y, x0.y)));
    double2 b1 = make_double2(fma(s2, t4.x, s1 * t3.x), fma(s2, t4.y, s1 * t3.y));
    double2 b2 = make_double2(fma(-s1, t4.x, s2 * t3.x), fma(-s1, t4.y, s2 * t3.y));
    b1 = c_muli<SIGN>(b1);
    b2 = c_muli<SIGN>(b2);
    x[1] = c_add(a1, b1);
    x[4] = c_sub(a1, b1);
    x[2] = c_add(a2, b2);
    x[3] = c_sub(a2, b2);
  }
};

// Odd prime P via the symmetric pairs (x_m +- x_{P-m}); used for P = 7.
template <int P, int SIGN> struct DFT_ODDPRIME {
  LD_HD static void run(double2* x) {
    constexpr int H = (P - 1) / 2;
    double2 sp[H], sm[H];
    sfor<H>([&](auto mc) {
      constexpr int m = decltype(mc)::value + 1;
      sp[m - 1] = c_add(x[m], x[P - m]);
      sm[m - 1] = c_sub(x[m], x[P - m]);
    });
    const double2 x0 = x[0];
    double2 y0 = x0;
    sfor<H>([&](auto mc) { y0 = c_add(y0, sp[decltype(mc)::value]); });
    sfor<H>([&](auto kc) {
      constexpr int k = decltype(kc)::value + 1;
      double2 a = x0, b = make_double2(0.0, 0.0);
      sfor<H>([&](auto mc) {
        constexpr int m = decltype(mc)::value + 1;
        constexpr int km = (k * m) % P;
        constexpr double c = TwC<P, km>::c, sn = TwC<P, km>::s;
        a = make_double2(fma(c, sp[m - 1].x, a.x), fma(c, sp[m - 1].y, a.y));
        b = make_double2(fma(sn, sm[m - 1].x, b.x), fma(sn, sm[m - 1].y, b.y));
      });
      const double2 ib = c_muli<SIGN>(b);
      x[k] = c_add(a, ib);
      x[P - k] = c_sub(a, ib);
    });
    x[0] = y0;
  }
};
template <int SIGN> struct DFT<7, SIGN> : DFT_ODDPRIME<7, SIGN> {};

// Cooley-Tukey R = R1*R2 with constant inner twiddles.
// input n = R2*n1 + n2, output k = k1 + R1*k2.
template <int R1, int R2, int SIGN> struct DFT_CT {
  LD_HD static void run(double2* x) {
    constexpr int R = R1 * R2;
    double2 y[R];
    sfor<R2>([&](auto n2c) {
      constexpr int n2 = decltype(n2c)::value;
      double2 t[R1];
      sfor<R1>([&](auto n1c) { t[decltype(n1c)::value] = x[R2 * decltype(n1c)::value + n2]; });
      DFT<R1, SIGN>::run(t);
      sfor<R1>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        y[n2 * R1 + k1] = tw_const<R, n2 * k1, SIGN>(t[k1]);
      });
    });
    sfor<R1>([&](auto k1c) {
      constexpr int k1 = decltype(k1c)::value;
      double2 t[R2];
      sfor<R2>([&](auto n2c) { t[decltype(n2c)::value] = y[decltype(n2c)::value * R1 + k1]; });
      DFT<R2, SIGN>::run(t);
      sfor<R2>([&](auto k2c) { x[k1 + R1 * decltype(k2c)::value] = t[decltype(k2c)::value]; });
    });
  }
};

constexpr int crt_index(int k1, int k2, int R1, int R2) {
  for (int k = 0; k < R1 * R2; ++k)
    if (k % R1 == k1 && k % R2 == k2) return k;
  return -1;
}

// Good-Thomas prime-factor R = R1*R2, gcd(R1,R2)=1: no twiddles.
// input n = (R2*n1 + R1*n2) mod R, output k = CRT(k1, k2).
template <int R1, int R2, int SIGN> struct DFT_PFA {
  LD_HD static void run(double2* x) {
    constexpr int R = R1 * R2;
    double2 y[R];
    sfor<R2>([&](auto n2c) {
      constexpr int n2 = decltype(n2c)::value;
      double2 t[R1];
      sfor<R1>([&](auto n1c) {
        constexpr int n1 = decltype(n1c)::value;
        t[n1] = x[(R2 * n1 + R1 * n2) % R];
      });
      DFT<R1, SIGN>::run(t);
      sfor<R1>([&](auto k1c) { y[n2 * R1 + decltype(k1c)::value] = t[decltype(k1c)::value]; });
    });
    sfor<R1>([&](auto k1c) {
      constexpr int k1 = decltype(k1c)::value;
      double2 t[R2];
      sfor<R2>([&](auto n2c) { t[decltype(n2c)::value] = y[decltype(n2c)::value * R1 + k1]; });
      DFT<R2, SIGN>::run(t);
      sfor<R2>([&](auto k2c) {
        constexpr int k2 = decltype(k2c)::value;
        x[crt_index(k1, k2, R1, R2)] = t[k2];
      });
    });
  }
};

template <int SIGN> struct DFT<6, SIGN> : DFT_PFA<2, 3, SIGN> {};
template <int SIGN> struct DFT<8, SIGN> : DFT_CT<2, 4, SIGN> {};
template <int SIGN> struct DFT<9, SIGN> : DFT_CT<3, 3, SIGN> {};
template <int SIGN> struct DFT<10, SIGN> : DFT_PFA<2, 5, SIGN> {};
template <int SIGN> struct DFT<12, SIGN> : DFT_PFA<3, 4, SIGN> {};
template <int SIGN> struct DFT<15, SIGN> : DFT_PFA<3, 5, SIGN> {};
template <int SIGN> struct DFT<16, SIGN> : DFT_CT<4, 4, SIGN> {};
template <int SIGN> struct DFT<18, SIGN> : DFT_PFA<2, 9, SIGN> {};
template <int SIGN> struct DFT<20, SIGN> : DFT_PFA<4, 5, SIGN> {};
template <int SIGN> struct DFT<24, SIGN> : DFT_PFA<3, 8, SIGN> {};
template <int SIGN> struct DFT<27, SIGN> : DFT_CT<3, 9, SIGN> {};
template <int SIGN> struct DFT<14, SIGN> : DFT_PFA<2, 7, SIGN> {};
template <int SIGN> struct DFT<21, SIGN> : DFT_PFA<3, 7, SIGN> {};
template <int SIGN> struct DFT<28, SIGN> : DFT_PFA<4, 7, SIGN> {};
template <int SIGN> struct DFT<32, SIGN> : DFT_CT<4, 8, SIGN> {};

// ------------------------------------------------------------ radix plan
// Factorisation of a transform length into in-register radices. Stage 0 takes
// the largest odd radix >= 9 when there is one, so its stride-R shared-memory
// writes are bank-conflict free; otherwise (power-of-two-ish lengths) the
// shared-memory layout is swizzled instead (Plan::swizzle).
constexpr int kRadixPref[] = {16, 15, 12, 14, 9, 10, 8, 7, 6, 5, 4, 3, 2};
// Largest radix for a line length: long lines whose fused middle stage would
// hold two radix-16 tasks run register-lean radix-8 plans instead.
#ifndef LATTDSE_MAXR_LONG
#define LATTDSE_MAXR_LONG 16
#endif
constexpr int max_radix(int L) { return L >= 4096 ? LATTDSE_MAXR_LONG : 32; }

constexpr int pick_radix(int rem, int maxr = 32) {
  for (int r : kRadixPref)
    if (r <= maxr && rem % r == 0) return r;
  return rem;  // rejected by the static_assert in Plan
}
constexpr int first_radix(int L) {
  for (int r : {21, 15, 9})
    if (r <= max_radix(L) && L % r == 0) return r;
  return pick_radix(L, max_radix(L));
}

// Explicit plans. The first four: long lines the greedy rule would end with
// a radix-2/3 stage (three balanced stages instead). 1080: measured per
// pass on config 3 with the lean pass4 kernels (profiles/r2/p4_sweep*.txt,
// us per ROW launch over 64 members): (9, 12, 10) 283, (10, 12, 9) 287,
// (9, 10, 12) 310, (15, 8, 9) 326, (9, 8, 15) 328 -- balanced task counts
// per stage (120 / 90 / 108 tasks on 128 threads) and a small radix in the
// fused mid stage, which holds the data and the prefetched diagonal
// together, beat the larger radices. 486: (9, 9, 6) and (9, 6, 9) tie.
struct PlanOverride {
  int L, r[4];
};
// build-time experiments: -include a header defining LATTDSE_PLAN_X/Y as
// "L, r0, r1, r2, r3" (scripts/build_variant.sh) takes precedence
#ifndef LATTDSE_PLAN_X
#define LATTDSE_PLAN_X 0, 0, 0, 0, 0
#endif
#ifndef LATTDSE_PLAN_Y
#define LATTDSE_PLAN_Y 0, 0, 0, 0, 0
#endif
constexpr int kPlanX[5] = {LATTDSE_PLAN_X};
constexpr int kPlanY[5] = {LATTDSE_PLAN_Y};
constexpr PlanOverride kPlanOverride[] = {
    {kPlanX[0] ? kPlanX[0] : -1, {kPlanX[1], kPlanX[2], kPlanX[3], kPlanX[4]}},
    {kPlanY[0] ? kPlanY[0] : -1, {kPlanY[1], kPlanY[2], kPlanY[3], kPlanY[4]}},
    {2592, {9, 16, 18, 0}},  {3240, {15, 12, 18, 0}}, {3888, {27, 16, 9, 0}},
    {4320, {15, 16, 18, 0}}, {1080, {9, 12, 10, 0}},  {0, {0, 0, 0, 0}},
};
constexpr int override_radix(int L, int s) {
  for (const auto& o : kPlanOverride)
    if (o.L == L) return s < 4 ? o.r[s] : 0;
  return -1;
}

template <int L> struct Plan {
  static constexpr int radix(int s) {
    if (override_radix(L, 0) > 0) {
      int rem = L;
      for (int i = 0; i < s; ++i) rem /= override_radix(L, i);
      return rem > 1 ? override_radix(L, s) : 1;
    }
    int rem = L;
    int r = first_radix(L);
    for (int i = 0; i < s; ++i) {
      rem /= r;
      r = pick_radix(rem, max_radix(L));
    }
    return r;
  }
  static constexpr int count() {
    int n = 0, rem = L;
    while (rem > 1) {
      rem /= radix(n);
      ++n;
    }
    return n;
  }
  static constexpr int nst = count();
  // Ns = product of the radices of the earlier stages
  static constexpr int ns(int s) {
    int p = 1;
    for (int i = 0; i < s; ++i) p *= radix(i);
    return p;
  }
  static constexpr int max_tasks() {
    int m = 0;
    for (int s = 0; s < nst; ++s) m = (L / radix(s)) > m ? (L / radix(s)) : m;
    return m;
  }
  // Per-stage twiddle table: stage s >= 1 owns (R_s - 1) * Ns_s entries
  // laid out [r-1][k] = exp(-2 pi i r k / (Ns_s R_s)), so the threads of a
  // warp (consecutive k) read consecutive entries.
  static constexpr int tw_offset(int s) {
    int o = 0;
    for (int i = 1; i < s; ++i) o += (radix(i) - 1) * ns(i);
    return o;
  }
  static constexpr int tw_size = tw_offset(nst);
  // even radix in stage 0 of either direction (PlanX<L, true> starts with the
  // last radix) -> stride-R stage-0 writes conflict; pad 1 slot per 16
  static constexpr bool swizzle = (radix(0) % 2 == 0 || radix(nst - 1) % 2 == 0) && L >= 16;
  static constexpr int phys(int i) { return swizzle ? i + (i >> 4) : i; }
  static constexpr bool valid() {
    for (int s = 0; s < nst; ++s) {
      int r = radix(s);
      if (r > 32) return false;
    }
    return L >= 2;
  }
  static_assert(valid(), "transform length must factor into radices <= 32 from kRadixPref");
};

// The plan in forward (REV = false) or reversed radix order. The second
// transform of a fused pass uses the reversed order so that its first stage
// touches exactly the elements the first transform's last stage produced.
template <int L, bool REV> struct PlanX {
  using P = Plan<L>;
  static constexpr int nst = P::nst;
  static constexpr int radix(int s) { return REV ? P::radix(nst - 1 - s) : P::radix(s); }
  static constexpr int ns(int s) {
    int p = 1;
    for (int i = 0; i < s; ++i) p *= radix(i);
    return p;
  }
  static constexpr int tw_offset(int s) {
    int o = 0;
    for (int i = 1; i < s; ++i) o += (radix(i) - 1) * ns(i);
    return o;
  }
};

// Host: per-stage twiddle table for a radix plan (layout of Plan::tw_offset),
// correctly rounded via long double. out must hold sum_{s>=1} (R_s-1) Ns_s.
inline int build_stage_twiddles(const int* radix, int nst, double2* out) {
  const long double pi = 3.141592653589793238462643383279502884L;
  int o = 0, ns = radix[0];
  for (int s = 1; s < nst; ++s) {
    const int R = radix[s];
    const long long len = (long long)ns * R;
    for (int r = 1; r < R; ++r)
      for (int k = 0; k < ns; ++k) {
        const long long q = ((long long)r * k) % len;
        const long double a = -2.0L * pi * (long double)q / (long double)len;
        if (out) out[o] = make_double2((double)cosl(a), (double)sinl(a));
        ++o;
      }
    ns *= R;
  }
  return o;
}

template <int L> inline int plan_twiddles(double2* out, bool rev = false) {
  int radix[32];
  for (int s = 0; s < Plan<L>::nst; ++s) radix[s] = Plan<L>::radix(rev ? Plan<L>::nst - 1 - s : s);
  return build_stage_twiddles(radix, Plan<L>::nst, out);
}

}  // namespace lattdse_dev
