// Host-side emulation of the pass kernels (no GPU needed): every CTA of the
// grid is run sequentially, each stage as "all threads read, then all threads
// write", which is exactly the ordering the __syncthreads() in DevExec
// enforce. Checks the small DFTs and every pass program against naive O(L^2)
// DFTs in long double. Built and run by tests/test_fft_core_emulation.py.
#include <array>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <string>

#include "fft_pass.cuh"

using namespace lattdse_dev;
using cld = std::complex<long double>;

struct HostExec {
  template <class St, class C> static void stage(const C& c) {
    using Regs = double2[St::TPT][St::R];
    std::vector<std::array<double2, St::TPT * St::R>> regs(St::nt);
    for (int tid = 0; tid < St::nt; ++tid) St::read(c, tid, *reinterpret_cast<Regs*>(regs[tid].data()));
    for (int tid = 0; tid < St::nt; ++tid) St::write(c, tid, *reinterpret_cast<Regs*>(regs[tid].data()));
  }
};

static int g_fail = 0;
static void check(const char* what, double err, double tol) {
  bool ok = err <= tol;
  std::printf("%-48s err=%.3e %s\n", what, err, ok ? "ok" : "FAIL");
  if (!ok) g_fail = 1;
}

static const long double kPi = 3.141592653589793238462643383279502884L;

static double2 root(long long t, long long n, int sign) {  // exp(sign 2 pi i t/n)
  long double a = 2.0L * kPi * (long double)(t % n) / (long double)n;
  return make_double2((double)cosl(a), (double)(sign * sinl(a)));
}

static std::vector<cld> naive_dft(const std::vector<cld>& x, int sign) {
  size_t n = x.size();
  std::vector<cld> y(n);
  for (size_t k = 0; k < n; ++k) {
    cld acc = 0;
    for (size_t j = 0; j < n; ++j) {
      long double a = 2.0L * kPi * (long double)((j * k) % n) / (long double)n;
      acc += x[j] * cld(cosl(a), sign * sinl(a));
    }
    y[k] = acc;
  }
  return y;
}

template <int R, int SIGN> void test_dft() {
  std::mt19937_64 rng(R * 7 + SIGN);
  std::uniform_real_distribution<double> u(-1, 1);
  double2 v[R];
  std::vector<cld> x(R);
  for (int i = 0; i < R; ++i) {
    v[i] = make_double2(u(rng), u(rng));
    x[i] = cld(v[i].x, v[i].y);
  }
  DFT<R, SIGN>::run(v);
  auto y = naive_dft(x, SIGN);
  double e = 0;
  for (int i = 0; i < R; ++i) e = std::max(e, (double)std::abs(y[i] - cld(v[i].x, v[i].y)));
  char buf[64];
  std::snprintf(buf, sizeof buf, "DFT<%d,%+d>", R, SIGN);
  check(buf, e, 1e-14 * R);
}

struct Tables {
  std::vector<double2> fft_tw;
  std::vector<double2> tw_lo, tw_hi;
  int shift = 0;
  std::vector<double2> fft_tw2;
  template <int L> void build_plan() {
    fft_tw.resize(std::max(1, plan_twiddles<L>(nullptr)));
    plan_twiddles<L>(fft_tw.data());
    fft_tw2.resize(std::max(1, plan_twiddles<L>(nullptr, true)));
    plan_twiddles<L>(fft_tw2.data(), true);
  }
  void build(int L, long long M) {
    shift = 0;
    while ((1LL << (2 * shift)) < M) ++shift;
    long long nlo = 1LL << shift, nhi = (M + nlo - 1) / nlo;
    tw_lo.resize(nlo);
    tw_hi.resize(nhi);
    for (long long t = 0; t < nlo; ++t) tw_lo[t] = root(t, M, -1);
    for (long long t = 0; t < nhi; ++t) tw_hi[t] = root(t * nlo, M, -1);
  }
};

template <int AXIS, int L, int B, int NT, int PROG, int SIGN1>
void emulate(PassArgs a, int nlines, int nbatch) {
  std::vector<double2> sm(SmemGeom<L, B>::bytes / 16);
  for (int bat = 0; bat < nbatch; ++bat)
    for (int blk = 0; blk < (nlines + B - 1) / B; ++blk) {
      Ctx<AXIS, L, B, PROG> c{sm.data(), a, blk * B, bat};
      run_pass<HostExec, AXIS, L, B, NT, PROG, SIGN1>(c);
    }
}

// Lines along the contiguous (ROW) or strided (COL) axis: single transform.
template <int AXIS, int L, int B, int NT, int SIGN> void test_lines(int other) {
  // 2-D view: ROW -> other rows of length L; COL -> L rows of length other
  int nrows = AXIS == AX_ROW ? other : L, ncols = AXIS == AX_ROW ? L : other;
  std::mt19937_64 rng(L * 131 + AXIS);
  std::uniform_real_distribution<double> u(-1, 1);
  int nb = 2;
  long long n = (long long)nrows * ncols;
  std::vector<double2> x(n * nb), y(n * nb), diag(n);
  for (auto& v : x) v = make_double2(u(rng), u(rng));
  for (auto& v : diag) {
    double th = u(rng) * 3;
    v = make_double2(std::cos(th), std::sin(th));
  }
  Tables tb;
  tb.build(L, 4);
  tb.template build_plan<L>();
  PassArgs a{};
  a.in = x.data();
  a.out = y.data();
  a.in_bstride = a.out_bstride = n;
  a.nvalid_in = a.nvalid_mid = a.nvalid_out = n;
  a.ncols = ncols;
  a.nlines = AXIS == AX_ROW ? nrows : ncols;
  a.diag_kind = DG_CPLX;
  a.diag = diag.data();
  a.fft_tw = tb.fft_tw.data();
  a.fft_tw2 = tb.fft_tw2.data();
  a.tw_lo = tb.tw_lo.data();
  a.tw_hi = tb.tw_hi.data();
  a.tw_shift = tb.shift;
  emulate<AXIS, L, B, NT, PROG_LOADDIAG, SIGN>(a, AXIS == AX_ROW ? nrows : ncols, nb);
  double e = 0, mx = 0;
  for (int bat = 0; bat < nb; ++bat)
    for (int line = 0; line < (AXIS == AX_ROW ? nrows : ncols); ++line) {
      std::vector<cld> v(L);
      auto idx = [&](int i) { return AXIS == AX_ROW ? (long long)line * L + i : (long long)i * ncols + line; };
      for (int i = 0; i < L; ++i) {
        long long j = idx(i);
        cld xv(x[bat * n + j].x, x[bat * n + j].y), dv(diag[j].x, diag[j].y);
        v[i] = xv * dv;
      }
      auto w = naive_dft(v, SIGN);
      for (int i = 0; i < L; ++i) {
        long long j = idx(i);
        e = std::max(e, (double)std::abs(w[i] - cld(y[bat * n + j].x, y[bat * n + j].y)));
        mx = std::max(mx, (double)std::abs(w[i]));
      }
    }
  char buf[96];
  std::snprintf(buf, sizeof buf, "lines axis=%d L=%d B=%d NT=%d sign=%+d", AXIS, L, B, NT, SIGN);
  check(buf, e / mx, 4e-16 * 20);
}

// Double program: T1(SIGN1) -> x diag (mask) -> T2(-SIGN1), in place.
template <int AXIS, int L, int B, int NT, int SIGN1> void test_double(int other, long long nmid) {
  int nrows = AXIS == AX_ROW ? other : L, ncols = AXIS == AX_ROW ? L : other;
  std::mt19937_64 rng(L * 17 + AXIS + 5);
  std::uniform_real_distribution<double> u(-1, 1);
  long long n = (long long)nrows * ncols;
  std::vector<double2> x(n), y(n), lut(64);
  std::vector<unsigned short> idx16(n);
  for (auto& v : x) v = make_double2(u(rng), u(rng));
  for (auto& v : lut) {
    double th = u(rng) * 3;
    v = make_double2(std::cos(th), std::sin(th));
  }
  for (auto& i : idx16) i = (unsigned short)(rng() % 64);
  y = x;
  Tables tb;
  tb.build(L, 4);
  tb.template build_plan<L>();
  PassArgs a{};
  a.in = y.data();
  a.out = y.data();
  a.in_bstride = a.out_bstride = n;
  a.nvalid_in = a.nvalid_out = n;
  a.nvalid_mid = nmid;
  a.ncols = ncols;
  a.nlines = AXIS == AX_ROW ? nrows : ncols;
  a.diag_kind = DG_LUT16;
  a.diag_idx = idx16.data();
  a.lut = lut.data();
  a.fft_tw = tb.fft_tw.data();
  a.fft_tw2 = tb.fft_tw2.data();
  a.tw_lo = tb.tw_lo.data();
  a.tw_hi = tb.tw_hi.data();
  a.tw_shift = tb.shift;
  emulate<AXIS, L, B, NT, PROG_DOUBLE, SIGN1>(a, AXIS == AX_ROW ? nrows : ncols, 1);
  double e = 0, mx = 0;
  for (int line = 0; line < (AXIS == AX_ROW ? nrows : ncols); ++line) {
    std::vector<cld> v(L);
    auto idx = [&](int i) { return AXIS == AX_ROW ? (long long)line * L + i : (long long)i * ncols + line; };
    for (int i = 0; i < L; ++i) v[i] = cld(x[idx(i)].x, x[idx(i)].y);
    auto w = naive_dft(v, SIGN1);
    for (int i = 0; i < L; ++i) {
      long long j = idx(i);
      cld d(lut[idx16[j]].x, lut[idx16[j]].y);
      w[i] = j < nmid ? w[i] * d : cld(0);
    }
    auto z = naive_dft(w, -SIGN1);
    for (int i = 0; i < L; ++i) {
      long long j = idx(i);
      e = std::max(e, (double)std::abs(z[i] - cld(y[j].x, y[j].y)));
      mx = std::max(mx, (double)std::abs(z[i]));
    }
  }
  char buf[96];
  std::snprintf(buf, sizeof buf, "double axis=%d L=%d B=%d NT=%d sign=%+d", AXIS, L, B, NT, SIGN1);
  check(buf, e / mx, 4e-16 * 40);
}

// Four-step forward DFT of length M = M1*M2: COL(LOADDIAG, FFT_M1, post-tw)
// then ROW(FFT_M2 with store); output X[k1 + M1 k2] at (row k1, col k2).
template <int M1, int M2> void test_fourstep(long long nvalid) {
  const long long M = (long long)M1 * M2;
  std::mt19937_64 rng(M);
  std::uniform_real_distribution<double> u(-1, 1);
  std::vector<double2> x(nvalid), work(M), ones(M, make_double2(1, 0));
  for (auto& v : x) v = make_double2(u(rng), u(rng));
  Tables t1, t2;
  t1.build(M1, M);
  t2.build(M2, M);
  t1.template build_plan<M1>();
  t2.template build_plan<M2>();
  PassArgs a{};
  a.in = x.data();
  a.out = work.data();
  a.in_bstride = nvalid;
  a.out_bstride = M;
  a.nvalid_in = nvalid;
  a.nvalid_mid = a.nvalid_out = M;
  a.ncols = M2;
  a.nlines = M2;
  a.diag_kind = DG_CPLX;
  a.diag = ones.data();
  a.post_tw = 1;
  a.fft_tw = t1.fft_tw.data();
  a.fft_tw2 = t1.fft_tw2.data();
  a.tw_lo = t1.tw_lo.data();
  a.tw_hi = t1.tw_hi.data();
  a.tw_shift = t1.shift;
  emulate<AX_COL, M1, 2, 64, PROG_LOADDIAG, -1>(a, M2, 1);
  PassArgs b = a;
  b.in = work.data();
  b.out = work.data();
  b.in_bstride = M;
  b.nvalid_in = M;
  b.post_tw = 0;
  b.diag_kind = DG_NONE;
  b.ncols = M2;
  b.nlines = M1;
  b.fft_tw = t2.fft_tw.data();
  b.fft_tw2 = t2.fft_tw2.data();
  emulate<AX_ROW, M2, 1, 64, PROG_LOADDIAG, -1>(b, M1, 1);
  std::vector<cld> xv(M, cld(0));
  for (long long j = 0; j < nvalid; ++j) xv[j] = cld(x[j].x, x[j].y);
  auto X = naive_dft(xv, -1);
  double e = 0, mx = 0;
  for (int k1 = 0; k1 < M1; ++k1)
    for (int k2 = 0; k2 < M2; ++k2) {
      cld got(work[(long long)k1 * M2 + k2].x, work[(long long)k1 * M2 + k2].y);
      e = std::max(e, (double)std::abs(got - X[k1 + (long long)M1 * k2]));
      mx = std::max(mx, (double)std::abs(X[k1 + (long long)M1 * k2]));
    }
  char buf[96];
  std::snprintf(buf, sizeof buf, "fourstep %dx%d nvalid=%lld", M1, M2, nvalid);
  check(buf, e / mx, 1e-14);
}

// Good-Thomas forward DFT of length M = M1*M2 (gcd 1): COL(LOADDIAG, pfa
// gather from natural order) then ROW(FFT). X[k] lands at (k mod M1, k mod M2).
template <int M1, int M2> void test_pfa(long long nvalid) {
  const long long M = (long long)M1 * M2;
  std::mt19937_64 rng(M + 5);
  std::uniform_real_distribution<double> u(-1, 1);
  std::vector<double2> x(nvalid), work(M), dg(nvalid);
  for (auto& v : x) v = make_double2(u(rng), u(rng));
  for (auto& v : dg) v = make_double2(u(rng), u(rng));
  Tables t1, t2;
  t1.template build_plan<M1>();
  t2.template build_plan<M2>();
  PassArgs a{};
  a.in = x.data();
  a.out = work.data();
  a.in_bstride = nvalid;
  a.out_bstride = M;
  a.nvalid_in = nvalid;
  a.nvalid_mid = a.nvalid_out = M;
  a.ncols = M2;
  a.nlines = M2;
  a.diag_kind = DG_CPLX;
  a.diag = dg.data();
  a.fft_tw = t1.fft_tw.data();
  a.fft_tw2 = t1.fft_tw2.data();
  a.pfa = 1;
  a.pM1 = M1;
  a.pM2 = M2;
  a.pM = M;
  emulate<AX_COL, M1, 2, 64, PROG_LOADDIAG, -1>(a, M2, 1);
  PassArgs b{};
  b.in = work.data();
  b.out = work.data();
  b.in_bstride = b.out_bstride = M;
  b.nvalid_in = b.nvalid_mid = b.nvalid_out = M;
  b.ncols = M2;
  b.nlines = M1;
  b.fft_tw = t2.fft_tw.data();
  b.fft_tw2 = t2.fft_tw2.data();
  emulate<AX_ROW, M2, 1, 64, PROG_LOADDIAG, -1>(b, M1, 1);
  std::vector<cld> xv(M, cld(0));
  for (long long j = 0; j < nvalid; ++j) xv[j] = cld(x[j].x, x[j].y) * cld(dg[j].x, dg[j].y);
  auto X = naive_dft(xv, -1);
  double e = 0, mx = 0;
  for (long long k = 0; k < M; ++k) {
    long long p = (k % M1) * M2 + (k % M2);
    e = std::max(e, (double)std::abs(cld(work[p].x, work[p].y) - X[k]));
    mx = std::max(mx, (double)std::abs(X[k]));
  }
  // inverse: ROW IFFT then COL STOREDIAG (pfa scatter to natural order, x diag)
  PassArgs c = b;
  emulate<AX_ROW, M2, 1, 64, PROG_LOADDIAG, 1>(c, M1, 1);
  std::vector<double2> back(nvalid), ones(nvalid, make_double2(1.0 / (double)M, 0));
  PassArgs d = a;
  d.in = work.data();
  d.out = back.data();
  d.in_bstride = M;
  d.out_bstride = nvalid;
  d.nvalid_in = M;
  d.nvalid_out = nvalid;
  d.diag = ones.data();
  emulate<AX_COL, M1, 2, 64, PROG_STOREDIAG, 1>(d, M2, 1);
  double e2 = 0;
  for (long long j = 0; j < nvalid; ++j) e2 = std::max(e2, (double)std::abs(cld(back[j].x, back[j].y) - xv[j]));
  char buf[96];
  std::snprintf(buf, sizeof buf, "pfa %dx%d nvalid=%lld fwd", M1, M2, nvalid);
  check(buf, e / mx, 1e-14);
  std::snprintf(buf, sizeof buf, "pfa %dx%d nvalid=%lld round trip", M1, M2, nvalid);
  check(buf, e2, 1e-14);
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "c1") {
    const long long M1 = 1215, M2 = 1728, M = M1 * M2;
    const long long N = 1048583;
    std::vector<double2> buf(M, make_double2(1.0, 0.5)), inN(N, make_double2(0.5, 0.25)), dN(N, make_double2(1, 0));
    Tables t1;
    t1.build(M1, M);
    t1.template build_plan<M1>();
    PassArgs a{};
    a.in = inN.data();
    a.out = buf.data();
    a.in_bstride = N;
    a.out_bstride = M;
    a.nvalid_in = N;
    a.nvalid_mid = a.nvalid_out = M;
    a.ncols = M2;
    a.nlines = M2;
    a.post_tw = 1;
    a.diag_kind = DG_CPLX;
    a.diag = dN.data();
    a.fft_tw = t1.fft_tw.data();
    a.fft_tw2 = t1.fft_tw2.data();
    a.tw_lo = t1.tw_lo.data();
    a.tw_hi = t1.tw_hi.data();
    a.tw_shift = t1.shift;
    std::printf("tw_lo %zu tw_hi %zu shift %d\n", t1.tw_lo.size(), t1.tw_hi.size(), t1.shift);
    emulate<AX_COL, 1215, 2, 256, PROG_LOADDIAG, -1>(a, M2, 1);
    std::printf("c1 col entry emulated ok %f\n", buf[12345].x);
    return 0;
  }
  if (argc > 1) {
    test_lines<AX_COL, 1215, 2, 256, -1>(4);
    test_lines<AX_COL, 1215, 2, 256, 1>(3);
    test_double<AX_COL, 1215, 2, 256, 1>(4, 1000);
    test_lines<AX_ROW, 1728, 1, 224, -1>(2);
    test_double<AX_ROW, 1728, 1, 224, -1>(2, 100000);
    test_lines<AX_COL, 4096, 2, 256, -1>(2);
    test_double<AX_ROW, 4096, 1, 256, 1>(1, 100000);
    return g_fail;
  }

  test_dft<2, -1>(); test_dft<3, -1>(); test_dft<4, -1>(); test_dft<5, -1>();
  test_dft<6, -1>(); test_dft<8, -1>(); test_dft<9, -1>(); test_dft<10, -1>();
  test_dft<12, -1>(); test_dft<15, -1>(); test_dft<16, -1>(); test_dft<18, 1>();
  test_dft<20, 1>(); test_dft<24, 1>(); test_dft<27, 1>(); test_dft<32, 1>();
  test_dft<3, 1>(); test_dft<5, 1>(); test_dft<9, 1>(); test_dft<16, 1>();
  test_dft<7, -1>(); test_dft<7, 1>(); test_dft<14, 1>(); test_dft<21, -1>(); test_dft<28, 1>();
  test_lines<AX_ROW, 1728, 1, 128, -1>(3);
  test_lines<AX_ROW, 720, 2, 128, 1>(4);
  test_lines<AX_COL, 1215, 2, 128, -1>(4);
  test_lines<AX_COL, 96, 4, 64, 1>(8);
  test_lines<AX_ROW, 16, 4, 32, -1>(8);
  test_lines<AX_ROW, 16, 4, 32, 1>(7);
  test_lines<AX_COL, 12, 8, 32, 1>(5);
  test_double<AX_ROW, 729, 1, 128, -1>(3, 1000000);
  test_double<AX_COL, 90, 2, 64, 1>(6, 300);
  test_double<AX_COL, 12, 2, 32, 1>(4, 30);
  test_fourstep<12, 10>(61);
  test_fourstep<96, 90>(4099);
  test_pfa<9, 16>(70);
  test_pfa<27, 64>(800);
  test_pfa<64, 135>(4099);
  test_lines<AX_COL, 1029, 2, 160, -1>(3);
  test_double<AX_ROW, 1029, 1, 160, 1>(2, 1500);
  std::printf(g_fail ? "SOME FAILED\n" : "ALL OK\n");
  return g_fail;
}
