// ===========================================================================
// TEST INFRASTRUCTURE ONLY -- CPU ORACLE. Never linked into or called by the
// product (paper_1808_06357_b200/). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load oracle/_build/liboracle.so.
//
// A plain C++ (+OpenMP) restatement of the reference's specification for the
// hot path. The reference implements only lattice-core; its solver exists as
// SPEC.md prose, restated here literally:
//   points        SPEC.md:49-57, lattice.cpp:279-330 (exact numerators mod L)
//   cbc           SPEC.md:117-137 (exhaustive, no shortlist)
//   antialias     SPEC.md:178-187, PAPER.md:1321-1326 (literal shell walk:
//                 ascending ||h||^2, lexicographic inside a shell, first seen)
//   analyze       SPEC.md:243-251 (r-dim FFT of the n1 x .. x nr tensor, 1/N)
//   synthesize    SPEC.md:253-261 (inverse, unnormalised)
//   propagator    SPEC.md:319-323 (kin_phase, pot_half_phase)
//   strang_step   SPEC.md:336-344 (synthesize, xpotH, analyze, xkin,
//                 synthesize, xpotH, analyze -- no fusion)
//   l2_norm       SPEC.md:356-362;  energy SPEC.md:364-372
// with its own FFT (recursive mixed radix + Bluestein) independent of both the
// GPU kernels and the product's setup FFT.
//
// Parity status: pinned by the reference's own lattice-core outputs
// (tests/golden/lattice_ref.json, built from /root/reference sources) and by
// the SPEC known-answer tests (naive DFT, dense 8x8 expm, commuting cases,
// closed-form wce); the reference has no solver to run, see DESIGN.md §Oracle.
// ===========================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

using cd = std::complex<double>;
using i64 = std::int64_t;

namespace {

const long double PI_L = 3.141592653589793238462643383279502884L;

// ------------------------------------------------------------------- FFT
bool smooth7(i64 n) {
  for (int p : {2, 3, 5, 7})
    while (n % p == 0) n /= p;
  return n == 1;
}
i64 next_smooth7(i64 n) {
  while (!smooth7(n)) ++n;
  return n;
}

struct Fft {
  i64 n0;
  std::vector<cd> w;  // exp(-2 pi i k / n0)
  std::vector<int> fac;
  // large sizes: n0 = n1 * n2, sub-transforms run in parallel (four-step)
  i64 n1 = 0, n2 = 0;
  Fft* f1 = nullptr;
  Fft* f2 = nullptr;
  explicit Fft(i64 n) : n0(n), w(n) {
    for (i64 k = 0; k < n; ++k) {
      long double a = -2.0L * PI_L * (long double)k / (long double)n;
      w[k] = cd((double)cosl(a), (double)sinl(a));
    }
    i64 m = n;
    for (int p : {4, 2, 3, 5, 7})
      while (m % p == 0) {
        fac.push_back(p);
        m /= p;
      }
    if (n >= (1 << 14)) {
      n1 = 1;
      for (int p : fac)
        if (n1 * n1 < n) n1 *= p;
      n2 = n / n1;
      f1 = new Fft(n1);
      f2 = new Fft(n2);
    }
  }
  ~Fft() {
    delete f1;
    delete f2;
  }
  Fft(const Fft&) = delete;
  Fft& operator=(const Fft&) = delete;
  // out[0..n) = DFT of in[0], in[s], in[2s] ...; depth indexes fac (sequential)
  void rec(const cd* in, i64 s, cd* out, i64 n, int depth, int sign) const {
    if (n == 1) {
      out[0] = in[0];
      return;
    }
    const int p = fac[depth];
    const i64 m = n / p;
    for (int q = 0; q < p; ++q) rec(in + q * s, s * p, out + q * m, m, depth + 1, sign);
    const i64 ws = n0 / n;  // w_n^t = w[t*ws]
    for (i64 k = 0; k < m; ++k) {
      cd y[7], z[7];
      for (int r = 0; r < p; ++r) {
        cd t = w[(r * k * ws) % n0];
        if (sign > 0) t = std::conj(t);
        y[r] = out[r * m + k] * t;
      }
      for (int a = 0; a < p; ++a) {
        cd acc = 0;
        for (int r = 0; r < p; ++r) {
          cd t = w[((a * r) % p) * (n0 / p)];
          if (sign > 0) t = std::conj(t);
          acc += y[r] * t;
        }
        z[a] = acc;
      }
      for (int a = 0; a < p; ++a) out[k + a * m] = z[a];
    }
  }
  void run(const cd* in, cd* out, int sign) const {
    if (!f1) {
      rec(in, 1, out, n0, 0, sign);
      return;
    }
    // X[k1 + n1 k2] = sum_j2 w_n2^(j2 k2) w_n^(j2 k1) sum_j1 x[n2 j1 + j2] w_n1^(j1 k1)
    std::vector<cd> tmp((size_t)n0);
#pragma omp parallel for schedule(static)
    for (i64 j2 = 0; j2 < n2; ++j2) {
      std::vector<cd> col(n1);
      f1->rec(in + j2, n2, col.data(), n1, 0, sign);
      for (i64 k1 = 0; k1 < n1; ++k1) {
        cd t = w[(j2 * k1) % n0];
        if (sign > 0) t = std::conj(t);
        tmp[k1 * n2 + j2] = col[k1] * t;
      }
    }
#pragma omp parallel for schedule(static)
    for (i64 k1 = 0; k1 < n1; ++k1) {
      std::vector<cd> row(n2);
      f2->rec(tmp.data() + k1 * n2, 1, row.data(), n2, 0, sign);
      for (i64 k2 = 0; k2 < n2; ++k2) out[k1 + n1 * k2] = row[k2];
    }
  }
};

// Unnormalised DFT of any length; Bluestein (with 7-smooth M) for the rest.
struct Dft {
  i64 n, M = 0;
  Fft* direct = nullptr;
  Fft* conv = nullptr;
  std::vector<cd> chirp, bhat;  // chirp_j = exp(-pi i j^2/n); bhat = FFT_M(conj chirp, wrapped)
  explicit Dft(i64 n_) : n(n_) {
    if (smooth7(n)) {
      direct = new Fft(n);
      return;
    }
    M = next_smooth7(2 * n - 1);
    conv = new Fft(M);
    chirp.resize(n);
    for (i64 j = 0; j < n; ++j) {
      i64 q = (i64)(((__int128)j * j) % (2 * n));
      long double a = -PI_L * (long double)q / (long double)n;
      chirp[j] = cd((double)cosl(a), (double)sinl(a));
    }
    std::vector<cd> b(M, 0.0);
    b[0] = std::conj(chirp[0]);
    for (i64 j = 1; j < n; ++j) b[j] = b[M - j] = std::conj(chirp[j]);
    bhat.resize(M);
    conv->run(b.data(), bhat.data(), -1);
  }
  ~Dft() {
    delete direct;
    delete conv;
  }
  // sign -1 forward, +1 inverse (unnormalised)
  void run(const cd* in, cd* out, int sign) const {
    if (direct) {
      direct->run(in, out, sign);
      return;
    }
    // inverse via conjugation: IDFT(x) = conj(DFT(conj x))
    std::vector<cd> a(M, 0.0), A(M);
    for (i64 j = 0; j < n; ++j) a[j] = (sign < 0 ? in[j] : std::conj(in[j])) * chirp[j];
    conv->run(a.data(), A.data(), -1);
    for (i64 t = 0; t < M; ++t) A[t] *= bhat[t];
    conv->run(A.data(), a.data(), +1);
    const double inv = 1.0 / (double)M;
    for (i64 k = 0; k < n; ++k) {
      cd v = a[k] * chirp[k] * inv;
      out[k] = sign < 0 ? v : std::conj(v);
    }
  }
};

// ------------------------------------------------------------- lattice bits
struct Lat {
  int d, r;
  std::vector<std::vector<i64>> Z;  // r columns of length d
  std::vector<i64> n;
  i64 N, L;
};

Lat make_lat(int d, int r, const i64* Z, const i64* n) {
  Lat l;
  l.d = d;
  l.r = r;
  l.Z.assign(r, std::vector<i64>(d));
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < d; ++j) l.Z[i][j] = Z[i * d + j];
  l.n.assign(n, n + r);
  l.N = 1;
  l.L = 1;
  for (i64 m : l.n) {
    l.N *= m;
    l.L = std::lcm(l.L, m);
  }
  return l;
}

i64 modp(__int128 v, i64 m) {
  __int128 q = v % m;
  return (i64)(q < 0 ? q + m : q);
}

// points: kappa -> k (last index fastest) -> x_j = sum_i (L/n_i) z_ij k_i mod L
std::vector<i64> points(const Lat& l) {
  std::vector<i64> out((size_t)l.N * l.d);
#pragma omp parallel for schedule(static)
  for (i64 kap = 0; kap < l.N; ++kap) {
    i64 rem = kap;
    std::vector<i64> k(l.r);
    for (int i = l.r - 1; i >= 0; --i) {
      k[i] = rem % l.n[i];
      rem /= l.n[i];
    }
    for (int j = 0; j < l.d; ++j) {
      __int128 acc = 0;
      for (int i = 0; i < l.r; ++i) acc += (__int128)(l.L / l.n[i]) * l.Z[i][j] * k[i];
      out[kap * l.d + j] = modp(acc, l.L);
    }
  }
  return out;
}

i64 flat_residue(const Lat& l, const i64* h) {
  i64 chi = 0;
  for (int i = 0; i < l.r; ++i) {
    __int128 dot = 0;
    for (int j = 0; j < l.d; ++j) dot += (__int128)l.Z[i][j] * h[j];
    i64 w = 1;
    for (int t = i + 1; t < l.r; ++t) w *= l.n[t];
    chi += modp(dot, l.n[i]) * w;
  }
  return chi;
}

// ------------------------------------------------------- solver state
struct Oracle {
  Lat lat;
  std::vector<i64> pts;
  std::vector<double> v;
  std::vector<std::uint32_t> norm2;
  double eps = 1, dt = 0;
  std::vector<cd> kin, potH;
  std::vector<Dft*> dfts;  // one per axis

  ~Oracle() {
    for (auto* p : dfts) delete p;
  }

  // r-dim transform over the n1 x ... x nr tensor, axis by axis
  void transform(std::vector<cd>& x, int sign) const {
    const int r = lat.r;
    for (int ax = 0; ax < r; ++ax) {
      const i64 len = lat.n[ax];
      i64 inner = 1, outer = 1;
      for (int t = ax + 1; t < r; ++t) inner *= lat.n[t];
      for (int t = 0; t < ax; ++t) outer *= lat.n[t];
      if (len == 1) continue;
      const i64 lines = inner * outer;
      if (lines == 1) {
        std::vector<cd> y(len);
        dfts[ax]->run(x.data(), y.data(), sign);
        x.swap(y);
        continue;
      }
#pragma omp parallel for schedule(static)
      for (i64 line = 0; line < lines; ++line) {
        const i64 o = line / inner, in = line % inner;
        std::vector<cd> a(len), b(len);
        for (i64 t = 0; t < len; ++t) a[t] = x[(o * len + t) * inner + in];
        dfts[ax]->run(a.data(), b.data(), sign);
        for (i64 t = 0; t < len; ++t) x[(o * len + t) * inner + in] = b[t];
      }
    }
  }
  void analyze(std::vector<cd>& x) const {
    transform(x, -1);
    const double inv = 1.0 / (double)lat.N;
    for (auto& c : x) c *= inv;
  }
  void synthesize(std::vector<cd>& x) const { transform(x, +1); }

  void set_dt(double dt_) {
    dt = dt_;
    kin.resize(lat.N);
    potH.resize(lat.N);
    for (i64 c = 0; c < lat.N; ++c) {
      const double a = -eps * dt * 2.0 * M_PI * M_PI * (double)norm2[c];
      kin[c] = std::polar(1.0, a);
    }
    for (i64 k = 0; k < lat.N; ++k) potH[k] = std::polar(1.0, -dt * v[k] / (2.0 * eps));
  }

  void strang_step(std::vector<cd>& uhat) const {
    std::vector<cd>& u = uhat;
    synthesize(u);
    for (i64 k = 0; k < lat.N; ++k) u[k] *= potH[k];
    analyze(u);
    for (i64 c = 0; c < lat.N; ++c) u[c] *= kin[c];
    synthesize(u);
    for (i64 k = 0; k < lat.N; ++k) u[k] *= potH[k];
    analyze(u);
  }
};

double v_eval(const double* a, const double* b, int d, const i64* num, i64 L) {
  double acc = 0;
  for (int j = 0; j < d; ++j) acc += a[j] * (1.0 - std::cos(2.0 * M_PI * (double)num[j] / (double)L));
  for (int j = 0; j + 1 < d; ++j) {
    i64 dn = modp((__int128)num[j] - num[j + 1], L);
    acc += b[j] * std::cos(2.0 * M_PI * (double)dn / (double)L);
  }
  return acc;
}

cd g_eval(const double* c, const int* p, double sigma, int d, const i64* num, i64 L) {
  double ex = 0;
  __int128 ph = 0;
  for (int j = 0; j < d; ++j) {
    const double x = (double)num[j] / (double)L;
    const double s = std::sin(M_PI * (x - c[j]));
    ex -= s * s / (2.0 * sigma * sigma);
    ph += (__int128)p[j] * num[j];
  }
  const i64 q = modp(ph, L);
  return std::exp(ex) * std::polar(1.0, 2.0 * M_PI * (double)q / (double)L);
}

// omega(j/n) = 2 pi^2 B2(j/n) from the exact numerator 6 j (j - n) + n^2
std::vector<double> omega_table(i64 n) {
  std::vector<double> om(n);
  const long double pi2 = PI_L * PI_L;
  for (i64 j = 0; j < n; ++j) {
    __int128 num = 6 * (__int128)j * (j - n) + (__int128)n * n;
    om[j] = (double)((long double)num * (pi2 / (3.0L * (long double)n * (long double)n)));
  }
  return om;
}

}  // namespace

extern "C" {

// ---- FFT (validated against numpy / naive DFT in tests)
void orc_dft(const double* in, double* out, i64 n, int sign) {
  Dft f(n);
  f.run(reinterpret_cast<const cd*>(in), reinterpret_cast<cd*>(out), sign);
}

// ---- points (row-major N x d numerators)
void orc_points(int d, int r, const i64* Z, const i64* n, i64* out) {
  Lat l = make_lat(d, r, Z, n);
  auto p = points(l);
  std::memcpy(out, p.data(), p.size() * sizeof(i64));
}

// ---- exhaustive CBC (SPEC.md:128-137 with candidates gcd(c,n)=1 and the
// documented tie tolerance); returns criterion per component
void orc_cbc_exhaustive(i64 n, int d, i64* z, double* wce) {
  const auto om = omega_table(n);
  std::vector<double> P(n, 1.0);
  auto score = [&](i64 c) {
    long double acc = 0;
    i64 r = 0;
    for (i64 k = 0; k < n; ++k) {
      acc += (long double)P[k] * (1.0L + (long double)om[r]);
      r += c;
      if (r >= n) r -= n;
    }
    return (double)(acc / (long double)n - 1.0L);
  };
  auto apply = [&](i64 c) {
    i64 r = 0;
    for (i64 k = 0; k < n; ++k) {
      P[k] = P[k] * (1.0 + om[r]);
      r += c;
      if (r >= n) r -= n;
    }
  };
  z[0] = 1;
  wce[0] = score(1);
  apply(1);
  for (int s = 1; s < d; ++s) {
    std::vector<double> sc(n, INFINITY);
#pragma omp parallel for schedule(dynamic, 16)
    for (i64 c = 1; c < n; ++c)
      if (std::gcd(c, n) == 1) sc[c] = score(c);
    double best = INFINITY;
    for (i64 c = 1; c < n; ++c) best = std::min(best, sc[c]);
    i64 win = -1;
    for (i64 c = 1; c < n && win < 0; ++c)
      if (sc[c] <= best + 1e-13 * std::fabs(best)) win = c;
    z[s] = win;
    wce[s] = sc[win];
    apply(win);
  }
}

// ---- literal shell walk: returns 0 or -1 if the cap is hit
int orc_aaset(int d, int r, const i64* Z, const i64* n, double cap, std::uint32_t* norm2, std::int16_t* h) {
  Lat l = make_lat(d, r, Z, n);
  if (cap <= 0) cap = 4.0 * std::pow((double)l.N, 1.0 / d) + 16.0;
  const i64 cap2 = (i64)std::floor(cap * cap);
  std::vector<char> seen(l.N, 0);
  i64 filled = 0;
  std::vector<i64> hv(d);
  // enumerate vectors of squared norm exactly s in lexicographic order
  struct Walk {
    const Lat& l;
    std::vector<i64>& hv;
    std::vector<char>& seen;
    i64& filled;
    std::uint32_t* norm2;
    std::int16_t* h;
    i64 s;
    void go(int j, i64 rem) {
      const int d = l.d;
      if (j == d - 1) {
        i64 x = (i64)std::llround(std::sqrt((double)rem));
        if (x * x != rem) return;
        for (i64 v : (x == 0 ? std::vector<i64>{0} : std::vector<i64>{-x, x})) {
          hv[j] = v;
          i64 chi = flat_residue(l, hv.data());
          if (!seen[chi]) {
            seen[chi] = 1;
            ++filled;
            norm2[chi] = (std::uint32_t)s;
            if (h)
              for (int t = 0; t < d; ++t) h[chi * d + t] = (std::int16_t)hv[t];
          }
        }
        return;
      }
      i64 m = (i64)std::floor(std::sqrt((double)rem));
      while ((m + 1) * (m + 1) <= rem) ++m;
      while (m * m > rem) --m;
      for (i64 x = -m; x <= m; ++x) {
        hv[j] = x;
        go(j + 1, rem - x * x);
      }
    }
  };
  for (i64 s = 0; filled < l.N; ++s) {
    if (s > cap2) return -1;
    Walk w{l, hv, seen, filled, norm2, h, s};
    w.go(0, s);
  }
  return 0;
}

// ---- solver
void* orc_create(int d, int r, const i64* Z, const i64* n, const std::uint32_t* norm2, double eps, const double* a,
                 const double* b) {
  auto* o = new Oracle;
  o->lat = make_lat(d, r, Z, n);
  o->pts = points(o->lat);
  o->eps = eps;
  o->norm2.assign(norm2, norm2 + o->lat.N);
  o->v.resize(o->lat.N);
  for (i64 k = 0; k < o->lat.N; ++k) o->v[k] = v_eval(a, b, d, o->pts.data() + k * d, o->lat.L);
  for (int ax = 0; ax < r; ++ax) o->dfts.push_back(new Dft(o->lat.n[ax]));
  return o;
}
void orc_destroy(void* h) { delete static_cast<Oracle*>(h); }
void orc_set_dt(void* h, double dt) { static_cast<Oracle*>(h)->set_dt(dt); }
void orc_potential(void* h, double* out) {
  auto* o = static_cast<Oracle*>(h);
  std::copy(o->v.begin(), o->v.end(), out);
}

// g samples normalised so (1/N) sum |g|^2 = 1; returns the constant C
double orc_initial_samples(void* h, const double* c, const int* p, double sigma, double* out) {
  auto* o = static_cast<Oracle*>(h);
  cd* u = reinterpret_cast<cd*>(out);
  const int d = o->lat.d;
  long double s = 0;
  for (i64 k = 0; k < o->lat.N; ++k) {
    u[k] = g_eval(c, p, sigma, d, o->pts.data() + k * d, o->lat.L);
    s += std::norm(u[k]);
  }
  const double C = (double)(1.0L / sqrtl(s / (long double)o->lat.N));
  for (i64 k = 0; k < o->lat.N; ++k) u[k] *= C;
  return C;
}

void orc_analyze(void* h, double* x) {
  auto* o = static_cast<Oracle*>(h);
  std::vector<cd> v(reinterpret_cast<cd*>(x), reinterpret_cast<cd*>(x) + o->lat.N);
  o->analyze(v);
  std::memcpy(x, v.data(), v.size() * sizeof(cd));
}
void orc_synthesize(void* h, double* x) {
  auto* o = static_cast<Oracle*>(h);
  std::vector<cd> v(reinterpret_cast<cd*>(x), reinterpret_cast<cd*>(x) + o->lat.N);
  o->synthesize(v);
  std::memcpy(x, v.data(), v.size() * sizeof(cd));
}
// nsteps literal Strang steps on coefficients (in place)
void orc_steps(void* h, double* uhat, i64 nsteps) {
  auto* o = static_cast<Oracle*>(h);
  std::vector<cd> v(reinterpret_cast<cd*>(uhat), reinterpret_cast<cd*>(uhat) + o->lat.N);
  for (i64 s = 0; s < nsteps; ++s) o->strang_step(v);
  std::memcpy(uhat, v.data(), v.size() * sizeof(cd));
}
double orc_l2_norm(void* h, const double* uhat) {
  auto* o = static_cast<Oracle*>(h);
  const cd* u = reinterpret_cast<const cd*>(uhat);
  long double s = 0;
  for (i64 c = 0; c < o->lat.N; ++c) s += std::norm(u[c]);
  return (double)sqrtl(s);
}
double orc_energy(void* h, const double* uhat) {
  auto* o = static_cast<Oracle*>(h);
  const cd* u = reinterpret_cast<const cd*>(uhat);
  long double kin = 0, pot = 0;
  for (i64 c = 0; c < o->lat.N; ++c) kin += (long double)(0.5 * o->eps * 4.0 * M_PI * M_PI * o->norm2[c]) * std::norm(u[c]);
  std::vector<cd> s(u, u + o->lat.N);
  o->synthesize(s);
  for (i64 k = 0; k < o->lat.N; ++k) pot += (long double)o->v[k] * std::norm(s[k]);
  return (double)(kin + pot / ((long double)o->eps * (long double)o->lat.N));
}

}  // extern "C"
