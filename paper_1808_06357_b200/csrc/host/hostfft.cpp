#include "hostfft.hpp"

#include <cmath>
#include <stdexcept>

namespace lattdse::hostfft {

namespace {

const long double kPiL = 3.141592653589793238462643383279502884L;

cd root(std::int64_t t, std::int64_t n, int sign) {
  long double a = 2.0L * kPiL * static_cast<long double>(t % n) / static_cast<long double>(n);
  return cd(static_cast<double>(cosl(a)), static_cast<double>(sign * sinl(a)));
}

bool smooth5(std::int64_t n) {
  for (int p : {2, 3, 5})
    while (n % p == 0) n /= p;
  return n == 1;
}

// Stockham autosort, radices 4/2/3/5, n 5-smooth. Out-of-place ping-pong.
void stockham(std::vector<cd>& x, int sign) {
  const std::int64_t n = static_cast<std::int64_t>(x.size());
  if (n <= 1) return;
  std::vector<int> radices;
  for (std::int64_t m = n; m > 1;) {
    int r = (m % 4 == 0) ? 4 : (m % 2 == 0 ? 2 : (m % 3 == 0 ? 3 : 5));
    radices.push_back(r);
    m /= r;
  }
  std::vector<cd> tw(n);
  for (std::int64_t t = 0; t < n; ++t) tw[t] = root(t, n, sign);
  std::vector<cd> y(n);
  cd* in = x.data();
  cd* out = y.data();
  std::int64_t ns = 1;
  const cd w3 = root(1, 3, sign), w5a = root(1, 5, sign), w5b = root(2, 5, sign);
  for (int r : radices) {
    const std::int64_t T = n / r, step = n / (ns * r);
#pragma omp parallel for schedule(static) if (n > (1 << 15))
    for (std::int64_t j = 0; j < T; ++j) {
      cd v[5];
      const std::int64_t k = j % ns;
      for (int q = 0; q < r; ++q) v[q] = in[j + q * T];
      for (int q = 1; q < r; ++q) v[q] *= tw[(q * k * step) % n];
      cd o[5];
      if (r == 2) {
        o[0] = v[0] + v[1];
        o[1] = v[0] - v[1];
      } else if (r == 4) {
        cd a = v[0] + v[2], b = v[0] - v[2], c = v[1] + v[3];
        cd d = (v[1] - v[3]) * cd(0, sign);
        o[0] = a + c; o[2] = a - c; o[1] = b + d; o[3] = b - d;
      } else if (r == 3) {
        o[0] = v[0] + v[1] + v[2];
        o[1] = v[0] + w3 * v[1] + w3 * w3 * v[2];
        o[2] = v[0] + w3 * w3 * v[1] + w3 * v[2];
      } else {
        cd w[5] = {1.0, w5a, w5b, std::conj(w5b), std::conj(w5a)};
        for (int a = 0; a < 5; ++a) {
          cd s = 0;
          for (int b = 0; b < 5; ++b) s += v[b] * w[(a * b) % 5];
          o[a] = s;
        }
      }
      const std::int64_t base = (j / ns) * ns * r + k;
      for (int q = 0; q < r; ++q) out[base + q * ns] = o[q];
    }
    std::swap(in, out);
    ns *= r;
  }
  if (in != x.data()) std::copy(in, in + n, x.data());
}

}  // namespace

std::int64_t next_smooth(std::int64_t n) {
  if (n < 1) return 1;
  while (!smooth5(n)) ++n;
  return n;
}

void dft(std::vector<cd>& x, int sign) {
  const std::int64_t n = static_cast<std::int64_t>(x.size());
  if (n <= 1) return;
  if (smooth5(n)) {
    stockham(x, sign);
    return;
  }
  // Bluestein: jk = (j^2 + k^2 - (k-j)^2)/2, chirp c_j = exp(sign*pi*i*j^2/n),
  // j^2 reduced mod 2n exactly.
  const std::int64_t m = next_smooth(2 * n - 1);
  std::vector<cd> chirp(n);
  for (std::int64_t j = 0; j < n; ++j) {
    const std::int64_t q = static_cast<std::int64_t>((static_cast<__int128>(j) * j) % (2 * n));
    long double a = kPiL * static_cast<long double>(q) / static_cast<long double>(n);
    chirp[j] = cd(static_cast<double>(cosl(a)), static_cast<double>(sign * sinl(a)));
  }
  std::vector<cd> a(m, 0.0), b(m, 0.0);
  for (std::int64_t j = 0; j < n; ++j) a[j] = x[j] * chirp[j];
  b[0] = std::conj(chirp[0]);
  for (std::int64_t j = 1; j < n; ++j) b[j] = b[m - j] = std::conj(chirp[j]);
  stockham(a, -1);
  stockham(b, -1);
  for (std::int64_t t = 0; t < m; ++t) a[t] *= b[t];
  stockham(a, +1);
  const double inv = 1.0 / static_cast<double>(m);
  for (std::int64_t k = 0; k < n; ++k) x[k] = a[k] * chirp[k] * inv;
}

}  // namespace lattdse::hostfft
