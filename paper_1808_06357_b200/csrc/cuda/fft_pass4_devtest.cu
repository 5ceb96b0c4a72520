// pass4 vs v1 on one pass launch at config-3-like shapes: same PassArgs,
// results compared, both timed over a batch that streams from HBM.
//   fft_pass4_devtest            correctness + timing of the built-in cases
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "fft_pass4.cuh"
#include "pass_instantiate.cuh"

using namespace lattdse_dev;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); std::exit(2); } } while (0)

static double2 root(long long t, long long n) {
  long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)(t % n) / (long double)n;
  return make_double2((double)cosl(a), (double)sinl(a));
}

// AXIS, L: the pass; B4/LPT/NT4/MB4: pass4 launch geometry; other = the other factor of the view
template <int AXIS, int L, int B4, int LPT, int NT4, int MB4, bool TW, bool PP = (2 * B4 * L * 16 <= 72 * 1024)>
int run(int other, int batch, int pf, bool lut = false) {
  using G1 = lattdse::dev::Geometry<AXIS, L>;
  const long long nrows = AXIS == AX_COL ? L : other, ncols = AXIS == AX_COL ? other : L;
  const long long M = nrows * ncols;
  const long long nmid = AXIS == AX_COL ? M / 2 + 3 : M;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1, 1);
  std::vector<double2> x((size_t)M * batch), diag(M);
  for (auto& v : x) v = make_double2(u(rng), u(rng));
  for (auto& v : diag) v = make_double2(u(rng), u(rng));
  std::vector<double2> fft_tw(std::max(1, plan_twiddles<L>(nullptr))), fft_tw2(std::max(1, plan_twiddles<L>(nullptr, true)));
  plan_twiddles<L>(fft_tw.data());
  plan_twiddles<L>(fft_tw2.data(), true);
  int shift = 0;
  while ((1LL << (2 * shift)) < M) ++shift;
  long long nlo = 1LL << shift, nhi = (M + nlo - 1) / nlo;
  std::vector<double2> lo(nlo), hi(nhi);
  for (long long t = 0; t < nlo; ++t) lo[t] = root(t, M);
  for (long long t = 0; t < nhi; ++t) hi[t] = root(t * nlo, M);
  std::vector<unsigned short> idx(M);
  std::vector<double2> lutv(256);
  for (auto& v : idx) v = (unsigned short)(rng() % 256);
  for (auto& v : lutv) v = make_double2(u(rng), u(rng));
  double2 *d0, *d1, *dd, *dtw, *dtw2, *dlo, *dhi, *dlut;
  unsigned short* didx;
  CK(cudaMalloc(&d0, x.size() * 16)); CK(cudaMalloc(&d1, x.size() * 16)); CK(cudaMalloc(&dd, M * 16));
  CK(cudaMalloc(&dtw, fft_tw.size() * 16)); CK(cudaMalloc(&dtw2, fft_tw2.size() * 16));
  CK(cudaMalloc(&dlo, nlo * 16)); CK(cudaMalloc(&dhi, nhi * 16)); CK(cudaMalloc(&dlut, 256 * 16)); CK(cudaMalloc(&didx, M * 2));
  CK(cudaMemcpy(d0, x.data(), x.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d1, x.data(), x.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dd, diag.data(), M * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtw, fft_tw.data(), fft_tw.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtw2, fft_tw2.data(), fft_tw2.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dlo, lo.data(), nlo * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dhi, hi.data(), nhi * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dlut, lutv.data(), 256 * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(didx, idx.data(), M * 2, cudaMemcpyHostToDevice));
  PassArgs a{};
  a.in = d0; a.out = d0; a.in_bstride = a.out_bstride = M;
  a.nvalid_in = a.nvalid_out = M; a.nvalid_mid = nmid;
  a.ncols = (int)ncols;
  const long long nlines = AXIS == AX_ROW ? nrows : ncols;
  a.nlines = (int)nlines;
  if (lut) { a.diag_kind = DG_LUT16; a.diag_idx = didx; a.lut = dlut; } else { a.diag_kind = DG_CPLX; a.diag = dd; }
  a.pre_tw = a.post_tw = TW ? 1 : 0; a.tw_shift = shift; a.tw_lo = dlo; a.tw_hi = dhi; a.fft_tw = dtw; a.fft_tw2 = dtw2;
  a.mid_rb = (int)(nmid / ncols); a.mid_cb = (int)(nmid % ncols); a.pf = pf;
  constexpr int SIGN = AXIS == AX_ROW ? -1 : 1;
  constexpr int mb1 = G1::wide_col ? 1 : (G1::NT > 320 ? 2 : (AXIS == AX_ROW && L < 4096 ? 3 : 2));
  auto f1 = fft_pass_kernel<AXIS, L, G1::B, G1::NT, PROG_DOUBLE, SIGN, mb1>;
  const int sm1 = SmemGeom<L, G1::B>::bytes;
  CK(cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1));
  const dim3 g1((unsigned)((nlines + G1::B - 1) / G1::B), batch);
  const int sm4 = P4Geom<AXIS, L, B4, LPT, PP>::bytes;
  const dim3 g4((unsigned)(nlines / B4), batch);
  auto launch4 = [&](const PassArgs& p) {
    if (lut) {
      auto f4 = fft_pass4_kernel<AXIS, L, B4, LPT, PP, NT4, SIGN, TW, DG_LUT16, MB4>;
      CK(cudaFuncSetAttribute(f4, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
      f4<<<g4, NT4, sm4>>>(p);
    } else {
      auto f4 = fft_pass4_kernel<AXIS, L, B4, LPT, PP, NT4, SIGN, TW, DG_CPLX, MB4>;
      CK(cudaFuncSetAttribute(f4, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
      f4<<<g4, NT4, sm4>>>(p);
    }
  };
  PassArgs p = a;
  p.in = p.out = d1;
  f1<<<g1, G1::NT, sm1>>>(a);
  CK(cudaGetLastError());
  launch4(p);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<double2> r0(x.size()), r1(x.size());
  CK(cudaMemcpy(r0.data(), d0, x.size() * 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(r1.data(), d1, x.size() * 16, cudaMemcpyDeviceToHost));
  double e = 0, mx = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    e = std::max(e, std::abs(r0[i].x - r1[i].x) + std::abs(r0[i].y - r1[i].y));
    mx = std::max(mx, std::abs(r0[i].x) + std::abs(r0[i].y));
  }
  const bool ok = e / mx < 1e-13;
  std::printf("axis=%d L=%d other=%d batch=%d B4=%d LPT=%d NT4=%d mb=%d lut=%d: max|p4-v1|/max = %.3e %s\n", AXIS, L, other, batch, B4,
              LPT, NT4, MB4, (int)lut, e / mx, ok ? "ok" : "MISMATCH");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 20;
  float ms = 0;
  for (int w = 0; w < 2; ++w) f1<<<g1, G1::NT, sm1>>>(a);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) f1<<<g1, G1::NT, sm1>>>(a);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  const double gb = 32.0 * M * batch / 1e9;
  std::printf("  TIME v1    B=%d NT=%d: %8.1f us  (%.0f GB/s)\n", G1::B, G1::NT, 1e3 * ms / reps, gb / (ms / reps * 1e-3));
  for (int w = 0; w < 2; ++w) launch4(p);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch4(p);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  std::printf("  TIME pass4 L=%d B=%d LPT=%d pp=%d NT=%d mb=%d pf=%d smem=%d: %8.1f us  (%.0f GB/s)\n", L, B4, LPT, (int)PP, NT4, MB4, pf, sm4, 1e3 * ms / reps,
              gb / (ms / reps * 1e-3));
  cudaFree(d0); cudaFree(d1); cudaFree(dd); cudaFree(dtw); cudaFree(dtw2); cudaFree(dlo); cudaFree(dhi); cudaFree(dlut); cudaFree(didx);
  return ok ? 0 : 1;
}

#ifndef P4_CASES
#define P4_CASES                                                        \
  CASE((run<AX_COL, 486, 4, 1, 352, 2, true>(1080, batch, 0)))          \
  CASE((run<AX_ROW, 1080, 1, 1, 160, 3, false>(486, batch, 0)))         \
  CASE((run<AX_COL, 486, 4, 1, 352, 3, true>(1080, batch, 0)))          \
  CASE((run<AX_ROW, 1080, 1, 1, 160, 4, false>(486, batch, 0)))         \
  CASE((run<AX_COL, 486, 4, 1, 352, 2, false>(1080, 8, 0, true)))
#endif

int main(int argc, char** argv) {
  const int batch = argc > 1 ? std::atoi(argv[1]) : 64;
  const int only = argc > 2 ? std::atoi(argv[2]) : -1;
  int bad = 0, idx = 0;
#define CASE(x) if (only < 0 || only == idx) bad += x; ++idx;
  P4_CASES
  std::printf(bad ? "FAILED %d\n" : "all ok\n", bad);
  return bad;
}
