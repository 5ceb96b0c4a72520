// Device-vs-emulation check of single pass launches at production sizes:
// the same PassArgs are executed by the sm_100a kernel and by the host
// emulation (HostExec); results must agree to rounding.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "fft_pass.cuh"
#include "pass_instantiate.cuh"
#include "cluster_col.inl"

using namespace lattdse_dev;

struct HostExec {
  template <class St, class C> static void stage(const C& c) {
    using Regs = double2[St::TPT][St::R];
    std::vector<std::vector<double2>> regs(St::nt, std::vector<double2>(St::TPT * St::R));
    for (int tid = 0; tid < St::nt; ++tid) St::read(c, tid, *reinterpret_cast<Regs*>(regs[tid].data()));
    for (int tid = 0; tid < St::nt; ++tid) St::write(c, tid, *reinterpret_cast<Regs*>(regs[tid].data()));
  }
};

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); return 2; } } while (0)

static double2 root(long long t, long long n) {
  long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)(t % n) / (long double)n;
  return make_double2((double)cosl(a), (double)sinl(a));
}

template <int AXIS, int L, int B, int NT, int PROG, int SIGN, int MINB = 1>
int run(long long nrows, long long ncols, int post_tw, int pre_tw, long long nin = -1, bool timing = false) {
  const long long M = nrows * ncols;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1, 1);
  const long long NI = nin > 0 ? nin : M;
  std::vector<double2> x(M), diag(NI), xin(NI);
  for (auto& v : x) v = make_double2(u(rng), u(rng));
  for (auto& v : diag) v = make_double2(u(rng), u(rng));
  for (auto& v : xin) v = make_double2(u(rng), u(rng));
  std::vector<double2> fft_tw(std::max(1, plan_twiddles<L>(nullptr)));
  plan_twiddles<L>(fft_tw.data());
  std::vector<double2> fft_tw2(std::max(1, plan_twiddles<L>(nullptr, true)));
  plan_twiddles<L>(fft_tw2.data(), true);
  int shift = 0;
  while ((1LL << (2 * shift)) < M) ++shift;
  long long nlo = 1LL << shift, nhi = (M + nlo - 1) / nlo;
  std::vector<double2> lo(nlo), hi(nhi);
  for (long long t = 0; t < nlo; ++t) lo[t] = root(t, M);
  for (long long t = 0; t < nhi; ++t) hi[t] = root(t * nlo, M);
  double2 *dx, *dd, *dtw, *dtw2, *dlo, *dhi, *din;
  CK(cudaMalloc(&dx, M * 16)); CK(cudaMalloc(&dd, NI * 16)); CK(cudaMalloc(&din, NI * 16));
  CK(cudaMemcpy(din, xin.data(), NI * 16, cudaMemcpyHostToDevice)); CK(cudaMalloc(&dtw, fft_tw.size() * 16)); CK(cudaMalloc(&dtw2, fft_tw2.size() * 16));
  CK(cudaMalloc(&dlo, nlo * 16)); CK(cudaMalloc(&dhi, nhi * 16));
  CK(cudaMemcpy(dx, x.data(), M * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dd, diag.data(), NI * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtw, fft_tw.data(), fft_tw.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtw2, fft_tw2.data(), fft_tw2.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dlo, lo.data(), nlo * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dhi, hi.data(), nhi * 16, cudaMemcpyHostToDevice));
  PassArgs a{};
  a.in = nin > 0 ? din : dx; a.out = dx; a.in_bstride = NI; a.out_bstride = M;
  a.nvalid_in = NI; a.nvalid_out = M; a.nvalid_mid = M / 2;
  a.ncols = (int)ncols;
  const long long nlines = AXIS == AX_ROW ? nrows : ncols;
  a.nlines = (int)nlines;
  a.diag_kind = DG_CPLX; a.diag = dd;
  a.pre_tw = pre_tw; a.post_tw = post_tw; a.tw_shift = shift; a.tw_lo = dlo; a.tw_hi = dhi; a.fft_tw = dtw; a.fft_tw2 = dtw2;
  const int smem = SmemGeom<L, B>::bytes;
  auto fn = fft_pass_kernel<AXIS, L, B, NT, PROG, SIGN, MINB>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  fn<<<dim3((unsigned)((nlines + B - 1) / B), 1), NT, smem>>>(a);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  if (timing) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 50;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) fn<<<dim3((unsigned)((nlines + B - 1) / B), 1), NT, smem>>>(a);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("TIME axis=%d L=%d B=%d NT=%d prog=%d minb=%d ablate=%d: %.2f us/launch\n", AXIS, L, B, NT, PROG, MINB,
                LATTDSE_ABLATE, 1e3 * ms / reps);
    cudaFree(din); cudaFree(dx); cudaFree(dd); cudaFree(dtw); cudaFree(dlo); cudaFree(dhi);
    return 0;
  }
  std::vector<double2> got(M);
  CK(cudaMemcpy(got.data(), dx, M * 16, cudaMemcpyDeviceToHost));
  // host emulation on host copies
  PassArgs h = a;
  std::vector<double2> hx = x;
  h.in = nin > 0 ? xin.data() : hx.data(); h.out = hx.data(); h.diag = diag.data(); h.fft_tw = fft_tw.data(); h.fft_tw2 = fft_tw2.data(); h.tw_lo = lo.data(); h.tw_hi = hi.data();
  std::vector<double2> sm(SmemGeom<L, B>::bytes / 16);
  for (long long blk = 0; blk < (nlines + B - 1) / B; ++blk) {
    Ctx<AXIS, L, B, PROG> c{sm.data(), h, (int)(blk * B), 0};
    run_pass<HostExec, AXIS, L, B, NT, PROG, SIGN>(c);
  }
  double e = 0, mx = 0;
  for (long long i = 0; i < M; ++i) {
    e = std::max(e, std::abs(got[i].x - hx[i].x) + std::abs(got[i].y - hx[i].y));
    mx = std::max(mx, std::abs(hx[i].x) + std::abs(hx[i].y));
  }
  std::printf("axis=%d L=%d B=%d NT=%d prog=%d sign=%+d %lldx%lld: max|dev-emu|/max = %.3e %s\n", AXIS, L, B, NT,
              PROG, SIGN, nrows, ncols, e / mx, e / mx < 1e-13 ? "ok" : "MISMATCH");
  cudaFree(din); cudaFree(dx); cudaFree(dd); cudaFree(dtw); cudaFree(dlo); cudaFree(dhi);
  return e / mx < 1e-13 ? 0 : 1;
}

// production launch geometry of (AXIS, L) (pass_instantiate.cuh), PROG_DOUBLE
template <int AXIS, int L> int time_prod(long long nrows, long long ncols, int tw) {
  using G = lattdse::dev::Geometry<AXIS, L>;
  constexpr int mb = G::wide_col ? 1 : (G::NT > 320 ? 2 : (AXIS == AX_ROW && L < 4096 ? 3 : 2));
  return run<AXIS, L, G::B, G::NT, PROG_DOUBLE, AXIS == AX_ROW ? -1 : 1, mb>(nrows, ncols, tw, tw, -1, true);
}

// cluster COL pass (cluster_col.inl) vs the plain COL pass on an n x ncols
// grid, PROG_DOUBLE with a full complex diagonal; then both timed
template <int LLOC, int C, int B, int NT, int MINB>
int run_cluster(long long ncols, bool timing) {
  constexpr int L = LLOC * C;
  const long long M = (long long)L * ncols;
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<double> u(-1, 1);
  std::vector<double2> x(M), diag(M);
  for (auto& v : x) v = make_double2(u(rng), u(rng));
  for (auto& v : diag) v = make_double2(u(rng), u(rng));
  std::vector<double2> tl(L);
  for (int k = 0; k < L; ++k) tl[k] = root(k, L);
  std::vector<double2> st(std::max(1, plan_twiddles<LLOC>(nullptr)));
  plan_twiddles<LLOC>(st.data());
  std::vector<double2> pt(std::max(1, plan_twiddles<L>(nullptr))), pt2(std::max(1, plan_twiddles<L>(nullptr, true)));
  plan_twiddles<L>(pt.data());
  plan_twiddles<L>(pt2.data(), true);
  double2 *d0, *d1, *dd, *dtl, *dst, *dpt, *dpt2;
  CK(cudaMalloc(&d0, M * 16)); CK(cudaMalloc(&d1, M * 16)); CK(cudaMalloc(&dd, M * 16));
  CK(cudaMalloc(&dtl, L * 16)); CK(cudaMalloc(&dst, st.size() * 16)); CK(cudaMalloc(&dpt, pt.size() * 16)); CK(cudaMalloc(&dpt2, pt2.size() * 16));
  CK(cudaMemcpy(d0, x.data(), M * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d1, x.data(), M * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dd, diag.data(), M * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtl, tl.data(), L * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dst, st.data(), st.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpt, pt.data(), pt.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpt2, pt2.data(), pt2.size() * 16, cudaMemcpyHostToDevice));
  PassArgs a{};
  a.in = d0; a.out = d0; a.in_bstride = a.out_bstride = M;
  a.nvalid_in = a.nvalid_mid = a.nvalid_out = M;
  a.ncols = (int)ncols; a.nlines = (int)ncols;
  a.diag_kind = DG_CPLX; a.diag = dd;
  a.tw_lo = dtl; a.fft_tw = dst;
  auto fc = cluster_col_kernel<LLOC, C, B, NT, -1, MINB>;
  const int smc = ClusterGeom<LLOC, C, B>::bytes;
  CK(cudaFuncSetAttribute(fc, cudaFuncAttributeMaxDynamicSharedMemorySize, smc));
  const dim3 gc((unsigned)(C * (ncols / B)), 1);
  PassArgs p = a;
  p.in = p.out = d1; p.fft_tw = dpt; p.fft_tw2 = dpt2; p.tw_lo = nullptr;
  using G = lattdse::dev::Geometry<AX_COL, L>;
  auto fp = fft_pass_kernel<AX_COL, L, G::B, G::NT, PROG_DOUBLE, -1, 1>;
  const int smp = SmemGeom<L, G::B>::bytes;
  CK(cudaFuncSetAttribute(fp, cudaFuncAttributeMaxDynamicSharedMemorySize, smp));
  const dim3 gp((unsigned)((ncols + G::B - 1) / G::B), 1);
  fc<<<gc, NT, smc>>>(a);
  CK(cudaGetLastError());
  fp<<<gp, G::NT, smp>>>(p);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<double2> g0(M), g1(M);
  CK(cudaMemcpy(g0.data(), d0, M * 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(g1.data(), d1, M * 16, cudaMemcpyDeviceToHost));
  double e = 0, mx = 0;
  for (long long i = 0; i < M; ++i) {
    e = std::max(e, std::abs(g0[i].x - g1[i].x) + std::abs(g0[i].y - g1[i].y));
    mx = std::max(mx, std::abs(g1[i].x) + std::abs(g1[i].y));
  }
  const bool ok = e / mx < 1e-13;
  std::printf("cluster L=%d (Lloc %d x C %d, B=%d NT=%d minb=%d) %lld cols: max|cluster-plain|/max = %.3e %s\n", L, LLOC, C, B,
              NT, MINB, ncols, e / mx, ok ? "ok" : "MISMATCH");
  if (timing) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 20;
    float ms = 0;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) fc<<<gc, NT, smc>>>(a);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("TIME cluster L=%d Lloc=%d C=%d B=%d minb=%d: %.2f us/launch\n", L, LLOC, C, B, MINB, 1e3 * ms / reps);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) fp<<<gp, G::NT, smp>>>(p);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("TIME plain   L=%d B=%d NT=%d: %.2f us/launch\n", L, G::B, G::NT, 1e3 * ms / reps);
  }
  cudaFree(d0); cudaFree(d1); cudaFree(dd); cudaFree(dtl); cudaFree(dst); cudaFree(dpt); cudaFree(dpt2);
  return ok ? 0 : 1;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "cluster") {
    int bad = 0;
    bad |= run_cluster<512, 8, 8, 256, 2>(64, false);
    bad |= run_cluster<1024, 4, 4, 256, 2>(64, false);
    bad |= run_cluster<512, 8, 8, 256, 2>(4096, true);
    bad |= run_cluster<512, 8, 8, 256, 3>(4096, true);
    bad |= run_cluster<1024, 4, 4, 256, 2>(4096, true);
    bad |= run_cluster<1024, 4, 4, 256, 3>(4096, true);
    std::printf(bad ? "SOME FAILED\n" : "ALL OK\n");
    return bad;
  }
  int bad = 0;
  if (argc > 1 && std::string(argv[1]) == "time") {
    // config-1 production geometry (1296 x 1620)
    run<AX_ROW, 1620, 1, 192, PROG_DOUBLE, -1, 3>(1296, 1620, 0, 0, -1, true);
    run<AX_COL, 1296, 2, 288, PROG_DOUBLE, 1, 2>(1296, 1620, 1, 1, -1, true);
    run<AX_COL, 1296, 2, 288, PROG_DOUBLE, 1, 2>(1296, 1620, 0, 0, -1, true);  // no four-step twiddles
    if (argc > 2 && std::string(argv[2]) == "pow2") {  // power-of-two views of M = 2^21 (C1-sized)
      time_prod<AX_ROW, 2048>(1024, 2048, 0);
      time_prod<AX_COL, 1024>(1024, 2048, 1);
      time_prod<AX_ROW, 1024>(2048, 1024, 0);
      time_prod<AX_COL, 2048>(2048, 1024, 1);
      time_prod<AX_ROW, 512>(4096, 512, 0);
      time_prod<AX_COL, 4096>(4096, 512, 1);
      time_prod<AX_ROW, 4096>(512, 4096, 0);
      time_prod<AX_COL, 512>(512, 4096, 1);
      time_prod<AX_ROW, 1620>(1296, 1620, 0);
      time_prod<AX_COL, 1296>(1296, 1620, 1);
      // column passes with a padded (non-power-of-two) row pitch
      time_prod<AX_COL, 1024>(1024, 2064, 1);
      time_prod<AX_COL, 1024>(1024, 2056, 1);
      time_prod<AX_COL, 1024>(1024, 2050, 1);
      time_prod<AX_COL, 2048>(2048, 1040, 1);
      time_prod<AX_COL, 1024>(1024, 2064, 0);
      time_prod<AX_COL, 1296>(1296, 1620, 0);
    }
    if (argc > 2 && std::string(argv[2]) == "long") {  // C1's M = 2099520 with short columns, long rows
      time_prod<AX_ROW, 2592>(810, 2592, 0);
      time_prod<AX_COL, 810>(810, 2592, 1);
      time_prod<AX_ROW, 2880>(729, 2880, 0);
      time_prod<AX_COL, 729>(729, 2880, 1);
      time_prod<AX_ROW, 3240>(648, 3240, 0);
      time_prod<AX_COL, 648>(648, 3240, 1);
      time_prod<AX_ROW, 3888>(540, 3888, 0);
      time_prod<AX_COL, 540>(540, 3888, 1);
      time_prod<AX_ROW, 4320>(486, 4320, 0);
      time_prod<AX_COL, 486>(486, 4320, 1);
      time_prod<AX_ROW, 2160>(972, 2160, 0);
      time_prod<AX_COL, 972>(972, 2160, 1);
    }
    if (argc > 2 && std::string(argv[2]) == "longmb") {  // long rows at other register caps
      using namespace lattdse::dev;
      run<AX_ROW, 2592, 1, Geometry<AX_ROW, 2592>::NT, PROG_DOUBLE, -1, 1>(810, 2592, 0, 0, -1, true);
      run<AX_ROW, 2592, 1, Geometry<AX_ROW, 2592>::NT, PROG_DOUBLE, -1, 2>(810, 2592, 0, 0, -1, true);
      run<AX_ROW, 2880, 1, Geometry<AX_ROW, 2880>::NT, PROG_DOUBLE, -1, 1>(729, 2880, 0, 0, -1, true);
      run<AX_ROW, 2880, 1, Geometry<AX_ROW, 2880>::NT, PROG_DOUBLE, -1, 2>(729, 2880, 0, 0, -1, true);
      run<AX_ROW, 3240, 1, Geometry<AX_ROW, 3240>::NT, PROG_DOUBLE, -1, 1>(648, 3240, 0, 0, -1, true);
      run<AX_ROW, 3240, 1, Geometry<AX_ROW, 3240>::NT, PROG_DOUBLE, -1, 2>(648, 3240, 0, 0, -1, true);
      run<AX_ROW, 3888, 1, Geometry<AX_ROW, 3888>::NT, PROG_DOUBLE, -1, 1>(540, 3888, 0, 0, -1, true);
      run<AX_ROW, 4320, 1, Geometry<AX_ROW, 4320>::NT, PROG_DOUBLE, -1, 1>(486, 4320, 0, 0, -1, true);
      run<AX_ROW, 2160, 1, Geometry<AX_ROW, 2160>::NT, PROG_DOUBLE, -1, 2>(972, 2160, 0, 0, -1, true);
      run<AX_ROW, 4096, 1, 256, PROG_DOUBLE, -1, 2>(512, 4096, 0, 0, -1, true);
      run<AX_COL, 486, 4, Geometry<AX_COL, 486>::NT, PROG_DOUBLE, 1, 1>(486, 4320, 1, 1, -1, true);
      run<AX_COL, 486, 4, Geometry<AX_COL, 486>::NT, PROG_DOUBLE, 1, 3>(486, 4320, 1, 1, -1, true);
      run<AX_COL, 512, 4, 256, PROG_DOUBLE, 1, 2>(512, 4096, 1, 1, -1, true);
      run<AX_COL, 512, 4, 256, PROG_DOUBLE, 1, 3>(512, 4096, 1, 1, -1, true);
    }
    if (argc > 2 && std::string(argv[2]) == "colb4") {  // four columns per CTA at C1-compatible geometries
      run<AX_COL, 729, 4, 352, PROG_DOUBLE, 1, 1>(729, 2880, 1, 1, -1, true);
      run<AX_COL, 729, 4, 352, PROG_DOUBLE, 1, 2>(729, 2880, 1, 1, -1, true);
      run<AX_COL, 972, 4, 448, PROG_DOUBLE, 1, 1>(972, 2160, 1, 1, -1, true);
      run<AX_COL, 972, 4, 448, PROG_DOUBLE, 1, 2>(972, 2160, 1, 1, -1, true);
      run<AX_COL, 648, 4, 448, PROG_DOUBLE, 1, 1>(648, 3240, 1, 1, -1, true);
      run<AX_COL, 648, 4, 448, PROG_DOUBLE, 1, 2>(648, 3240, 1, 1, -1, true);
      run<AX_COL, 810, 4, 544, PROG_DOUBLE, 1, 1>(810, 2592, 1, 1, -1, true);
      run<AX_COL, 1296, 4, 576, PROG_DOUBLE, 1, 1>(1296, 1620, 1, 1, -1, true);
      run<AX_COL, 1215, 4, 544, PROG_DOUBLE, 1, 1>(1215, 1728, 1, 1, -1, true);
      run<AX_ROW, 1728, 1, 224, PROG_DOUBLE, -1, 3>(1215, 1728, 0, 0, -1, true);
      run<AX_COL, 1215, 2, 272, PROG_DOUBLE, 1, 2>(1215, 1728, 1, 1, -1, true);
    }
    if (argc > 2 && std::string(argv[2]) == "b8") {  // HBM-streaming short COL passes (config 4 first level): 4 vs 8 columns per CTA
      time_prod<AX_COL, 486>(486, 1 << 20, 1);
      run<AX_COL, 486, 8, 512, PROG_DOUBLE, 1, 1>(486, 1 << 20, 1, 1, -1, true);
      run<AX_COL, 486, 8, 352, PROG_DOUBLE, 1, 1>(486, 1 << 20, 1, 1, -1, true);
      time_prod<AX_COL, 324>(324, 1 << 20, 1);
      run<AX_COL, 324, 8, 512, PROG_DOUBLE, 1, 1>(324, 1 << 20, 1, 1, -1, true);
      time_prod<AX_COL, 432>(432, 1 << 20, 1);
      run<AX_COL, 432, 8, 512, PROG_DOUBLE, 1, 1>(432, 1 << 20, 1, 1, -1, true);
    }
    if (argc > 2 && std::string(argv[2]) == "c2") {  // config-2 column pass variants (4096 x 4096)
      run<AX_COL, 4096, 1, 256, PROG_DOUBLE, -1, 2>(4096, 4096, 0, 0, -1, true);
      run<AX_COL, 4096, 1, 256, PROG_DOUBLE, -1, 1>(4096, 4096, 0, 0, -1, true);
      run<AX_COL, 4096, 2, 512, PROG_DOUBLE, -1, 1>(4096, 4096, 0, 0, -1, true);
      run<AX_COL, 4096, 2, 256, PROG_DOUBLE, -1, 1>(4096, 4096, 0, 0, -1, true);
      run<AX_ROW, 4096, 1, 256, PROG_DOUBLE, 1, 2>(4096, 4096, 0, 0, -1, true);
      run<AX_COL, 64, 8, 128, PROG_DOUBLE, -1, 4>(64, 262144, 0, 0, -1, true);
      run<AX_COL, 64, 16, 256, PROG_DOUBLE, -1, 3>(64, 262144, 0, 0, -1, true);
      run<AX_COL, 64, 8, 128, PROG_LOADDIAG, -1, 4>(64, 262144, 1, 0, -1, true);
    }
    if (argc > 2 && std::string(argv[2]) == "tpt") {  // two tasks per thread (ILP for TLP)
      run<AX_ROW, 1620, 1, 96, PROG_DOUBLE, -1, 4>(1296, 1620, 0, 0, -1, true);
      run<AX_ROW, 1620, 1, 96, PROG_DOUBLE, -1, 5>(1296, 1620, 0, 0, -1, true);
      run<AX_ROW, 1620, 1, 128, PROG_DOUBLE, -1, 4>(1296, 1620, 0, 0, -1, true);
      run<AX_ROW, 1620, 2, 192, PROG_DOUBLE, -1, 2>(1296, 1620, 0, 0, -1, true);
      run<AX_ROW, 1620, 2, 384, PROG_DOUBLE, -1, 1>(1296, 1620, 0, 0, -1, true);
      run<AX_COL, 1296, 2, 160, PROG_DOUBLE, 1, 3>(1296, 1620, 1, 1, -1, true);
      run<AX_COL, 1296, 2, 160, PROG_DOUBLE, 1, 4>(1296, 1620, 1, 1, -1, true);
      run<AX_COL, 1296, 2, 192, PROG_DOUBLE, 1, 3>(1296, 1620, 1, 1, -1, true);
      run<AX_COL, 1296, 4, 288, PROG_DOUBLE, 1, 1>(1296, 1620, 1, 1, -1, true);
      run<AX_COL, 1296, 4, 576, PROG_DOUBLE, 1, 1>(1296, 1620, 1, 1, -1, true);
      run<AX_COL, 1296, 1, 160, PROG_DOUBLE, 1, 4>(1296, 1620, 1, 1, -1, true);
    }
    return 0;
  }
  if (argc > 1) {
    bad |= run<AX_COL, 1215, 2, 256, PROG_LOADDIAG, -1>(1215, 1728, 1, 0, 1048583);
    std::printf(bad ? "SOME FAILED\n" : "ALL OK\n");
    return bad;
  }
  bad |= run<AX_COL, 1215, 2, 256, PROG_LOADDIAG, -1>(1215, 1728, 1, 0);
  bad |= run<AX_COL, 1215, 2, 256, PROG_DOUBLE, 1>(1215, 1728, 1, 1);
  bad |= run<AX_COL, 1215, 2, 256, PROG_STOREDIAG, 1>(1215, 1728, 0, 1);
  bad |= run<AX_ROW, 1728, 1, 224, PROG_DOUBLE, -1>(1215, 1728, 0, 0);
  bad |= run<AX_COL, 720, 4, 256, PROG_DOUBLE, 1>(720, 729, 1, 1);
  bad |= run<AX_ROW, 4096, 1, 256, PROG_DOUBLE, 1>(512, 4096, 0, 0);
  bad |= run<AX_COL, 4096, 2, 256, PROG_DOUBLE, -1>(4096, 64, 0, 0);
  std::printf(bad ? "SOME FAILED\n" : "ALL OK\n");
  return bad;
}
