// Cluster COL pass: one fused PROG_DOUBLE column pass (FFT_L . x D . IFFT_L
// along the strided axis) for long columns, split across the C CTAs of a
// thread-block cluster through distributed shared memory.
//
// Why: a column of L = 4096 complex fp64 values is 64 KB, so the plain pass
// kernel (fft_pass.cuh) can hold only one or two columns per CTA: 16/32-byte
// row segments and one resident CTA per SM (config 2's COL pass was 61% of
// the step). Here a cluster of C CTAs owns B adjacent columns (B*16-byte
// row segments, 128 B at B = 8) and each CTA holds L/C rows of them.
//
// Decimation in frequency with n = Lloc*a + i (a < C the CTA rank, i < Lloc)
// and k = ka + C*kb:
//   X[ka + C kb] = sum_i W_Lloc^(i kb) [ W_L^(i ka) sum_a x[Lloc a + i] W_C^(a ka) ]
// Phase A: CTA r takes rows i in [r Lloc/C, (r+1) Lloc/C) of every block a
//   straight from global memory (coalesced B*16-byte segments), runs the
//   radix-C DFT over a, twiddles by W_L^(i ka) and stores output ka into
//   CTA ka's shared tile (DSMEM store). cluster barrier.
// Phase B: each CTA owns ka = its rank: local FFT_Lloc (Stockham stages of
//   fft_pass.cuh, all in shared memory), x D at frequency k1 = ka + C kb,
//   local IFFT_Lloc. cluster barrier.
// Phase C: the inverse of phase A: CTA r reads z_ka[i] from every CTA
//   (DSMEM load), untwiddles, radix-C inverse DFT, and stores rows Lloc a + i
//   straight to global memory. cluster barrier (peers may still be reading).
// The radix-C butterflies and both exchanges touch every element once; the
// state crosses HBM once per pass as in the plain kernel.
#pragma once

#include <cooperative_groups.h>

#include "fft_pass.cuh"

namespace lattdse_dev {

template <int LLOC, int C, int B> struct ClusterGeom {
  static constexpr int L = LLOC * C;
  static constexpr int SLICE = LLOC / C;   // rows i of each block a per CTA in phases A/C
  static constexpr int TASKS = B * SLICE;  // (b, i) positions per CTA in phases A/C
  static_assert(LLOC % C == 0, "Lloc must be a multiple of the cluster size");
  static constexpr int bytes = SmemGeom<LLOC, B>::tile * 16;
};

#if defined(__CUDACC__)
// a: in/out (in place allowed: every global read precedes the first cluster
// barrier, every global write follows it), in_bstride/out_bstride, ncols,
// diag_kind (DG_LUT16 / DG_CPLX / DG_NONE), diag_idx, lut, diag (indexed by
// array position k1*ncols + col), fft_tw = Plan<LLOC> stage twiddles,
// tw_lo = exp(-2 pi i t / L) for t < L. No masks (nvalid = full).
template <int LLOC, int C, int B, int NT, int SIGN, int MINB>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(NT, MINB)
    cluster_col_kernel(const __grid_constant__ PassArgs a) {
  namespace cg = cooperative_groups;
  using G = ClusterGeom<LLOC, C, B>;
  using Cx = Ctx<AX_COL, LLOC, B, PROG_DOUBLE>;
  extern __shared__ double2 lattdse_smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int col0 = (int)(blockIdx.x / C) * B;
  const long long bat = blockIdx.y;
  const double2* tw = a.tw_lo;
  constexpr int L = G::L;
  constexpr int TPT = (G::TASKS + NT - 1) / NT;

  // ---- phase A: global -> radix-C DFT over the blocks -> twiddle -> DSMEM.
  // All of a thread's global loads are issued before any DSMEM store: the
  // stores go through generic pointers the compiler cannot disambiguate
  // from `in`, so interleaving them would serialise one HBM round trip per
  // task (ncu: long-scoreboard stalls 12 per issued instruction).
  {
    const double2* in = a.in + bat * a.in_bstride;
    double2 x[TPT][C];
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = threadIdx.x + t * NT;
      if (G::TASKS % NT != 0 && q >= G::TASKS) break;
      const int b = q % B, i = r * G::SLICE + q / B;
#pragma unroll
      for (int k = 0; k < C; ++k) x[t][k] = in[(long long)(k * LLOC + i) * a.ncols + col0 + b];
    }
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = threadIdx.x + t * NT;
      if (G::TASKS % NT != 0 && q >= G::TASKS) break;
      const int b = q % B, i = r * G::SLICE + q / B;
      DFT<C, SIGN>::run(x[t]);
      Pow<C> pw;
      pw.init(__ldg_d2(tw + i), C > 4 ? __ldg_d2(tw + ((4 * i) % L)) : make_double2(1.0, 0.0), make_double2(1.0, 0.0));
      sfor<C>([&](auto kc) {
        constexpr int ka = decltype(kc)::value;
        double2 v = x[t][ka];
        if constexpr (ka > 0) {
          const double2 w = pw.template get<ka>();
          v = SIGN < 0 ? c_mul(v, w) : c_mulc(v, w);
        }
        double2* dst = cl.map_shared_rank(lattdse_smem, ka);
        dst[Cx::slot(b, i)] = v;
      });
    }
  }
  cl.sync();

  // ---- phase B: local FFT_Lloc, x D at k1 = r + C kb, local IFFT_Lloc
  Cx c{lattdse_smem, a, col0, bat};
  run_fft<DevExec, AX_COL, LLOC, B, NT, PROG_DOUBLE, SIGN, SRC_SMEM, DST_SMEM>(c);
  {
    // diagonal coefficients fetched as one batch per thread, then applied
    constexpr int PER = (B * LLOC + NT - 1) / NT;
    double2 dg[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int q = threadIdx.x + u * NT;
      dg[u] = make_double2(1.0, 0.0);
      if ((B * LLOC) % NT != 0 && q >= B * LLOC) break;
      const int b = q % B, kb = q / B;
      const long long j = (long long)(r + C * kb) * a.ncols + col0 + b;
      if (a.diag_kind == DG_LUT16)
        dg[u] = __ldg_d2(a.lut + ((const unsigned short*)a.diag_idx)[j]);
      else if (a.diag_kind == DG_CPLX)
        dg[u] = __ldg_d2(a.diag + j);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int q = threadIdx.x + u * NT;
      if ((B * LLOC) % NT != 0 && q >= B * LLOC) break;
      double2& v = lattdse_smem[Cx::slot(q % B, q / B)];
      v = c_mul(v, dg[u]);
    }
  }
  __syncthreads();
  run_fft<DevExec, AX_COL, LLOC, B, NT, PROG_DOUBLE, -SIGN, SRC_SMEM, DST_SMEM>(c);
  cl.sync();

  // ---- phase C: DSMEM -> untwiddle -> radix-C inverse DFT -> global
  // (all DSMEM loads first, for the same reason as phase A)
  {
    double2* out = a.out + bat * a.out_bstride;
    double2 z[TPT][C];
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = threadIdx.x + t * NT;
      if (G::TASKS % NT != 0 && q >= G::TASKS) break;
      const int b = q % B, i = r * G::SLICE + q / B;
#pragma unroll
      for (int k = 0; k < C; ++k) z[t][k] = cl.map_shared_rank(lattdse_smem, k)[Cx::slot(b, i)];
    }
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = threadIdx.x + t * NT;
      if (G::TASKS % NT != 0 && q >= G::TASKS) break;
      const int b = q % B, i = r * G::SLICE + q / B;
      Pow<C> pw;
      pw.init(__ldg_d2(tw + i), C > 4 ? __ldg_d2(tw + ((4 * i) % L)) : make_double2(1.0, 0.0), make_double2(1.0, 0.0));
      sfor<C>([&](auto kc) {
        constexpr int ka = decltype(kc)::value;
        if constexpr (ka > 0) {
          const double2 w = pw.template get<ka>();
          z[t][ka] = SIGN < 0 ? c_mulc(z[t][ka], w) : c_mul(z[t][ka], w);
        }
      });
      DFT<C, -SIGN>::run(z[t]);
#pragma unroll
      for (int k = 0; k < C; ++k) out[(long long)(k * LLOC + i) * a.ncols + col0 + b] = z[t][k];
    }
  }
  cl.sync();  // keep this CTA's tile alive until every peer has read it
}
#endif

}  // namespace lattdse_dev
