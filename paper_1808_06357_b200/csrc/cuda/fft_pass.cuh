// Fused Strang "pass" kernels: one launch reads a batch of lines of the
// 2-D view of the state from HBM/L2, runs up to two in-CTA FFTs along the
// line axis with a diagonal (phase) multiply between them, and writes back.
//
// The rank-1 Strang step on a length-N
// prime lattice is a length-M (M >= 2N-1) cyclic convolution handled by a
// four-step FFT over an M1 x M2 view, so one step is two passes:
//   COL pass: conj-twiddle, IFFT_M1, (mask j<N) x V[j], FFT_M1, twiddle
//   ROW pass: FFT_M2, x spectral table, IFFT_M2
// The rank-2 grid step is the same two passes without
// the four-step twiddles (ROW: IFFT x V FFT, COL: FFT x D IFFT).
//
// Each stage is a radix-R Stockham step (in-register DFT_R, twiddles from a
// correctly rounded table, one in-place shared-memory exchange). The first
// stage of the first transform reads straight from global memory and the last
// stage of the last transform writes straight to global memory, so a pass
// touches each element of the state exactly once in each direction.
#pragma once

#include "fft_core.cuh"

namespace lattdse_dev {

enum : int { AX_ROW = 0, AX_COL = 1 };
enum : int { DG_NONE = 0, DG_CPLX = 1, DG_LUT16 = 2, DG_LUT8 = 3, DG_SCALAR = 4 };
// PROG_DOUBLE: T1(SIGN1) -> mid diag (mask nvalid_mid) -> T2(-SIGN1)
// PROG_LOADDIAG: diag at load (mask nvalid_in) -> T(SIGN1)
// PROG_STOREDIAG: T(SIGN1) -> diag at store (mask nvalid_out)
enum : int { PROG_DOUBLE = 0, PROG_LOADDIAG = 1, PROG_STOREDIAG = 2 };

struct PassArgs {
  const double2* in;
  double2* out;
  long long in_bstride, out_bstride;       // batch strides in elements
  long long nvalid_in, nvalid_mid, nvalid_out;
  int ncols;                               // row length of the 2-D view
  int nlines;                              // lines along the pass axis (rows for ROW, cols for COL)
  int diag_kind;
  const double2* diag;                     // DG_CPLX
  const void* diag_idx;                    // DG_LUT16 / DG_LUT8
  const double2* lut;
  int pre_tw, post_tw, tw_shift;           // four-step twiddle exp(-2 pi i t / M)
  const double2* tw_lo;
  const double2* tw_hi;
  const double2* fft_tw;                   // exp(-2 pi i t / L), t < L
};

template <int L, int B> struct SmemGeom {
  static constexpr int pad() {
    if (B == 1) return 0;
    int want = B == 2 ? 4 : (B == 4 ? 2 : 1);
    return ((want - L % 8) % 8 + 8) % 8;
  }
  static constexpr int LS = L + pad();
  static constexpr int bytes = B * LS * 16;
};

template <int AXIS, int L, int B, int PROG> struct Ctx {
  double2* sm;
  const PassArgs* a;
  int line0;
  long long bat;

  LD_HD long long nat(int b, int i) const {
    if (AXIS == AX_ROW) return (long long)(line0 + b) * L + i;
    return (long long)i * a->ncols + (line0 + b);
  }
  LD_HD double2 twid(long long t) const {
    const long long mask = (1LL << a->tw_shift) - 1;
    return c_mul(a->tw_hi[t >> a->tw_shift], a->tw_lo[t & mask]);
  }
  LD_HD long long tw_index(int b, int i) const { return (long long)(line0 + b) * i; }
  LD_HD double2 apply_diag(double2 v, long long j) const {
    switch (a->diag_kind) {
      case DG_CPLX: return c_mul(v, a->diag[j]);
      case DG_LUT16: return c_mul(v, a->lut[((const unsigned short*)a->diag_idx)[j]]);
      case DG_LUT8: return c_mul(v, a->lut[((const unsigned char*)a->diag_idx)[j]]);
      case DG_SCALAR: return c_mul(v, a->lut[0]);
      default: return v;
    }
  }
  LD_HD bool live(int b) const { return line0 + b < a->nlines; }
  LD_HD double2 gload(int b, int i) const {
    long long j = nat(b, i);
    double2 v = make_double2(0.0, 0.0);
    if (!live(b)) return v;
    if (j < a->nvalid_in) {
      v = a->in[bat * a->in_bstride + j];
      if (PROG == PROG_LOADDIAG) v = apply_diag(v, j);  // diag tables hold nvalid_in entries
    }
    if (AXIS == AX_COL && a->pre_tw) v = c_mulc(v, twid(tw_index(b, i)));
    return v;
  }
  LD_HD void gstore(int b, int i, double2 v) const {
    if (!live(b)) return;
    if (AXIS == AX_COL && a->post_tw) v = c_mul(v, twid(tw_index(b, i)));
    long long j = nat(b, i);
    if (j >= a->nvalid_out) return;
    if (PROG == PROG_STOREDIAG) v = apply_diag(v, j);
    a->out[bat * a->out_bstride + j] = v;
  }
  LD_HD double2 mid(int b, int i, double2 v) const {
    long long j = nat(b, i);
    if (!live(b) || j >= a->nvalid_mid) return make_double2(0.0, 0.0);
    return apply_diag(v, j);
  }
};

enum : int { SRC_SMEM = 0, SRC_GLOBAL = 1 };
enum : int { DST_SMEM = 0, DST_SMEM_MID = 1, DST_GLOBAL = 2 };

template <int AXIS, int L, int B, int NT, int PROG, int S, int SIGN, int SRC, int DST> struct Stage {
  using P = Plan<L>;
  static constexpr int R = P::radix(S);
  static constexpr int Ns = P::ns(S);
  static constexpr int T = L / R;
  static constexpr int TASKS = B * T;
  static constexpr int TPT = (TASKS + NT - 1) / NT;
  static constexpr int LS = SmemGeom<L, B>::LS;
  static constexpr int src = SRC, dst = DST, nt = NT;
  using C = Ctx<AXIS, L, B, PROG>;

  LD_HD static void map(int q, int& b, int& j) {
    if (AXIS == AX_ROW) {
      b = q / T;
      j = q % T;
    } else {
      b = q % B;
      j = q / B;
    }
  }
  LD_HD static void read(const C& c, int tid, double2 (&v)[TPT][R]) {
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      int b, j;
      map(q, b, j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (SRC == SRC_GLOBAL)
          v[t][r] = c.gload(b, j + r * T);
        else
          v[t][r] = c.sm[b * LS + j + r * T];
      }
    }
  }
  LD_HD static void write(const C& c, int tid, double2 (&v)[TPT][R]) {
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      int b, j;
      map(q, b, j);
      const int k = j % Ns;
      if (Ns > 1) {
        const int step = L / (Ns * R);
#pragma unroll
        for (int r = 1; r < R; ++r) {
          double2 w = c.a->fft_tw[r * k * step];
          v[t][r] = SIGN < 0 ? c_mul(v[t][r], w) : c_mulc(v[t][r], w);
        }
      }
      DFT<R, SIGN>::run(v[t]);
      const int idxD = (j / Ns) * Ns * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        int pos = idxD + r * Ns;
        if (DST == DST_GLOBAL)
          c.gstore(b, pos, v[t][r]);
        else if (DST == DST_SMEM_MID)
          c.sm[b * LS + pos] = c.mid(b, pos, v[t][r]);
        else
          c.sm[b * LS + pos] = v[t][r];
      }
    }
  }
};

#if defined(__CUDACC__)
struct DevExec {
  template <class St, class C> __device__ __forceinline__ static void stage(const C& c) {
    double2 v[St::TPT][St::R];
    St::read(c, threadIdx.x, v);
    if (St::src == SRC_SMEM) __syncthreads();
    St::write(c, threadIdx.x, v);
    if (St::dst != DST_GLOBAL) __syncthreads();
  }
};
#endif

// Run one transform of sign SIGN over the CTA's lines.
#pragma nv_exec_check_disable
template <class Exec, int AXIS, int L, int B, int NT, int PROG, int SIGN, int FIRST, int LAST, class C>
LD_HD void run_fft(const C& c) {
  constexpr int nst = Plan<L>::nst;
  sfor<nst>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    constexpr int src = (s == 0) ? FIRST : SRC_SMEM;
    constexpr int dst = (s == nst - 1) ? LAST : DST_SMEM;
    Exec::template stage<Stage<AXIS, L, B, NT, PROG, s, SIGN, src, dst>>(c);
  });
}

#pragma nv_exec_check_disable
template <class Exec, int AXIS, int L, int B, int NT, int PROG, int SIGN1>
LD_HD void run_pass(const Ctx<AXIS, L, B, PROG>& c) {
  if constexpr (PROG == PROG_DOUBLE) {
    run_fft<Exec, AXIS, L, B, NT, PROG, SIGN1, SRC_GLOBAL, DST_SMEM_MID>(c);
    run_fft<Exec, AXIS, L, B, NT, PROG, -SIGN1, SRC_SMEM, DST_GLOBAL>(c);
  } else {
    run_fft<Exec, AXIS, L, B, NT, PROG, SIGN1, SRC_GLOBAL, DST_GLOBAL>(c);
  }
}

#if defined(__CUDACC__)
template <int AXIS, int L, int B, int NT, int PROG, int SIGN1>
__global__ void __launch_bounds__(NT) fft_pass_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ double2 lattdse_smem[];
  Ctx<AXIS, L, B, PROG> c{lattdse_smem, &a, (int)blockIdx.x * B, (long long)blockIdx.y};
  run_pass<DevExec, AXIS, L, B, NT, PROG, SIGN1>(c);
}
#endif

}  // namespace lattdse_dev
