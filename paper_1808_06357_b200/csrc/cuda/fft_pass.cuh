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
// correctly rounded table, one in-place shared-memory exchange).
//
// fft_pass_kernel: one CTA per tile of B lines; stage 0 loads straight from
// global, the last stage stores straight to global. It runs every program
// and layout; the per-step PROG_DOUBLE passes of the plain layouts have a
// leaner kernel of their own (fft_pass4.cuh).
#pragma once

#include "fft_core.cuh"

#ifndef LATTDSE_FUSED_MID
#define LATTDSE_FUSED_MID 1  // fuse T1's last stage, the diag and T2's first stage (reversed plan)
#endif
#ifndef LATTDSE_PINGPONG
#define LATTDSE_PINGPONG 1  // two shared buffers: stage s reads one, writes the other (1 barrier/stage)
#endif
#ifndef LATTDSE_MID_PREFETCH
#define LATTDSE_MID_PREFETCH 1  // batch the mid-diagonal loads ahead of the fused mid stage
#endif
#ifndef LATTDSE_ABLATE
#define LATTDSE_ABLATE 0  // devtest-only timing ablations: 1 mid diag, 2 stage twiddles, 4 stage-0 loads
#endif

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
  const double2* fft_tw;                   // per-stage twiddles, Plan<L>::tw_offset layout
  const double2* fft_tw2;                  // same for the reversed plan (second transform of PROG_DOUBLE)
  // Good-Thomas (prime-factor) rank-1 layout: position (n1, n2) of the
  // M1 x M2 view holds natural index (M2*n1 + M1*n2) mod M, gcd(M1,M2)=1.
  int pfa;
  int pM1, pM2;
  long long pM;
  // Sharded (distributed) layouts. COL pass on a column slab: storage row
  // length ncols (slab width), global column = col_off + local column,
  // natural index i*ncols_g + global column. ROW pass on a block-major row
  // slab: a row is rb_n blocks of rb_w elements, block q of row r at
  // q*rb_stride + r*rb_w (rb_w = 0: plain contiguous rows).
  int col_off;
  int ncols_g;
  int rb_w, rb_n;
  long long rb_stride;
  // Three-level rows on a block-major row slab (each row an Ma x Mb matrix,
  // Mb | rb_w): the single-transform COL passes of length Ma run inside the
  // rows with batch = slab row, batch stride rb_w; the Mb-long ROW lines are
  // contiguous, so the ROW pass sees the slab as plain lines (rb_w = 0).
  // Three-level rank-1 layout: a COL pass inside the rows of the M1 x M2 view
  // (each row an Ma x Mb matrix, one per batch index) needs the four-step
  // twiddles of length M2 = M / M1: W_M2^t = W_M^(M1 t). 0 or 1: plain.
  long long tw_mul;
  // Fused observables of PROG_STOREDIAG passes: when obs is
  // set, every stored value v (after the diagonal) adds |v|^2 and w_j |v|^2
  // to per-CTA partial sums obs[2*(blockIdx.y*gridDim.x + blockIdx.x) + {0,1}],
  // w_j = obs_w[j] (potential, natural order) or obs_wscale * obs_widx[j]
  // (kinetic weight from the norm index). The host finishes the sums in
  // long double: ||u||^2, the potential and the kinetic parts of E come out
  // of the passes that produce the samples / coefficients anyway.
  double* obs;
  const double* obs_w;
  const unsigned short* obs_widx;
  double obs_wscale;
  // pass4 (fft_pass4.cuh): mid mask by rows for COL passes (nvalid_mid =
  // mid_rb * ncols + mid_cb), and the L2 prefetch distance in tiles (0: off)
  int mid_rb, mid_cb;
  int pf;
};

// Shared-memory slots of one tile: B lines, each Plan<L>::phys-swizzled and
// padded so that B adjacent lines accessed "line-fastest" hit distinct banks.
template <int L, int B> struct SmemGeom {
  static constexpr int span = Plan<L>::phys(L - 1) + 1;
  static constexpr int pad() {
    if (B == 1) return 0;
    int want = B == 2 ? 4 : (B == 4 ? 2 : 1);
    return ((want - span % 8) % 8 + 8) % 8;
  }
  static constexpr int LS = span + pad();
  static constexpr int tile = B * LS;  // slots of one buffer
  // ping-pong only while two buffers still leave room for 2+ CTAs per SM
  static constexpr bool pp = LATTDSE_PINGPONG && tile * 16 <= 48 * 1024;
  static constexpr int bytes = (pp ? 2 : 1) * tile * 16;
};

LD_HD double2 __ldg_d2(const double2* p) {
#if defined(__CUDA_ARCH__)
  return __ldg(p);
#else
  return *p;
#endif
}

template <int AXIS, int L, int B, int PROG> struct Ctx {
  double2* sm;   // buffer 0 (buffer 1 follows at sm + SmemGeom::tile when ping-ponging)
  PassArgs a;  // by value: fields resolve to parameter-bank operands, not pointer loads
  int line0;
  long long bat;
  mutable double acc0 = 0.0, acc1 = 0.0;  // fused observables (PassArgs::obs)

  static constexpr int LS = SmemGeom<L, B>::LS;
  LD_HD static int slot(int b, int i) { return b * LS + Plan<L>::phys(i); }
  // buffer used as the source of stage-sequence position p (0, 1, 2, ...)
  LD_HD double2* buf(int p) const {
    return (SmemGeom<L, B>::pp && (p & 1)) ? sm + SmemGeom<L, B>::tile : sm;
  }

  // array position of element (b, i) in the 2-D view
  LD_HD long long pos(int b, int i) const {
    if (AXIS == AX_ROW) {
      if (a.rb_w > 0) {
        const int q = i / a.rb_w;
        return (long long)q * a.rb_stride + (long long)(line0 + b) * a.rb_w + (i - q * a.rb_w);
      }
      return (long long)(line0 + b) * L + i;
    }
    // inside a block-major slab row (the row is the batch index): single-
    // transform programs only, so the fused per-step passes compile unchanged
    if (PROG != PROG_DOUBLE && a.rb_w > 0) {
      const int p = i * a.ncols + line0 + b;
      const int q = p / a.rb_w;
      return (long long)q * a.rb_stride + (p - q * a.rb_w);
    }
    return (long long)i * a.ncols + (line0 + b);
  }
  // natural (sample / coefficient) index of element (b, i)
  LD_HD long long nat(int b, int i) const {
    if (AXIS == AX_COL && a.pfa) {
      long long n = (long long)a.pM2 * i + (long long)a.pM1 * (line0 + b);
      return n >= a.pM ? n - a.pM : n;
    }
    if (AXIS == AX_COL && a.ncols_g > 0) return (long long)i * a.ncols_g + (a.col_off + line0 + b);
    return pos(b, i);
  }
  // the compact (natural-order) side of single-transform programs
  LD_HD long long in_index(int b, int i) const { return PROG == PROG_LOADDIAG ? nat(b, i) : pos(b, i); }
  LD_HD long long out_index(int b, int i) const { return PROG == PROG_STOREDIAG ? nat(b, i) : pos(b, i); }
  LD_HD double2 twid(long long t) const {
    const long long mask = (1LL << a.tw_shift) - 1;
    return c_mul(a.tw_hi[t >> a.tw_shift], a.tw_lo[t & mask]);
  }
  LD_HD double2 apply_diag(double2 v, long long j) const {
    switch (a.diag_kind) {
      case DG_CPLX: return c_mul(v, a.diag[j]);
      case DG_LUT16: return c_mul(v, a.lut[((const unsigned short*)a.diag_idx)[j]]);
      case DG_LUT8: return c_mul(v, a.lut[((const unsigned char*)a.diag_idx)[j]]);
      case DG_SCALAR: return c_mul(v, a.lut[0]);
      default: return v;
    }
  }
  LD_HD bool live(int b) const { return line0 + b < a.nlines; }
  // v1 stage-0 source: global memory
  LD_HD double2 gload(int b, int i) const {
    long long j = in_index(b, i);
    double2 v = make_double2(0.0, 0.0);
    if (!live(b)) return v;
    if (j < a.nvalid_in) {
      v = a.in[bat * a.in_bstride + j];
      if (PROG == PROG_LOADDIAG) v = apply_diag(v, j);  // diag tables hold nvalid_in entries
    }
    return v;
  }
  LD_HD void gstore(int b, int i, double2 v) const {
    if (!live(b)) return;
    long long j = out_index(b, i);
    if (j >= a.nvalid_out) return;
    if (PROG == PROG_STOREDIAG) {
      v = apply_diag(v, j);
      if (a.obs) {
        const double q = fma(v.x, v.x, v.y * v.y);
        acc0 += q;
        acc1 = fma(a.obs_w ? a.obs_w[j] : a.obs_wscale * (double)a.obs_widx[j], q, acc1);
      }
    }
    a.out[bat * a.out_bstride + j] = v;
  }
  // Coefficients of the mid diagonal for elements j + r*T, r < R (zero where
  // masked), fetched as one batch of independent loads: issued before the
  // stage's twiddles and butterflies, their latency overlaps that work
  // instead of serialising one table load per element after it.
  template <int R, int T> LD_HD void mid_fetch(int b, int j, double2 (&dg)[R]) const {
    const bool lv = live(b);
    const double2 zero = make_double2(0.0, 0.0);
    if (LATTDSE_ABLATE & 1) {
#pragma unroll
      for (int r = 0; r < R; ++r) dg[r] = (lv && pos(b, j + r * T) < a.nvalid_mid) ? make_double2(1.0, 0.0) : zero;
    } else if (a.diag_kind == DG_CPLX) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long jj = pos(b, j + r * T);
        dg[r] = (lv && jj < a.nvalid_mid) ? __ldg_d2(a.diag + jj) : zero;
      }
    } else if (a.diag_kind == DG_LUT16) {
      // norm index first (one batch), then the phase LUT (one batch)
      const unsigned short* ix = (const unsigned short*)a.diag_idx;
      unsigned short id[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long jj = pos(b, j + r * T);
        id[r] = (lv && jj < a.nvalid_mid) ? ix[jj] : (unsigned short)0xFFFF;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) dg[r] = id[r] != 0xFFFF ? __ldg_d2(a.lut + id[r]) : zero;
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long jj = pos(b, j + r * T);
        dg[r] = (lv && jj < a.nvalid_mid) ? apply_diag(make_double2(1.0, 0.0), jj) : zero;
      }
    }
  }
  // the mid diagonal and its mask are indexed by array position
  LD_HD double2 mid(int b, int i, double2 v) const {
    long long j = pos(b, i);
    if (!live(b) || j >= a.nvalid_mid) return make_double2(0.0, 0.0);
    if (LATTDSE_ABLATE & 1) return v;
    return apply_diag(v, j);
  }
};


// Powers w^r, 0 <= r < R, of a twiddle from correctly rounded bases
// w, w^4, w^16: every power is at most three products deep.
template <int R> struct Pow {
  double2 b1, b2, b3, b4, b8, b12, b16;
  LD_HD void init(double2 w1, double2 w4, double2 w16) {
    b1 = w1;
    b2 = c_mul(w1, w1);
    b3 = c_mul(b2, w1);
    b4 = w4;
    b8 = c_mul(w4, w4);
    b12 = c_mul(b8, w4);
    b16 = w16;
  }
  template <int r> LD_HD double2 get() const {
    if constexpr (r == 0) return make_double2(1.0, 0.0);
    else if constexpr (r == 1) return b1;
    else if constexpr (r == 2) return b2;
    else if constexpr (r == 3) return b3;
    else if constexpr (r == 4) return b4;
    else if constexpr (r == 8) return b8;
    else if constexpr (r == 12) return b12;
    else if constexpr (r == 16) return b16;
    else if constexpr (r < 16) return c_mul(get<4 * (r / 4)>(), get<r % 4>());
    else return c_mul(b16, get<r - 16>());
  }
};

enum : int { SRC_SMEM = 0, SRC_GLOBAL = 1 };
enum : int { DST_SMEM = 0, DST_SMEM_MID = 1, DST_GLOBAL = 2 };

// Stage S of a transform, at position Q of the pass's stage sequence: reads
// shared buffer buf(Q), writes buf(Q+1) (the same buffer unless ping-ponging).
template <int AXIS, int L, int B, int NT, int PROG, int S, int SIGN, int SRC, int DST, bool REV = false, int Q = S>
struct Stage {
  using P = PlanX<L, REV>;
  static constexpr int R = P::radix(S);
  static constexpr int Ns = P::ns(S);
  static constexpr int T = L / R;
  static constexpr int TASKS = B * T;
  static constexpr int TPT = (TASKS + NT - 1) / NT;
  static constexpr int src = SRC, dst = DST, nt = NT;
  static constexpr bool pp = SmemGeom<L, B>::pp;
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
  // four-step twiddles W(col * (j + r*T)) = W(col*j) * W(col*T)^r for the
  // elements j + r*T a task touches in stage 0 / the last stage
  LD_HD static void fourstep(const C& c, int b, int j, double2 (&v)[R], bool conj) {
    const long long col = (long long)(c.a.col_off + c.line0 + b) * (c.a.tw_mul > 1 ? c.a.tw_mul : 1);
    const double2 base = c.twid(col * j);
    Pow<R> pw;
    pw.init(c.twid(col * T), R > 4 ? c.twid(col * 4 * T) : make_double2(1.0, 0.0),
            R > 16 ? c.twid(col * 16 * T) : make_double2(1.0, 0.0));
    // base * w^(4q + m) = (base * w^(4q)) * w^m: one product per element
    double2 bq[(R + 3) / 4];
    sfor<(R + 3) / 4>([&](auto qc) {
      constexpr int q = decltype(qc)::value;
      bq[q] = q == 0 ? base : c_mul(base, pw.template get<4 * q>());
    });
    sfor<R>([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      const double2 w = (r % 4 == 0) ? bq[r / 4] : c_mul(bq[r / 4], pw.template get<r % 4>());
      v[r] = conj ? c_mulc(v[r], w) : c_mul(v[r], w);
    });
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
        if (SRC == SRC_GLOBAL && (LATTDSE_ABLATE & 4))
          v[t][r] = c.buf(Q)[C::slot(b, j + r * T)];
        else if (SRC == SRC_GLOBAL)
          v[t][r] = c.gload(b, j + r * T);
        else
          v[t][r] = c.buf(Q)[C::slot(b, j + r * T)];
      }
      if (SRC != SRC_SMEM && AXIS == AX_COL && c.a.pre_tw) fourstep(c, b, j, v[t], true);
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
        // stage twiddles w^r from table rows r = 1, 4, 16
        const double2* tw = (REV ? c.a.fft_tw2 : c.a.fft_tw) + P::tw_offset(S) + k;
        Pow<R> pw;
        if (LATTDSE_ABLATE & 2)
          pw.init(make_double2(0.8, 0.6 + k * 1e-9), make_double2(0.6, 0.8), make_double2(0.0, 1.0));
        else
          pw.init(__ldg_d2(tw), R > 4 ? __ldg_d2(tw + 3 * Ns) : make_double2(1.0, 0.0),
                  R > 16 ? __ldg_d2(tw + 15 * Ns) : make_double2(1.0, 0.0));
        sfor<R>([&](auto rc) {
          constexpr int r = decltype(rc)::value;
          if constexpr (r > 0) {
            const double2 w = pw.template get<r>();
            v[t][r] = SIGN < 0 ? c_mul(v[t][r], w) : c_mulc(v[t][r], w);
          }
        });
      }
      DFT<R, SIGN>::run(v[t]);
      const int idxD = (j / Ns) * Ns * R + k;
      // last stage: idxD == j, outputs at j + r*T (the four-step pattern)
      if (DST == DST_GLOBAL && AXIS == AX_COL && c.a.post_tw) fourstep(c, b, j, v[t], false);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        int pos = idxD + r * Ns;
        if (DST == DST_GLOBAL)
          c.gstore(b, pos, v[t][r]);
        else if (DST == DST_SMEM_MID)
          c.buf(Q + 1)[C::slot(b, pos)] = c.mid(b, pos, v[t][r]);
        else
          c.buf(Q + 1)[C::slot(b, pos)] = v[t][r];
      }
    }
  }
};

// Fused middle of PROG_DOUBLE: the first transform's last stage (forward
// plan, sign SIGN), the diagonal multiply, and the second transform's first
// stage (reversed plan, sign -SIGN, Ns = 1) on the same registers: with the
// reversed plan both stages cover elements j + r*T of task j, so the
// intermediate never goes through shared memory.
template <int AXIS, int L, int B, int NT, int SIGN, int SRC, int DST, int Q> struct MidStage {
  using P1 = PlanX<L, false>;
  static constexpr int S1 = P1::nst - 1;
  static constexpr int R = P1::radix(S1);
  static constexpr int Ns = P1::ns(S1);
  static constexpr int T = L / R;
  static_assert(T == Ns, "last stage covers j + r*T");
  static constexpr int TASKS = B * T;
  static constexpr int TPT = (TASKS + NT - 1) / NT;
  static constexpr int src = SRC, dst = DST, nt = NT;
  static constexpr bool pp = SmemGeom<L, B>::pp;
  using First = Stage<AXIS, L, B, NT, PROG_DOUBLE, S1, SIGN, SRC, DST_SMEM, false, Q>;
  using C = Ctx<AXIS, L, B, PROG_DOUBLE>;

  LD_HD static void read(const C& c, int tid, double2 (&v)[TPT][R]) { First::read(c, tid, v); }
  LD_HD static void write(const C& c, int tid, double2 (&v)[TPT][R]) {
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      int b, j;
      First::map(q, b, j);
#if LATTDSE_MID_PREFETCH
      double2 dg[R];
      c.template mid_fetch<R, T>(b, j, dg);
#endif
      if (Ns > 1) {
        const double2* tw = c.a.fft_tw + P1::tw_offset(S1) + j;
        Pow<R> pw;
        pw.init(__ldg_d2(tw), R > 4 ? __ldg_d2(tw + 3 * Ns) : make_double2(1.0, 0.0),
                R > 16 ? __ldg_d2(tw + 15 * Ns) : make_double2(1.0, 0.0));
        sfor<R>([&](auto rc) {
          constexpr int r = decltype(rc)::value;
          if constexpr (r > 0) {
            const double2 w = pw.template get<r>();
            v[t][r] = SIGN < 0 ? c_mul(v[t][r], w) : c_mulc(v[t][r], w);
          }
        });
      }
      DFT<R, SIGN>::run(v[t]);
#if LATTDSE_MID_PREFETCH
#pragma unroll
      for (int r = 0; r < R; ++r) v[t][r] = c_mul(v[t][r], dg[r]);
#else
#pragma unroll
      for (int r = 0; r < R; ++r) v[t][r] = c.mid(b, j + r * T, v[t][r]);
#endif
      DFT<R, -SIGN>::run(v[t]);  // second transform, stage 0 (Ns = 1: no twiddle)
      // stage-0 outputs of the reversed plan: idxD = j*R, positions j*R + r
      if (DST == DST_GLOBAL && AXIS == AX_COL && c.a.post_tw) First::fourstep(c, b, j, v[t], false);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (DST == DST_GLOBAL)
          c.gstore(b, j * R + r, v[t][r]);
        else
          c.buf(Q + 1)[C::slot(b, j * R + r)] = v[t][r];
      }
    }
  }
};

#if defined(__CUDACC__)
struct DevExec {
  template <class St, class C> __device__ __forceinline__ static void stage(const C& c) {
    double2 v[St::TPT][St::R];
    St::read(c, threadIdx.x, v);
    if (!St::pp && St::src != SRC_GLOBAL) __syncthreads();  // in place: all reads before any write
    St::write(c, threadIdx.x, v);
    if (St::dst != DST_GLOBAL) __syncthreads();
  }
};
#endif

// Run stages [S0, nst) of one transform of sign SIGN over the CTA's lines.
#pragma nv_exec_check_disable
template <class Exec, int AXIS, int L, int B, int NT, int PROG, int SIGN, int FIRST, int LAST, bool REV = false,
          int S0 = 0, int S1 = Plan<L>::nst, int QB = 0, class C>
LD_HD void run_fft(const C& c) {
  constexpr int nst = Plan<L>::nst;
  sfor<S1 - S0>([&](auto sc) {
    constexpr int s = decltype(sc)::value + S0;
    constexpr int src = (s == 0) ? FIRST : SRC_SMEM;
    constexpr int dst = (s == nst - 1) ? LAST : DST_SMEM;
    Exec::template stage<Stage<AXIS, L, B, NT, PROG, s, SIGN, src, dst, REV, QB + s - S0>>(c);
  });
}

#pragma nv_exec_check_disable
template <class Exec, int AXIS, int L, int B, int NT, int PROG, int SIGN1, int FIRST = SRC_GLOBAL>
LD_HD void run_pass(const Ctx<AXIS, L, B, PROG>& c) {
  if constexpr (PROG == PROG_DOUBLE && !LATTDSE_FUSED_MID) {
    constexpr int nst = Plan<L>::nst;
    run_fft<Exec, AXIS, L, B, NT, PROG, SIGN1, FIRST, DST_SMEM_MID>(c);
    run_fft<Exec, AXIS, L, B, NT, PROG, -SIGN1, SRC_SMEM, DST_GLOBAL, false, 0, nst, nst>(c);
  } else if constexpr (PROG == PROG_DOUBLE) {
    constexpr int nst = Plan<L>::nst;
    // first transform up to (excluding) its last stage
    run_fft<Exec, AXIS, L, B, NT, PROG, SIGN1, FIRST, DST_SMEM, false, 0, nst - 1, 0>(c);
    // last stage + diag + first stage of the reversed second transform
    Exec::template stage<MidStage<AXIS, L, B, NT, SIGN1, (nst == 1 ? FIRST : SRC_SMEM),
                                  (nst == 1 ? DST_GLOBAL : DST_SMEM), nst - 1>>(c);
    // remaining stages of the second transform (reversed plan)
    run_fft<Exec, AXIS, L, B, NT, PROG, -SIGN1, SRC_SMEM, DST_GLOBAL, true, 1, nst, nst>(c);
  } else {
    run_fft<Exec, AXIS, L, B, NT, PROG, SIGN1, FIRST, DST_GLOBAL>(c);
  }
}

#if defined(__CUDACC__)
template <int AXIS, int L, int B, int NT, int PROG, int SIGN1, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) fft_pass_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ double2 lattdse_smem[];
  // programmatic dependent launch (solver.cu, LATTDSE_PDL): let the next pass
  // be scheduled onto SMs this grid's tail frees, and wait for the previous
  // pass's results before touching them (both are no-ops without the launch
  // attribute)
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  Ctx<AXIS, L, B, PROG> c{lattdse_smem, a, (int)blockIdx.x * B, (long long)blockIdx.y};
  run_pass<DevExec, AXIS, L, B, NT, PROG, SIGN1>(c);
  if constexpr (PROG == PROG_STOREDIAG) {
    if (a.obs) {  // block partials of the fused observables (uniform branch)
      double s0 = c.acc0, s1 = c.acc1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_down_sync(0xffffffffu, s0, o);
        s1 += __shfl_down_sync(0xffffffffu, s1, o);
      }
      double* red = reinterpret_cast<double*>(lattdse_smem);
      __syncthreads();  // the last stage may still be reading shared memory
      if ((threadIdx.x & 31) == 0) {
        red[2 * (threadIdx.x >> 5)] = s0;
        red[2 * (threadIdx.x >> 5) + 1] = s1;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int w = 0; w < (NT + 31) / 32; ++w) {
          t0 += red[2 * w];
          t1 += red[2 * w + 1];
        }
        const long long blk = (long long)blockIdx.y * gridDim.x + blockIdx.x;
        a.obs[2 * blk] = t0;
        a.obs[2 * blk + 1] = t1;
      }
    }
  }
}

#endif

}  // namespace lattdse_dev
