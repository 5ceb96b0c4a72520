// Sharded single-wave-function Strang stepping (include/lattdse/dist.hpp).
//
// Layouts per rank g (G ranks, M = M1*M2, Hb = M1/G, Wb = M2/G):
//   column slab  A_g, S_g, V_g, Vh_g : M1 x Wb row-major, global columns
//                                      [g*Wb, (g+1)*Wb), zeros where the
//                                      natural index j1*M2 + col >= N
//   row slab     B_g, K_g            : G blocks q of Hb x Wb (block-major):
//                                      rows [g*Hb, (g+1)*Hb), columns of
//                                      block q = [q*Wb, (q+1)*Wb)
// Exchange col->row: A_g block h (rows of h, contiguous) -> B_h block g.
// Exchange row->col: B_h block g -> A_g block h. Both sides contiguous, so
// the NCCL path is G grouped send/recv pairs with no pack/unpack kernels.
//
// Three-level (config 4, M beyond one COL x ROW split): every length-M2 row
// is an Ma x Mb matrix (M2 = Ma*Mb, G | Ma so each Mb-line lies inside one
// Wb-wide block). The row side of a step is then three local passes on the
// row slab -- COL pass of length Ma inside the rows (forward, four-step
// twiddle W_M2), ROW pass of length Mb (x K^), COL pass inverse -- and the
// step still needs exactly two exchanges.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <numeric>

#include "fft_pass.cuh"
#include "sampling.cuh"
#include "aaset_dev.hpp"
#include "lattdse/dist.hpp"
#include "pass_registry.hpp"

using namespace lattdse_dev;

namespace lattdse {

#define LD_CK(x)                                                                                      \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) raise(Errc::device_error, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

// ---------------------------------------------------------------- NCCL
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;

  static Nccl& get() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
      // the process's NCCL (e.g. torch's) if already loaded, else the system one
      for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (n.h) break;
      }
      if (!n.h) return;
      auto sym = [&](auto& fp, const char* s) { fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(n.h, s)); };
      sym(n.GetUniqueId, "ncclGetUniqueId");
      sym(n.CommInitRank, "ncclCommInitRank");
      sym(n.CommDestroy, "ncclCommDestroy");
      sym(n.GroupStart, "ncclGroupStart");
      sym(n.GroupEnd, "ncclGroupEnd");
      sym(n.Send, "ncclSend");
      sym(n.Recv, "ncclRecv");
      sym(n.AllReduce, "ncclAllReduce");
      sym(n.GetErrorString, "ncclGetErrorString");
      sym(n.CommGetAsyncError, "ncclCommGetAsyncError");
    });
    if (!n.h || !n.CommInitRank || !n.Send || !n.Recv)
      raise(Errc::nccl_error, "libnccl.so.2 not found or incomplete (dlopen)");
    return n;
  }
};

#define LD_NCCL(x)                                                                                  \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess) raise(Errc::nccl_error, std::string(#x) + ": " + Nccl::get().GetErrorString(r_)); \
  } while (0)

// --------------------------------------------------------------- kernels
__global__ void k_colslab(const double2* __restrict__ src, long long N, long long M1, long long M2, long long Wb,
                          long long col_off, double2* __restrict__ out) {
  const long long n = M1 * Wb;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const long long j1 = p / Wb, c = p - j1 * Wb;
    const long long j = j1 * M2 + col_off + c;
    out[p] = j < N ? src[j] : make_double2(0.0, 0.0);
  }
}
__global__ void k_slab2nat(const double2* __restrict__ slab, long long N, long long M1, long long M2, long long Wb,
                           long long col_off, double2* __restrict__ dst) {
  const long long n = M1 * Wb;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const long long j1 = p / Wb, c = p - j1 * Wb;
    const long long j = j1 * M2 + col_off + c;
    if (j < N) dst[j] = slab[p];
  }
}
__global__ void k_rowblk(const double2* __restrict__ src, long long M2, long long Hb, long long Wb, int G,
                         long long row_off, double2* __restrict__ out) {
  const long long n = (long long)G * Hb * Wb;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const long long q = p / (Hb * Wb), rem = p - q * Hb * Wb, r = rem / Wb, c = rem - r * Wb;
    out[p] = src[(row_off + r) * M2 + q * Wb + c];
  }
}
// unnormalised g on a column slab (zeros where the natural index >= N)
__global__ void k_slab_sample_g(const R1Points P, const double* __restrict__ c, const int* __restrict__ pj, double inv2s2,
                                long long M1, long long M2, long long Wb, long long col_off, double2* __restrict__ out) {
  const long long n = M1 * Wb;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const long long j1 = q / Wb, cc = q - j1 * Wb;
    const long long j = j1 * M2 + col_off + cc;
    out[q] = j < P.N ? sample_g_point(P, j, c, pj, inv2s2) : make_double2(0.0, 0.0);
  }
}
__global__ void k_scale_slab(double2* __restrict__ x, long long n, double s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = make_double2(x[i].x * s, x[i].y * s);
}
// ---- propagator tables built slab by slab (no unsharded table anywhere)
// c_j = exp(-pi i j^2 / N) (conj: +), j^2 reduced mod 2N exactly (solver.cu k_chirp)
__device__ __forceinline__ double2 chirp_at(long long j, long long N, bool conj) {
  unsigned long long q = (unsigned long long)(((unsigned __int128)j * (unsigned __int128)j) % (unsigned __int128)(2 * N));
  double sgn = 1.0;
  if (q >= (unsigned long long)N) {
    q -= (unsigned long long)N;
    sgn = -1.0;
  }
  double s, co;
  sincospi((double)q / (double)N, &s, &co);
  return make_double2(sgn * co, conj ? sgn * s : -sgn * s);
}
// natural index of column-slab position q
__device__ __forceinline__ long long slab_nat(long long q, long long M2, long long Wb, long long col_off) {
  const long long j1 = q / Wb;
  return j1 * M2 + col_off + (q - j1 * Wb);
}
// potential phase exp(i coef v(p_j)) on a column slab (zeros for j >= N): V, V^(1/2)
__global__ void k_slab_vphase(const R1Points P, const double* __restrict__ a, const double* __restrict__ b, double coef,
                              long long M1, long long M2, long long Wb, long long col_off, double2* __restrict__ out) {
  const long long n = M1 * Wb;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const long long j = slab_nat(q, M2, Wb, col_off);
    double2 v = make_double2(0.0, 0.0);
    if (j < P.N) {
      double sn, cs;
      sincos(coef * sample_v_point(P, j, a, b), &sn, &cs);
      v = make_double2(cs, sn);
    }
    out[q] = v;
  }
}
// what: 0 even wrap of the chirp c into length M, scaled (Bluestein kernel of the synthesis);
//       1 conj chirp (j < N); 2 kinetic phase D_j / N (norm index + LUT) times conj chirp (j < N)
__global__ void k_slab_chirp(int what, long long N, long long M, long long M1, long long M2, long long Wb, long long col_off,
                             double scale, const unsigned short* __restrict__ nidx, const double2* __restrict__ lut,
                             double2* __restrict__ out) {
  const long long n = M1 * Wb;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const long long t = slab_nat(q, M2, Wb, col_off);
    double2 v = make_double2(0.0, 0.0);
    if (what == 0) {
      if (t < N)
        v = chirp_at(t, N, false);
      else if (t > M - N)
        v = chirp_at(M - t, N, false);
      v = make_double2(v.x * scale, v.y * scale);
    } else if (t < N) {
      v = chirp_at(t, N, true);
      if (what == 2) v = c_mul(lut[nidx[t]], v);
    }
    out[q] = v;
  }
}
// K^ from F = FFT_M(zero-padded k) on a block-major row slab, in place. The
// circulant kernel is k wrapped periodically, wrap(k)[t] = k[t] (t < N) and
// k[t - (M - N)] (t > M - N); the second part is k without k[0], shifted by
// M - N, so FFT_M(wrap k)[m] = F[m] + w_m (F[m] - k[0]), w_m = exp(2 pi i m N / M):
// a pointwise map of F, no data moves between ranks. Slab position (row r of
// block q, column c) holds frequency m = k1 + M1 k2, k1 = row_off + r and k2 the
// column q Wb + c (three-level rows: column ka Mb + kb holds k2 = ka + Ma kb).
__global__ void k_khat_finish(double2* __restrict__ F, double2 k0, long long N, long long M, long long M1, long long Hb,
                              long long Wb, int G, long long row_off, long long Ma, long long Mb, double scale) {
  const long long n = (long long)G * Hb * Wb;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const long long q = p / (Hb * Wb), rem = p - q * Hb * Wb, r = rem / Wb, c = rem - r * Wb;
    const long long col = q * Wb + c;
    const long long k2 = Ma > 0 ? (col / Mb) + Ma * (col % Mb) : col;
    const unsigned long long m = (unsigned long long)(row_off + r) + (unsigned long long)M1 * (unsigned long long)k2;
    const unsigned long long e = (unsigned long long)(((unsigned __int128)m * (unsigned __int128)N) % (unsigned __int128)M);
    double sn, cs;
    sincospi(2.0 * (double)e / (double)M, &sn, &cs);
    const double2 w = make_double2(cs, sn);
    const double2 f = F[p];
    const double2 d = c_mul(w, make_double2(f.x - k0.x, f.y - k0.y));
    F[p] = make_double2((f.x + d.x) * scale, (f.y + d.y) * scale);
  }
}
__global__ void k_sumsq(const double2* __restrict__ x, long long n, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc += x[i].x * x[i].x + x[i].y * x[i].y;
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
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

std::vector<double2> roots(long long n, long long count, long long stride) {
  std::vector<double2> t(count);
  for (long long i = 0; i < count; ++i) {
    long long q = (i * stride) % n;
    long double a = -2.0L * kPiL * (long double)q / (long double)n;
    t[i] = make_double2((double)cosl(a), (double)sinl(a));
  }
  return t;
}

}  // namespace

// ------------------------------------------------------------------ Impl
struct DistSolver::Impl {
  int G = 2, rank = -1, device = 0;
  long long N = 0, M = 0, M1 = 0, M2 = 0, Hb = 0, Wb = 0;
  bool three = false;
  long long Ma = 0, Mb = 0;  // three-level: M2 = Ma * Mb
  cudaStream_t stream = nullptr;
  Lattice lat;
  AntiAliasSet aa;               // empty norm2: built on the device by the table solver
  ProblemSpec prob;
  std::vector<int> local;        // ranks living in this process
  struct Rank {
    DBuf<double2> A, B, S, V, Vh, K;
  };
  std::vector<Rank> rk;          // indexed like `local`
  DBuf<double2> tw_col, tw_row, tw_col2, tw_row2, tw_mid, tw_mid2, tw_lo, tw_hi, tmp;
  DBuf<double> partial;
  int tw_shift = 0;
  ncclComm_t comm = nullptr;
  bool have_dt = false;
  long long launches4 = 0;  // passes that ran on the lean kernels
  // row side in `chunks` row chunks (Hb % chunks == 0): the exchanges run on
  // their own stream, chunk by chunk, under the row passes of the other
  // chunks; 1: one blocking exchange each way
  int chunks = 1;
  cudaStream_t xstream = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_done;
  cudaEvent_t ev_col = nullptr, ev_back = nullptr;

  explicit Impl(const Lattice& l) : lat(l) {}

  int grid1d(long long n) const { return (int)std::min<long long>((n + 255) / 256, 148 * 16); }
  long long slab() const { return M1 * Wb; }

  void launch(int axis, int L, int prog, int sign, PassArgs a, long long nlines, long long nbatch = 1) {
    dev::PassKernel* k = dev::find_pass_kernel(axis, L, prog, sign);
    if (!k) raise(Errc::unsupported, "no pass kernel for L=" + std::to_string(L));
    // the lean per-step kernel (fft_pass4.cuh) where the slab pass is a plain
    // layout: the COL pass of a column slab (global column offset only enters
    // the four-step twiddles) and the ROW pass over contiguous lines (three-
    // level rows); block-major rows and the inner COL passes stay generic
    static const bool use_pass4 = !(std::getenv("LATTDSE_PASS4") && std::atoi(std::getenv("LATTDSE_PASS4")) == 0);
    if (use_pass4 && prog == PROG_DOUBLE && k->fn4[0] && a.diag_kind == DG_CPLX && a.rb_w == 0 && !a.pfa &&
        a.ncols_g == 0 && a.tw_mul <= 1 && !a.obs && nlines % k->B4 == 0 && nbatch <= 65535 &&
        (axis == AX_ROW ? (!a.pre_tw && !a.post_tw) : (a.pre_tw && a.post_tw && nlines == a.ncols))) {
      const long long span = axis == AX_COL ? (long long)L * a.ncols : nlines * (long long)L;
      if (a.nvalid_in >= span && a.nvalid_out >= span && a.nvalid_mid >= span) {
        if (!k->attr4_set) {
          for (const void* f : k->fn4)
            if (f) LD_CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem4));
          if (k->fn4w) LD_CK(cudaFuncSetAttribute(k->fn4w, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem4w));
          k->attr4_set = true;
        }
        a.nlines = (int)nlines;
        a.mid_rb = L;  // no mid mask (it is folded into the slab tables)
        a.mid_cb = 0;
        a.pf = 0;
        void* args4[] = {&a};
        LD_CK(cudaLaunchKernel(k->fn4[0], dim3((unsigned)(nlines / k->B4), (unsigned)nbatch), dim3(k->NT4), args4,
                               (size_t)k->smem4, stream));
        ++launches4;
        return;
      }
    }
    const void* fn = k->fn;
    if (prog == PROG_DOUBLE && k->fn_mb[k->default_mb]) fn = k->fn_mb[k->default_mb];
    if (!k->attr_set) {
      for (int m = 0; m <= 4; ++m) {
        const void* f = m == 0 ? k->fn : k->fn_mb[m];
        if (f) LD_CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem));
      }
      k->attr_set = true;
    }
    a.nlines = (int)nlines;
    void* args[] = {&a};
    LD_CK(cudaLaunchKernel(fn, dim3((unsigned)((nlines + k->B - 1) / k->B), (unsigned)nbatch), dim3(k->NT), args,
                           (size_t)k->smem, stream));
  }

  PassArgs col_args(int g) const {
    PassArgs a{};
    a.ncols = (int)Wb;
    a.col_off = (int)(g * Wb);
    a.fft_tw = tw_col.p;
    a.fft_tw2 = tw_col2.p;
    a.tw_lo = tw_lo.p;
    a.tw_hi = tw_hi.p;
    a.tw_shift = tw_shift;
    a.in_bstride = a.out_bstride = M1 * Wb;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = M1 * Wb;  // masks folded into the slab tables
    a.diag_kind = DG_CPLX;
    return a;
  }
  PassArgs row_args() const {
    PassArgs a{};
    a.ncols = (int)M2;
    a.fft_tw = tw_row.p;
    a.fft_tw2 = tw_row2.p;
    a.in_bstride = a.out_bstride = Hb * M2;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = Hb * M2;
    a.rb_w = (int)Wb;
    a.rb_n = G;
    a.rb_stride = Hb * Wb;
    a.diag_kind = DG_CPLX;
    return a;
  }
  // three-level: COL pass of length Ma inside each slab row (batch = row,
  // batch stride Wb in the block-major slab), four-step twiddles of length
  // M2: W_M2^t = W_M^(M1 t)
  PassArgs mid_args() const {
    PassArgs a{};
    a.ncols = (int)Mb;
    a.fft_tw = tw_mid.p;
    a.fft_tw2 = tw_mid2.p;
    a.tw_lo = tw_lo.p;
    a.tw_hi = tw_hi.p;
    a.tw_shift = tw_shift;
    a.tw_mul = M1;
    a.in_bstride = a.out_bstride = Wb;
    a.nvalid_in = a.nvalid_mid = a.nvalid_out = Hb * M2;
    a.rb_w = (int)Wb;
    a.rb_n = G;
    a.rb_stride = Hb * Wb;
    return a;
  }

  void upload_twiddles() {
    auto up = [&](DBuf<double2>& b, const std::vector<double2>& h) {
      b.alloc(h.size());
      LD_CK(cudaMemcpy(b.p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
    };
    auto stage_tw = [&](int axis, long long L, bool rev) {
      const dev::PassKernel* k = dev::find_pass_kernel(axis, (int)L, PROG_DOUBLE, -1);
      int radix[16];
      for (int s = 0; s < k->nst; ++s) radix[s] = k->radix[rev ? k->nst - 1 - s : s];
      std::vector<double2> t(std::max(1, build_stage_twiddles(radix, k->nst, nullptr)), make_double2(1.0, 0.0));
      build_stage_twiddles(radix, k->nst, t.data());
      return t;
    };
    up(tw_col, stage_tw(AX_COL, M1, false));
    up(tw_col2, stage_tw(AX_COL, M1, true));
    up(tw_row, stage_tw(AX_ROW, three ? Mb : M2, false));
    up(tw_row2, stage_tw(AX_ROW, three ? Mb : M2, true));
    if (three) {
      up(tw_mid, stage_tw(AX_COL, Ma, false));
      up(tw_mid2, stage_tw(AX_COL, Ma, true));
    }
    tw_shift = 0;
    while ((1LL << (2 * tw_shift)) < M) ++tw_shift;
    const long long nlo = 1LL << tw_shift, nhi = (M + nlo - 1) / nlo;
    up(tw_lo, roots(M, nlo, 1));
    up(tw_hi, roots(M, nhi, nlo));
  }

  // M1 x M2 >= 2N-1 with G | M1, G | M2 among the compiled lengths (smallest
  // M within 0.5%, then the lowest measured pass cost, as the unsharded
  // solver chooses); beyond that range the three-level M1 x (Ma x Mb) with
  // G | M1, G | Ma
  void choose_geometry() {
    const long long need = 2 * N - 1;
    long long mmin = -1;
    for (int L1 : dev::pass_lengths(AX_COL))
      for (int L2 : dev::pass_lengths(AX_ROW)) {
        const long long m = (long long)L1 * L2;
        if (m >= need && L1 % G == 0 && L2 % G == 0 && (mmin < 0 || m < mmin)) mmin = m;
      }
    if (mmin > 0) {
      double bc = 0;
      for (int L1 : dev::pass_lengths(AX_COL))
        for (int L2 : dev::pass_lengths(AX_ROW)) {
          const long long m = (long long)L1 * L2;
          if (m < need || L1 % G || L2 % G || (double)m > 1.005 * (double)mmin) continue;
          const double cost = (double)m * (dev::cost_col(L1) + dev::cost_row(L2));
          if (M == 0 || cost < bc) {
            M = m;
            M1 = L1;
            M2 = L2;
            bc = cost;
          }
        }
      three = false;
    } else {
      auto have3 = [&](int L1, int La, int Lb) {
        return L1 <= 4096 && La <= 4096 && Lb <= 4096 && L1 % G == 0 && La % G == 0 &&
               dev::find_pass_kernel(AX_COL, L1, PROG_DOUBLE, -1) && dev::find_pass_kernel(AX_COL, La, PROG_LOADDIAG, -1) &&
               dev::find_pass_kernel(AX_ROW, Lb, PROG_DOUBLE, -1);
      };
      long long m3 = -1;
      for (int L1 : dev::pass_lengths(AX_COL))
        for (int La : dev::pass_lengths(AX_COL))
          for (int Lb : dev::pass_lengths(AX_ROW)) {
            const long long m = (long long)L1 * La * Lb;
            if (m >= need && (m3 < 0 || m < m3) && have3(L1, La, Lb)) m3 = m;
          }
      if (m3 < 0) raise(Errc::unsupported, "no compiled M1 x Ma x Mb >= 2N-1 with G=" + std::to_string(G) + " | M1, Ma");
      double bc = 0;
      for (int L1 : dev::pass_lengths(AX_COL))
        for (int La : dev::pass_lengths(AX_COL))
          for (int Lb : dev::pass_lengths(AX_ROW)) {
            const long long m = (long long)L1 * La * Lb;
            if (m < need || (double)m > 1.005 * (double)m3 || !have3(L1, La, Lb)) continue;
            const double cost = (double)m * (dev::cost_col3(L1) + dev::cost_row3(La, Lb));
            if (M == 0 || cost < bc) {
              M = m;
              M1 = L1;
              Ma = La;
              Mb = Lb;
              bc = cost;
            }
          }
      M2 = Ma * Mb;
      three = true;
    }
    Hb = M1 / G;
    Wb = M2 / G;
  }

  // ---- sharded table build (set_dt): plain forward FFT_M of column slabs
  // column slab `src` of local rank i -> A_i (FFT_M1 down the columns, four-step twiddle)
  void col_forward(int i, const double2* src) {
    PassArgs a = col_args(local[i]);
    a.in = src;
    a.out = rk[i].A.p;
    a.diag_kind = DG_NONE;
    a.post_tw = 1;
    launch(AX_COL, (int)M1, PROG_LOADDIAG, -1, a, Wb);
  }
  // row slab B_i -> `dst` (row slab layout, the order K^ is stored in): FFT_M2 along the rows
  void row_forward(int i, double2* dst) {
    if (three) {
      PassArgs a = mid_args();
      a.in = a.out = rk[i].B.p;
      a.post_tw = 1;
      launch(AX_COL, (int)Ma, PROG_LOADDIAG, -1, a, Mb, Hb);
    }
    PassArgs a = row_args();
    a.in = rk[i].B.p;
    a.out = dst;
    a.diag_kind = DG_NONE;
    if (three) a.rb_w = 0;
    launch(AX_ROW, (int)(three ? Mb : M2), PROG_LOADDIAG, -1, a, three ? Hb * Ma : Hb);
  }
  // peak device bytes this process held in slab buffers during set_dt
  // (tests: it scales as 1/G; no unsharded table is ever allocated)
  size_t table_peak_bytes = 0;
  // asynchronous NCCL failures (a peer died, a network error) surface here
  // instead of as a hang in the next synchronisation: polled after every
  // exchange enqueue and after each step() (SURVEY.md §5 failure detection)
  void check_async() {
    if (!comm) return;
    Nccl& n = Nccl::get();
    if (!n.CommGetAsyncError) return;
    ncclResult_t st = ncclSuccess;
    LD_NCCL(n.CommGetAsyncError(comm, &st));
    if (st != ncclSuccess && st != ncclInProgress)
      raise(Errc::nccl_error, std::string("NCCL asynchronous error: ") + n.GetErrorString(st));
  }

  void exchange(bool col_to_row) {
    const long long blk = Hb * Wb;
    if (rank < 0) {  // virtual ranks: device copies
      for (int g = 0; g < G; ++g)
        for (int h = 0; h < G; ++h) {
          // col->row: A_g block h -> B_h block g ; row->col: B_h block g -> A_g block h
          if (col_to_row)
            LD_CK(cudaMemcpyAsync(rk[h].B.p + g * blk, rk[g].A.p + h * blk, blk * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, stream));
          else
            LD_CK(cudaMemcpyAsync(rk[g].A.p + h * blk, rk[h].B.p + g * blk, blk * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, stream));
        }
      return;
    }
    Nccl& n = Nccl::get();
    const int g = rank;
    Rank& R = rk[0];
    LD_NCCL(n.GroupStart());
    for (int h = 0; h < G; ++h) {
      if (h == g) continue;
      if (col_to_row) {
        LD_NCCL(n.Send(R.A.p + h * blk, 2 * blk, ncclDouble, h, comm, stream));
        LD_NCCL(n.Recv(R.B.p + h * blk, 2 * blk, ncclDouble, h, comm, stream));
      } else {
        LD_NCCL(n.Send(R.B.p + h * blk, 2 * blk, ncclDouble, h, comm, stream));
        LD_NCCL(n.Recv(R.A.p + h * blk, 2 * blk, ncclDouble, h, comm, stream));
      }
    }
    LD_NCCL(n.GroupEnd());
    check_async();
    if (col_to_row)
      LD_CK(cudaMemcpyAsync(R.B.p + g * blk, R.A.p + g * blk, blk * sizeof(double2), cudaMemcpyDeviceToDevice, stream));
    else
      LD_CK(cudaMemcpyAsync(R.A.p + g * blk, R.B.p + g * blk, blk * sizeof(double2), cudaMemcpyDeviceToDevice, stream));
  }

  void col_entry(int i) {
    const int g = local[i];
    PassArgs a = col_args(g);
    a.in = rk[i].S.p;
    a.out = rk[i].A.p;
    a.diag = rk[i].Vh.p;
    a.post_tw = 1;
    launch(AX_COL, (int)M1, PROG_LOADDIAG, -1, a, Wb);
  }
  void col_mid(int i) {
    const int g = local[i];
    PassArgs a = col_args(g);
    a.in = a.out = rk[i].A.p;
    a.diag = rk[i].V.p;
    a.pre_tw = a.post_tw = 1;
    launch(AX_COL, (int)M1, PROG_DOUBLE, +1, a, Wb);
  }
  void col_exit(int i) {
    const int g = local[i];
    PassArgs a = col_args(g);
    a.in = rk[i].A.p;
    a.out = rk[i].S.p;
    a.diag = rk[i].Vh.p;
    a.pre_tw = 1;
    launch(AX_COL, (int)M1, PROG_STOREDIAG, +1, a, Wb);
  }
  // the row side: FFT_M2 . (x K^) . IFFT_M2 on every row of the slab
  void row_mid(int i) {
    if (three) {  // FFT_Ma inside the rows, then x W_M2^(ka*nb)
      PassArgs a = mid_args();
      a.in = a.out = rk[i].B.p;
      a.post_tw = 1;
      launch(AX_COL, (int)Ma, PROG_LOADDIAG, -1, a, Mb, Hb);
    }
    PassArgs a = row_args();
    a.in = a.out = rk[i].B.p;
    a.diag = rk[i].K.p;
    if (three) a.rb_w = 0;  // slab = Hb*Ma contiguous Mb-lines (Mb | Wb); K^ sliced the same way
    launch(AX_ROW, (int)(three ? Mb : M2), PROG_DOUBLE, -1, a, three ? Hb * Ma : Hb);
    if (three) {  // x conj W_M2^(ka*nb), then IFFT_Ma
      PassArgs b = mid_args();
      b.in = b.out = rk[i].B.p;
      b.pre_tw = 1;
      launch(AX_COL, (int)Ma, PROG_STOREDIAG, +1, b, Mb, Hb);
    }
  }

  // rows [k Hc, (k+1) Hc) of every block, one way; on stream `st`
  void exchange_chunk(bool col_to_row, int k, cudaStream_t st) {
    const long long blk = Hb * Wb, Hc = Hb / chunks, off = (long long)k * Hc * Wb, cnt = Hc * Wb;
    if (rank < 0) {
      for (int g = 0; g < G; ++g)
        for (int h = 0; h < G; ++h) {
          if (col_to_row)
            LD_CK(cudaMemcpyAsync(rk[h].B.p + g * blk + off, rk[g].A.p + h * blk + off, cnt * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, st));
          else
            LD_CK(cudaMemcpyAsync(rk[g].A.p + h * blk + off, rk[h].B.p + g * blk + off, cnt * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, st));
        }
      return;
    }
    Nccl& n = Nccl::get();
    const int g = rank;
    Rank& R = rk[0];
    double2* src = col_to_row ? R.A.p : R.B.p;
    double2* dst = col_to_row ? R.B.p : R.A.p;
    LD_NCCL(n.GroupStart());
    for (int h = 0; h < G; ++h) {
      if (h == g) continue;
      LD_NCCL(n.Send(src + h * blk + off, 2 * cnt, ncclDouble, h, comm, st));
      LD_NCCL(n.Recv(dst + h * blk + off, 2 * cnt, ncclDouble, h, comm, st));
    }
    LD_NCCL(n.GroupEnd());
    check_async();
    LD_CK(cudaMemcpyAsync(dst + g * blk + off, src + g * blk + off, cnt * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  }
  // the row side on rows [k Hc, (k+1) Hc) of local rank i's slab
  void row_mid_chunk(int i, int k) {
    const long long Hc = Hb / chunks, off = (long long)k * Hc * Wb;
    double2* B = rk[i].B.p + off;
    if (three) {
      PassArgs a = mid_args();
      a.in = a.out = B;
      a.post_tw = 1;
      launch(AX_COL, (int)Ma, PROG_LOADDIAG, -1, a, Mb, Hc);
      // Mb-lines are contiguous inside a block only: one ROW launch per block
      for (int q = 0; q < G; ++q) {
        PassArgs r = row_args();
        r.rb_w = 0;
        r.in = r.out = B + (long long)q * Hb * Wb;
        r.diag = rk[i].K.p + off + (long long)q * Hb * Wb;
        r.in_bstride = r.out_bstride = Hc * Wb;
        r.nvalid_in = r.nvalid_mid = r.nvalid_out = Hc * Wb;
        launch(AX_ROW, (int)Mb, PROG_DOUBLE, -1, r, Hc * Wb / Mb);
      }
      PassArgs b = mid_args();
      b.in = b.out = B;
      b.pre_tw = 1;
      launch(AX_COL, (int)Ma, PROG_STOREDIAG, +1, b, Mb, Hc);
    } else {
      PassArgs a = row_args();
      a.in = a.out = B;
      a.diag = rk[i].K.p + off;
      launch(AX_ROW, (int)M2, PROG_DOUBLE, -1, a, Hc);
    }
  }
  // exchange -> row passes -> exchange as a pipeline over row chunks: the
  // copies of chunk k+2 (in) and chunk k (out) run on `xstream` under the
  // row passes of chunk k+1 on `stream`
  void row_side_pipelined() {
    const int nl = (int)local.size();
    LD_CK(cudaEventRecord(ev_col, stream));
    LD_CK(cudaStreamWaitEvent(xstream, ev_col, 0));
    auto in = [&](int k) {
      exchange_chunk(true, k, xstream);
      LD_CK(cudaEventRecord(ev_in[k], xstream));
    };
    for (int k = 0; k < std::min(2, chunks); ++k) in(k);
    for (int k = 0; k < chunks; ++k) {
      LD_CK(cudaStreamWaitEvent(stream, ev_in[k], 0));
      for (int i = 0; i < nl; ++i) row_mid_chunk(i, k);
      LD_CK(cudaEventRecord(ev_done[k], stream));
      if (k + 2 < chunks) in(k + 2);
      LD_CK(cudaStreamWaitEvent(xstream, ev_done[k], 0));
      exchange_chunk(false, k, xstream);
    }
    LD_CK(cudaEventRecord(ev_back, xstream));
    LD_CK(cudaStreamWaitEvent(stream, ev_back, 0));
  }
  void setup_chunks(int want) {
    chunks = 1;
    for (int c = std::max(1, want); c >= 1; --c)
      if (Hb % c == 0) {
        chunks = c;
        break;
      }
    if (chunks > 1 && !xstream) {
      LD_CK(cudaStreamCreateWithFlags(&xstream, cudaStreamNonBlocking));
      LD_CK(cudaEventCreateWithFlags(&ev_col, cudaEventDisableTiming));
      LD_CK(cudaEventCreateWithFlags(&ev_back, cudaEventDisableTiming));
    }
    while ((int)ev_in.size() < chunks) {
      cudaEvent_t a, b;
      LD_CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      LD_CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      ev_in.push_back(a);
      ev_done.push_back(b);
    }
  }

  void enqueue_steps(long long n) {
    if (!have_dt) raise(Errc::config_error, "set_dt must be called before stepping");
    if (n <= 0) return;
    const int nl = (int)local.size();
    for (int i = 0; i < nl; ++i) col_entry(i);
    for (long long k = 0; k < n; ++k) {
      if (chunks > 1) {
        row_side_pipelined();
      } else {
        exchange(true);
        for (int i = 0; i < nl; ++i) row_mid(i);
        exchange(false);
      }
      for (int i = 0; i < nl; ++i) {
        if (k + 1 < n)
          col_mid(i);
        else
          col_exit(i);
      }
    }
    LD_CK(cudaGetLastError());
  }

  // sum over this process's slabs of sum |x|^2 (block partials, long double on the host)
  double local_sumsq(const std::vector<const double2*>& xs) {
    const int blocks = 592;
    partial.alloc((size_t)blocks * xs.size() + 1);
    for (size_t i = 0; i < xs.size(); ++i) k_sumsq<<<blocks, 256, 0, stream>>>(xs[i], slab(), partial.p + i * blocks);
    std::vector<double> h((size_t)blocks * xs.size());
    LD_CK(cudaMemcpyAsync(h.data(), partial.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
    LD_CK(cudaStreamSynchronize(stream));
    long double tot = 0;
    for (double x : h) tot += x;
    return (double)tot;
  }
  double allreduce_sum(double v) {
    if (!comm) return v;
    LD_CK(cudaMemcpyAsync(partial.p, &v, sizeof(double), cudaMemcpyHostToDevice, stream));
    LD_NCCL(Nccl::get().AllReduce(partial.p, partial.p, 1, ncclDouble, ncclSum, comm, stream));
    LD_CK(cudaMemcpyAsync(&v, partial.p, sizeof(double), cudaMemcpyDeviceToHost, stream));
    LD_CK(cudaStreamSynchronize(stream));
    return v;
  }
};

// --------------------------------------------------------------- DistSolver
DistSolver::DistSolver(const Lattice& lat, const AntiAliasSet& aa, const ProblemSpec& prob, const DistOptions& opt)
    : p_(std::make_unique<Impl>(lat)) {
  Impl& s = *p_;
  if (lat.rank() != 1) raise(Errc::unsupported, "the sharded solver handles rank-1 lattices");
  if (prob.initial.size() != 1) raise(Errc::invalid_argument, "the sharded solver steps one wave function");
  if (opt.world < 1) raise(Errc::invalid_argument, "world must be >= 1");
  if (opt.rank >= opt.world) raise(Errc::invalid_argument, "rank must be < world");
  if (!aa.norm2.empty() && aa.n_total != lat.n_total()) raise(Errc::spec_mismatch, "anti-aliasing set does not match the lattice");
  s.G = opt.world;
  s.rank = opt.rank;
  s.device = opt.device;
  s.N = lat.n_total();
  s.aa = aa;
  s.prob = prob;
  LD_CK(cudaSetDevice(s.device));
  LD_CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  s.choose_geometry();
  s.upload_twiddles();
  {
    // NCCL ranks overlap the exchanges with the row passes in 4 row chunks;
    // virtual ranks (device copies, nothing to hide) keep one, unless asked
    const char* e = std::getenv("LATTDSE_DIST_CHUNKS");
    s.setup_chunks(e ? std::atoi(e) : (opt.rank >= 0 && opt.world > 1 ? 4 : 1));
  }
  if (s.rank < 0)
    for (int g = 0; g < s.G; ++g) s.local.push_back(g);
  else
    s.local.push_back(s.rank);
  s.rk.resize(s.local.size());
  for (auto& r : s.rk) {
    r.S.alloc((size_t)s.slab());
    LD_CK(cudaMemsetAsync(r.S.p, 0, (size_t)s.slab() * sizeof(double2), s.stream));
  }
  LD_CK(cudaStreamSynchronize(s.stream));
  if (s.rank >= 0 && s.G > 1) {
    if (!opt.nccl_id) raise(Errc::invalid_argument, "NCCL mode needs the rank-0 unique id");
    ncclUniqueId id;
    std::memcpy(&id, opt.nccl_id, sizeof id);
    LD_NCCL(Nccl::get().CommInitRank(&s.comm, s.G, id, s.rank));
  }
}

DistSolver::~DistSolver() {
  if (!p_) return;
  if (p_->stream) cudaStreamSynchronize(p_->stream);
  if (p_->xstream) cudaStreamSynchronize(p_->xstream);
  if (p_->comm) Nccl::get().CommDestroy(p_->comm);
  for (auto e : p_->ev_in) cudaEventDestroy(e);
  for (auto e : p_->ev_done) cudaEventDestroy(e);
  if (p_->ev_col) cudaEventDestroy(p_->ev_col);
  if (p_->ev_back) cudaEventDestroy(p_->ev_back);
  if (p_->xstream) cudaStreamDestroy(p_->xstream);
  if (p_->stream) cudaStreamDestroy(p_->stream);
}

void DistSolver::nccl_unique_id(void* out128) {
  ncclUniqueId id;
  LD_NCCL(Nccl::get().GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof id);
}

// The propagator tables (K^ in ROW-pass order, V, V^(1/2)), slab by slab:
// nothing of size M or N complex is ever allocated, so a rank's peak memory
// is its slabs (1/G of the problem) plus the 2 N-byte norm index.
//   V, V^(1/2): the potential sampled at the slab's own points (sampling.cuh,
//       the same point function as the unsharded solver: identical bits);
//   K^ = FFT_M(wrap(k)) / M, k = F_N^-1(D / N):
//     1. B2^ = FFT_M(even wrap of the chirp) / M with the solver's own
//        distributed forward transform (COL pass, exchange, ROW pass);
//     2. k by Bluestein: (D/N . conj chirp) -> FFT_M -> x B2^ -> IFFT_M ->
//        x conj chirp, i.e. one Strang-shaped round trip (COL entry,
//        exchange, ROW mid, exchange, COL exit) with these tables;
//     3. F = FFT_M(zero-padded k), then K^ = (F + w (F - k[0])) / M pointwise
//        (k_khat_finish): the periodic wrap is a shift by M - N, a phase in
//        the spectrum, so no data crosses slabs; k[0] is one all-reduce.
// LATTDSE_DIST_TABLES=full keeps the round-1 path (a transient unsharded
// Solver whose tables are sliced) for A/B runs; dimensions beyond the device
// sampler's limit use it too.
void DistSolver::set_dt(double dt) {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  s.have_dt = false;
  const char* mode = std::getenv("LATTDSE_DIST_TABLES");
  if ((mode && std::string(mode) == "full") || s.lat.dim() > kMaxDimDev) {
    set_dt_full_table(dt);
    return;
  }
  for (auto& r : s.rk) {
    r.A.release();
    r.B.release();
    r.V.release();
    r.Vh.release();
    r.K.release();
  }
  const long long slab = s.slab();
  const int nl = (int)s.local.size();
  const int g1 = s.grid1d(slab);
  size_t free0 = 0, free1 = 0, total_b = 0;
  LD_CK(cudaMemGetInfo(&free0, &total_b));
  // norm index (2 N bytes, replicated) and the kinetic LUT exp(-i eps dt 2 pi^2 s) / N
  DBuf<unsigned short> nidx;
  nidx.alloc((size_t)s.N);
  std::uint32_t max_norm2 = s.aa.max_norm2;
  if (s.aa.norm2.empty()) {
    max_norm2 = dev::aaset_norms_device(s.lat, nidx.p, s.stream);
  } else {
    std::vector<unsigned short> ni((size_t)s.N);
    for (long long c = 0; c < s.N; ++c) ni[(size_t)c] = (unsigned short)s.aa.norm2[(size_t)c];
    LD_CK(cudaMemcpy(nidx.p, ni.data(), ni.size() * sizeof(unsigned short), cudaMemcpyHostToDevice));
  }
  if (max_norm2 > 65534) raise(Errc::unsupported, "||h||^2 above 65535 does not fit the uint16 norm index");
  std::vector<double2> lut(max_norm2 + 1);
  for (std::uint32_t q = 0; q <= max_norm2; ++q) {
    long double a = -(long double)s.prob.eps * (long double)dt * 2.0L * kPiL * kPiL * (long double)q;
    long double r = fmodl(a, 2.0L * kPiL);
    lut[q] = make_double2((double)(cosl(r) / (long double)s.N), (double)(sinl(r) / (long double)s.N));
  }
  DBuf<double2> dlut;
  dlut.alloc(lut.size());
  LD_CK(cudaMemcpy(dlut.p, lut.data(), lut.size() * sizeof(double2), cudaMemcpyHostToDevice));

  std::vector<DBuf<double2>> T(nl), C(nl);  // B2^ (row slab) and a column-slab scratch per local rank
  for (int i = 0; i < nl; ++i) {
    s.rk[i].A.alloc((size_t)slab);
    s.rk[i].B.alloc((size_t)slab);
    s.rk[i].K.alloc((size_t)slab);
    T[i].alloc((size_t)slab);
    C[i].alloc((size_t)slab);
  }
  // per-rank peak of this build: everything allocated since entry (work slabs
  // A, B, K^, B2^, scratch, norm index, LUT) plus the state slab held before
  LD_CK(cudaMemGetInfo(&free1, &total_b));
  s.table_peak_bytes = (free0 > free1 ? free0 - free1 : 0) / (size_t)nl + (size_t)slab * sizeof(double2);
  const double invM = 1.0 / (double)s.M;
  auto chirp = [&](int what, int i, double scale, double2* out) {
    k_slab_chirp<<<g1, 256, 0, s.stream>>>(what, s.N, s.M, s.M1, s.M2, s.Wb, s.local[i] * s.Wb, scale, nidx.p, dlut.p, out);
    LD_CK(cudaGetLastError());
  };
  // 1. B2^ = FFT_M(even wrap of c) / M
  for (int i = 0; i < nl; ++i) {
    chirp(0, i, invM, C[i].p);
    s.col_forward(i, C[i].p);
  }
  s.exchange(true);
  for (int i = 0; i < nl; ++i) s.row_forward(i, T[i].p);
  // 2. k = conj c . IFFT_M(B2^ . FFT_M(D/N . conj c)): conj chirp parked in K_i (column-slab sized)
  for (int i = 0; i < nl; ++i) {
    chirp(2, i, 1.0, C[i].p);
    chirp(1, i, 1.0, s.rk[i].K.p);
    s.col_forward(i, C[i].p);
  }
  s.exchange(true);
  for (int i = 0; i < nl; ++i) {
    double2* keep = s.rk[i].K.p;
    s.rk[i].K.p = T[i].p;  // row_mid multiplies by K_i: B2^ for this round trip
    s.row_mid(i);
    s.rk[i].K.p = keep;
  }
  s.exchange(false);
  for (int i = 0; i < nl; ++i) {
    PassArgs a = s.col_args(s.local[i]);
    a.in = s.rk[i].A.p;
    a.out = C[i].p;
    a.diag = s.rk[i].K.p;
    a.pre_tw = 1;
    s.launch(AX_COL, (int)s.M1, PROG_STOREDIAG, +1, a, s.Wb);
  }
  // k[0]: first element of global column 0 (rank 0), summed over the ranks
  double k0[2] = {0.0, 0.0};
  for (int i = 0; i < nl; ++i)
    if (s.local[i] == 0) {
      LD_CK(cudaMemcpyAsync(k0, C[i].p, sizeof(double2), cudaMemcpyDeviceToHost, s.stream));
      LD_CK(cudaStreamSynchronize(s.stream));
    }
  k0[0] = s.allreduce_sum(k0[0]);
  k0[1] = s.allreduce_sum(k0[1]);
  // 3. F = FFT_M(k zero-padded) into K_i, then the wrap as a spectral phase
  for (int i = 0; i < nl; ++i) s.col_forward(i, C[i].p);
  s.exchange(true);
  for (int i = 0; i < nl; ++i) {
    s.row_forward(i, s.rk[i].K.p);
    k_khat_finish<<<g1, 256, 0, s.stream>>>(s.rk[i].K.p, make_double2(k0[0], k0[1]), s.N, s.M, s.M1, s.Hb, s.Wb, s.G,
                                            s.local[i] * s.Hb, s.three ? s.Ma : 0, s.three ? s.Mb : 1, invM);
    LD_CK(cudaGetLastError());
  }
  LD_CK(cudaStreamSynchronize(s.stream));
  T.clear();
  C.clear();
  nidx.release();
  // V, V^(1/2) at the slab's own points
  R1Points P{};
  P.N = s.N;
  P.d = s.lat.dim();
  const auto steps = s.lat.numerator_steps();
  for (int j = 0; j < P.d; ++j) P.z[j] = steps[0][j];
  DBuf<double> da, db;
  da.alloc(std::max<size_t>(1, s.prob.potential.a.size()));
  db.alloc(std::max<size_t>(1, s.prob.potential.b.size()));
  LD_CK(cudaMemcpy(da.p, s.prob.potential.a.data(), s.prob.potential.a.size() * sizeof(double), cudaMemcpyHostToDevice));
  if (!s.prob.potential.b.empty())
    LD_CK(cudaMemcpy(db.p, s.prob.potential.b.data(), s.prob.potential.b.size() * sizeof(double), cudaMemcpyHostToDevice));
  for (int i = 0; i < nl; ++i) {
    auto& r = s.rk[i];
    r.V.alloc((size_t)slab);
    r.Vh.alloc((size_t)slab);
    k_slab_vphase<<<g1, 256, 0, s.stream>>>(P, da.p, db.p, -dt / s.prob.eps, s.M1, s.M2, s.Wb, s.local[i] * s.Wb, r.V.p);
    k_slab_vphase<<<g1, 256, 0, s.stream>>>(P, da.p, db.p, -dt / (2.0 * s.prob.eps), s.M1, s.M2, s.Wb, s.local[i] * s.Wb, r.Vh.p);
    LD_CK(cudaGetLastError());
  }
  LD_CK(cudaStreamSynchronize(s.stream));
  s.have_dt = true;
}

// Round-1 path: a transient unsharded Solver, forced to the same geometry,
// builds the tables; they are sliced into the slabs (staged through host
// memory when they do not fit next to it).
void DistSolver::set_dt_full_table(double dt) {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  s.have_dt = false;
  for (auto& r : s.rk) {
    r.A.release();
    r.B.release();
    r.V.release();
    r.Vh.release();
    r.K.release();
  }
  const long long slab = s.slab();
  const size_t sb = (size_t)slab * sizeof(double2);
  std::vector<std::vector<double2>> host;  // staged [rank][table] when the slabs do not fit
  size_t free_entry = 0, total_entry = 0;
  LD_CK(cudaMemGetInfo(&free_entry, &total_entry));
  {
    SolverOptions so;
    so.device = s.device;
    so.force_M1 = s.M1;
    so.force_M2 = s.M2;
    so.force_M2a = s.three ? s.Ma : 0;
    so.group = 1;
    Solver full(s.lat, s.aa, s.prob, so);
    full.set_dt(dt);
    {
      size_t f1 = 0, tb = 0;
      LD_CK(cudaMemGetInfo(&f1, &tb));
      s.table_peak_bytes = (free_entry > f1 ? free_entry - f1 : 0) + (size_t)s.slab() * sizeof(double2);
    }
    const auto* K = (const double2*)full.device_table(0);
    const auto* V = (const double2*)full.device_table(1);
    const auto* Vh = (const double2*)full.device_table(2);
    size_t free_b = 0, total_b = 0;
    LD_CK(cudaMemGetInfo(&free_b, &total_b));
    const bool direct = (double)free_b > 3.0 * (double)sb * (double)s.local.size() + 2e9;
    DBuf<double2> t;
    if (!direct) {
      t.alloc((size_t)slab);
      host.assign(s.local.size(), std::vector<double2>((size_t)slab * 3));
    }
    for (size_t i = 0; i < s.local.size(); ++i) {
      const int g = s.local[i];
      auto& r = s.rk[i];
      double2* dst[3];
      if (direct) {
        r.V.alloc((size_t)slab);
        r.Vh.alloc((size_t)slab);
        r.K.alloc((size_t)slab);
        dst[0] = r.V.p;
        dst[1] = r.Vh.p;
        dst[2] = r.K.p;
      } else {
        dst[0] = dst[1] = dst[2] = t.p;
      }
      for (int w = 0; w < 3; ++w) {
        if (w < 2)
          k_colslab<<<s.grid1d(slab), 256, 0, s.stream>>>(w == 0 ? V : Vh, s.N, s.M1, s.M2, s.Wb, g * s.Wb, dst[w]);
        else
          k_rowblk<<<s.grid1d(slab), 256, 0, s.stream>>>(K, s.M2, s.Hb, s.Wb, s.G, g * s.Hb, dst[w]);
        LD_CK(cudaGetLastError());
        if (!direct)
          LD_CK(cudaMemcpyAsync(host[i].data() + (size_t)w * slab, t.p, sb, cudaMemcpyDeviceToHost, s.stream));
      }
    }
    LD_CK(cudaStreamSynchronize(s.stream));
  }  // table solver and staging buffer freed
  for (size_t i = 0; i < s.local.size(); ++i) {
    auto& r = s.rk[i];
    if (!host.empty()) {
      r.V.alloc((size_t)slab);
      r.Vh.alloc((size_t)slab);
      r.K.alloc((size_t)slab);
      LD_CK(cudaMemcpy(r.V.p, host[i].data(), sb, cudaMemcpyHostToDevice));
      LD_CK(cudaMemcpy(r.Vh.p, host[i].data() + slab, sb, cudaMemcpyHostToDevice));
      LD_CK(cudaMemcpy(r.K.p, host[i].data() + 2 * slab, sb, cudaMemcpyHostToDevice));
      std::vector<double2>().swap(host[i]);
    }
    r.A.alloc((size_t)slab);
    r.B.alloc((size_t)slab);
  }
  LD_CK(cudaGetLastError());
  s.have_dt = true;
}

void DistSolver::set_state(const std::complex<double>* samples) {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  s.tmp.alloc(s.N);
  LD_CK(cudaMemcpyAsync(s.tmp.p, samples, s.N * sizeof(double2), cudaMemcpyHostToDevice, s.stream));
  const long long slab = s.slab();
  for (size_t i = 0; i < s.local.size(); ++i)
    k_colslab<<<s.grid1d(slab), 256, 0, s.stream>>>(s.tmp.p, s.N, s.M1, s.M2, s.Wb, s.local[i] * s.Wb, s.rk[i].S.p);
  LD_CK(cudaStreamSynchronize(s.stream));
  s.tmp.release();
}

// g sampled on the device straight into the slabs (sampling.cuh, the same
// point function as the unsharded solver), normalised by the all-rank sum
void DistSolver::discretize_initial() {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  problems::Initial& g = s.prob.initial[0];
  const int d = s.lat.dim();
  if (d > kMaxDimDev) {  // host sampling fallback for very high dimension
    auto gv = problems::sample_g(s.lat, g);
    set_state(gv.data());
    return;
  }
  R1Points P{};
  P.N = s.N;
  P.d = d;
  const auto steps = s.lat.numerator_steps();
  for (int j = 0; j < d; ++j) P.z[j] = steps[0][j];
  DBuf<double> dc;
  DBuf<int> dp;
  dc.alloc(d);
  dp.alloc(d);
  LD_CK(cudaMemcpy(dc.p, g.c.data(), d * sizeof(double), cudaMemcpyHostToDevice));
  LD_CK(cudaMemcpy(dp.p, g.p.data(), d * sizeof(int), cudaMemcpyHostToDevice));
  std::vector<const double2*> xs;
  for (size_t i = 0; i < s.local.size(); ++i) {
    k_slab_sample_g<<<s.grid1d(s.slab()), 256, 0, s.stream>>>(P, dc.p, dp.p, 1.0 / (2.0 * g.sigma * g.sigma), s.M1, s.M2,
                                                              s.Wb, s.local[i] * s.Wb, s.rk[i].S.p);
    LD_CK(cudaGetLastError());
    xs.push_back(s.rk[i].S.p);
  }
  const double tot = s.allreduce_sum(s.local_sumsq(xs));
  if (!(tot > 0)) raise(Errc::non_normalizable, "initial condition vanishes on the lattice");
  const double C = 1.0 / std::sqrt(tot / (double)s.N);
  g.C = C;
  for (size_t i = 0; i < s.local.size(); ++i) k_scale_slab<<<s.grid1d(s.slab()), 256, 0, s.stream>>>(s.rk[i].S.p, s.slab(), C);
  LD_CK(cudaStreamSynchronize(s.stream));
  LD_CK(cudaGetLastError());
}

void DistSolver::get_state(std::complex<double>* samples) {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  s.tmp.alloc(s.N);
  LD_CK(cudaMemcpyAsync(s.tmp.p, samples, s.N * sizeof(double2), cudaMemcpyHostToDevice, s.stream));
  const long long slab = s.slab();
  for (size_t i = 0; i < s.local.size(); ++i)
    k_slab2nat<<<s.grid1d(slab), 256, 0, s.stream>>>(s.rk[i].S.p, s.N, s.M1, s.M2, s.Wb, s.local[i] * s.Wb, s.tmp.p);
  LD_CK(cudaMemcpyAsync(samples, s.tmp.p, s.N * sizeof(double2), cudaMemcpyDeviceToHost, s.stream));
  LD_CK(cudaStreamSynchronize(s.stream));
}

void DistSolver::step(std::int64_t nsteps) {
  LD_CK(cudaSetDevice(p_->device));
  p_->enqueue_steps(nsteps);
  LD_CK(cudaStreamSynchronize(p_->stream));
  p_->check_async();
}

double DistSolver::time_steps(std::int64_t nsteps) {
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
  return ms;
}

double DistSolver::l2_norm() {
  Impl& s = *p_;
  LD_CK(cudaSetDevice(s.device));
  std::vector<const double2*> xs;
  for (auto& r : s.rk) xs.push_back(r.S.p);
  return std::sqrt(s.allreduce_sum(s.local_sumsq(xs)) / (double)s.N);
}

std::int64_t DistSolver::M() const { return p_->M; }
std::int64_t DistSolver::M1() const { return p_->M1; }
std::int64_t DistSolver::M2() const { return p_->M2; }
std::int64_t DistSolver::Ma() const { return p_->three ? p_->Ma : 0; }
int DistSolver::world() const { return p_->G; }
double DistSolver::table_peak_bytes() const { return (double)p_->table_peak_bytes; }
double DistSolver::exchange_bytes_per_rank() const {
  return 16.0 * (double)p_->Hb * (double)p_->Wb * (double)(p_->G - 1);
}

}  // namespace lattdse
