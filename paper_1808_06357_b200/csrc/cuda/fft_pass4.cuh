// pass4: the per-step PROG_DOUBLE passes (strang_step, SPEC.md:336-344;
// Algorithm 1) of the plain layouts, rewritten lean.
//
// Why (profiles/r2base, ncu of the config-3 step kernels): the generic v1
// kernels (fft_pass.cuh) spend 40% of their issue slots on index / mask /
// layout arithmetic that the per-step passes never need (sharded slabs,
// Good-Thomas order, per-element 64-bit masks, swizzled slots), their fused
// mid stage runs on 2 of 5 warps while the others wait at the barrier, and
// every CTA exposes one HBM round trip before its first butterfly.  Here:
//  - plain layout only: every address of a task is ONE base plus
//    compile-time offsets (shared memory) or a fixed stride (global);
//  - masks reduced to one comparison per element against a per-line row
//    limit (the mid mask j < N of the circulant embedding), none on the
//    load / store side (full tiles only, checked on the host);
//  - four-step twiddles W_M^(col * (j + r T)) = W^(col j) * (W^(col T))^r with
//    the R powers of every column computed once per CTA into shared memory;
//  - LPT lines per thread share the stage twiddles and the index math;
//  - each CTA prefetches into L2 the tile a later CTA (pf tiles ahead in
//    launch order) will load, so that load is an L2 hit, not an HBM trip.
// Everything else (single-transform programs, sharded / three-level inner
// passes, partial tiles) stays on the v1 kernels.
#pragma once

#include "fft_pass.cuh"

namespace lattdse_dev {

// Stage sequence of a pass: positions 0 .. 2 nst - 2 (forward plan stages
// 0 .. nst-1, the last of them fused with the reversed plan's stage 0, then
// reversed plan stages 1 .. nst-1). The buffer an inner stage (radix R,
// Ns > 1) writes is skewed by c slots per output block of Ns R elements,
// c = Ns (1 - R) mod 8: consecutive tasks then fall into consecutive
// 16-byte bank groups across block boundaries (unskewed, a run of Ns
// consecutive slots is followed by a jump of Ns R - Ns + 1 slots, and a
// quarter warp straddling it hits a bank group twice: 1.5-1.9 wavefronts
// per access for Ns = 9, 10; tools/p4_conflicts.py). Block-aligned skews
// keep every access of a task affine in r: the writer adds c (j / Ns) to
// its base, the reader (T a multiple of the block) c (j / P) to its base
// and c T / P to its stride.
template <int L> struct P4Seq {
  static constexpr int nst = Plan<L>::nst;
  static constexpr int R(int q) { return q < nst ? PlanX<L, false>::radix(q) : PlanX<L, true>::radix(q - nst + 1); }
  static constexpr int Ns(int q) { return q < nst ? PlanX<L, false>::ns(q) : PlanX<L, true>::ns(q - nst + 1); }
  static constexpr bool inner(int q) { return q > 0 && q != nst - 1 && q < 2 * nst - 2; }
  static constexpr int P(int q) { return inner(q) ? Ns(q) * R(q) : 0; }  // skew period of the buffer position q writes
  static constexpr int C(int q) { return inner(q) ? ((Ns(q) * (1 - R(q))) % 8 + 8) % 8 : 0; }
  // Power-of-two style plans (first or last radix a multiple of 4): their
  // Ns = 1 stage writes j R + r collide 4- to 8-fold, so every buffer is
  // swizzled by one slot per 16, phys(i) = i + i / 16 (as the generic kernels
  // do). Addresses stay "base + compile-time offset": phys(base + off) =
  // phys(base) + phys(off) whenever the low four bits do not carry, which
  // holds for every access of such a plan -- reads j + r T with 16 | T,
  // writes (j - k) R + k + r Ns with Ns = 1 and R in {4, 8, 16} (base a
  // multiple of R, off = r < R), 16 | Ns, or Ns = 8 with k < 8 (off = 8 r).
  static constexpr bool swz = (R(0) % 4 == 0 || R(nst - 1) % 4 == 0) && L >= 64;
  static constexpr bool swz_ok() {
    if (!swz) return true;
    for (int q = 0; q < 2 * nst - 1; ++q) {
      const int r = R(q), ns = Ns(q), t = L / r;
      if (q > 0 && t % 16 != 0) return false;                                  // reads of stage q
      if (C(q) != 0) return false;                                              // never together with the skew
      if (q != nst - 1 && q != 2 * nst - 2) {                                   // Stockham write of stage q
        if (ns == 1 ? !(r == 4 || r == 8 || r == 16) : !(ns % 16 == 0 || ns == 8)) return false;
      }
    }
    const int rl = R(nst - 1);  // the fused mid stage writes with the reversed plan's stage 0 (Ns = 1)
    return rl == 4 || rl == 8 || rl == 16;
  }
  static constexpr int ph(int i) { return swz ? i + i / 16 : i; }
  static constexpr int extent() {
    int m = ph(L - 1) + 1;
    for (int q = 0; q < 2 * nst - 1; ++q)
      if (P(q) > 0 && L + C(q) * (L / P(q)) > m) m = L + C(q) * (L / P(q));
    return m;
  }
};

// PP: two stage buffers (one barrier per stage) instead of one in place (two)
template <int AXIS, int L, int B, int LPT, bool PP> struct P4Geom {
  static_assert(B % LPT == 0, "lines per thread must divide the tile");
  static constexpr int BG = B / LPT;  // line groups: a thread owns lines bg, bg + BG, ...
  static constexpr int L0 = P4Seq<L>::extent();
  // COL tasks run line-fastest across a warp: pad the line stride so the BG
  // lines of a quarter warp fall into distinct 16-byte bank groups
  static constexpr int pad() {
    if (AXIS == AX_ROW || BG == 1) return 0;
    const int want = BG == 2 ? 4 : (BG == 4 ? 2 : 1);
    return ((want - L0 % 8) % 8 + 8) % 8;
  }
  static constexpr int LS = L0 + pad();
  static constexpr int tile = B * LS;
  static constexpr bool pp = PP;
  static constexpr int R0 = Plan<L>::radix(0);
  static constexpr int Rl = Plan<L>::radix(Plan<L>::nst - 1);
  static constexpr int tw_slots = AXIS == AX_COL ? B * (R0 > Rl ? R0 : Rl) : 0;  // column twiddle powers (first or last radix)
  static constexpr int bytes = (pp ? 2 : 1) * tile * 16 + tw_slots * 16;
};

#if defined(__CUDACC__)

template <int AXIS, int L, int B, int LPT, bool PP, int NT, int SIGN1, bool TW, int DK> struct Pass4 {
  using G = P4Geom<AXIS, L, B, LPT, PP>;
  using SQ = P4Seq<L>;
  static constexpr int BG = G::BG, LS = G::LS, nst = Plan<L>::nst;
  static_assert(nst >= 2, "pass4 needs at least two stages");
  static_assert(P4Seq<L>::swz_ok(), "plan needs a swizzle this kernel cannot keep affine");

  const PassArgs& a;
  double2* sm;   // buffer 0; buffer 1 at sm + tile when ping-ponging
  double2* twp;  // [B][R0] powers of the column twiddles (COL, TW)
  const double2* gin;
  double2* gout;
  int line0;
  long long twm = 1;  // four-step twiddles of a length M / twm (rows of a three-level view): W_M^(twm t)

  __device__ __forceinline__ static int pb(int x) { return SQ::swz ? x + (x >> 4) : x; }  // swizzled runtime base
  template <int P_, int C_> __device__ __forceinline__ static int skew(int j) {
    if constexpr (C_ == 0) return 0;
    else return C_ * (j / P_);
  }
  __device__ __forceinline__ double2* buf(int p) const { return (G::pp && (p & 1)) ? sm + G::tile : sm; }
  __device__ __forceinline__ static void map(int q, int T, int& bg, int& j) {
    if (AXIS == AX_ROW) {
      bg = q / T;
      j = q - bg * T;
    } else {
      bg = q % BG;
      j = q / BG;
    }
  }
  __device__ __forceinline__ double2 twid(long long t) const {
    const long long mask = (1LL << a.tw_shift) - 1;
    return c_mul(__ldg(a.tw_hi + (t >> a.tw_shift)), __ldg(a.tw_lo + (t & mask)));
  }
  // global element (line b, index i): position and its stride in r
  __device__ __forceinline__ long long gpos(int b, int j) const {
    return AXIS == AX_ROW ? (long long)(line0 + b) * L + j : (long long)j * a.ncols + (line0 + b);
  }
  // mid mask by line: element i of line b is live iff i < mid_limit(b).
  // COL: i*ncols + col < nvalid_mid with mid_rb = nvalid_mid / ncols and
  // mid_cb = nvalid_mid % ncols from the host; ROW: row*L + i < nvalid_mid.
  __device__ __forceinline__ int mid_limit(int b) const {
    if (AXIS == AX_COL) return a.mid_rb + ((line0 + b) < a.mid_cb ? 1 : 0);
    const long long rem = a.nvalid_mid - (long long)(line0 + b) * L;
    return rem >= L ? L : (rem < 0 ? 0 : (int)rem);
  }
  __device__ __forceinline__ long long gstep(int T) const { return AXIS == AX_ROW ? (long long)T : (long long)T * a.ncols; }

  // w^r, r < R, applied to v (conjugated for the inverse direction)
  template <int R, int SIGN> __device__ __forceinline__ static void apply_pow(const Pow<R>& pw, double2 (&v)[R]) {
    sfor<R>([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      if constexpr (r > 0) {
        const double2 w = pw.template get<r>();
        v[r] = SIGN < 0 ? c_mul(v[r], w) : c_mulc(v[r], w);
      }
    });
  }
  template <int R, int Ns, bool REV, int S> __device__ __forceinline__ Pow<R> stage_pow(int k) const {
    using P = PlanX<L, REV>;
    const double2* tw = (REV ? a.fft_tw2 : a.fft_tw) + P::tw_offset(S) + k;
    Pow<R> pw;
    pw.init(__ldg(tw), R > 4 ? __ldg(tw + 3 * Ns) : make_double2(1.0, 0.0),
            R > 16 ? __ldg(tw + 15 * Ns) : make_double2(1.0, 0.0));
    return pw;
  }
  // four-step twiddles of task j, line b (elements j + r T0): base * twp[b][r]
  template <int R, bool CONJ> __device__ __forceinline__ void fourstep(int b, int j, double2 (&v)[R]) const {
    const double2 base = twid((long long)(a.col_off + line0 + b) * twm * j);
    const double2* p = twp + b * R;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2 w = r == 0 ? base : c_mul(base, p[r]);
      v[r] = CONJ ? c_mulc(v[r], w) : c_mul(v[r], w);
    }
  }

  // ---- stage 0 of the first transform: global -> (conj four-step) -> DFT -> smem
  template <bool PRE = TW> __device__ __forceinline__ void first_stage(int tid) const {
    using P = PlanX<L, false>;
    constexpr int R = P::radix(0), T = L / R, TASKS = BG * T, TPT = (TASKS + NT - 1) / NT;
    double2 v[TPT][LPT][R];
    int bgs[TPT], js[TPT];
    const long long st = gstep(T);
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      map(q, T, bgs[t], js[t]);
#pragma unroll
      for (int l = 0; l < LPT; ++l) {
        const double2* p = gin + gpos(bgs[t] + l * BG, js[t]);
#pragma unroll
        for (int r = 0; r < R; ++r) v[t][l][r] = p[r * st];
      }
    }
    if (PRE) __syncthreads();  // twp ready (the loads above are already in flight)
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
#pragma unroll
      for (int l = 0; l < LPT; ++l) {
        if (PRE) fourstep<R, true>(bgs[t] + l * BG, js[t], v[t][l]);
        DFT<R, SIGN1>::run(v[t][l]);
        double2* o = buf(1) + (bgs[t] + l * BG) * LS + pb(js[t] * R);
#pragma unroll
        for (int r = 0; r < R; ++r) o[SQ::ph(r)] = v[t][l][r];
      }
    }
  }

  // ---- inner stage S (smem -> twiddle -> DFT -> smem) at sequence position Q
  template <int S, bool REV, int SIGN, int Q> __device__ __forceinline__ void inner_stage(int tid) const {
    using P = PlanX<L, REV>;
    constexpr int R = P::radix(S), Ns = P::ns(S), T = L / R, TASKS = BG * T, TPT = (TASKS + NT - 1) / NT;
    static_assert(R == SQ::R(Q) && Ns == SQ::Ns(Q), "sequence position");
    constexpr int Pr = SQ::P(Q - 1), Cr = SQ::C(Q - 1), Tr = Cr ? T + Cr * (T / Pr) : T;  // skew of the buffer read
    constexpr int Cw = SQ::C(Q);                                                          // and of the one written
    static_assert(Cr == 0 || T % Pr == 0, "reader stride spans whole skew blocks");
    double2 v[TPT][LPT][R];
    int bgs[TPT], js[TPT];
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      map(q, T, bgs[t], js[t]);
#pragma unroll
      for (int l = 0; l < LPT; ++l) {
        const double2* p = buf(Q) + (bgs[t] + l * BG) * LS + pb(js[t]) + skew<Pr, Cr>(js[t]);
#pragma unroll
        for (int r = 0; r < R; ++r) v[t][l][r] = p[SQ::ph(r * Tr)];
      }
    }
    if (!G::pp) __syncthreads();  // in place: every read before any write
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      const int j = js[t], k = j % Ns;
      const Pow<R> pw = stage_pow<R, Ns, REV, S>(k);
#pragma unroll
      for (int l = 0; l < LPT; ++l) {
        apply_pow<R, SIGN>(pw, v[t][l]);
        DFT<R, SIGN>::run(v[t][l]);
        double2* o = buf(Q + 1) + (bgs[t] + l * BG) * LS + pb((j - k) * R + k) + skew<Ns, Cw>(j);
#pragma unroll
        for (int r = 0; r < R; ++r) o[SQ::ph(r * Ns)] = v[t][l][r];
      }
    }
  }

  // diagonal coefficients of elements j + r T of line b (zero where masked)
  template <int R, int T> __device__ __forceinline__ void diag_fetch(int b, int j, double2 (&dg)[R]) const {
    const long long p0 = gpos(b, j), st = gstep(T);
    const int lim = mid_limit(b);
    const double2 zero = make_double2(0.0, 0.0);
    if (DK == DG_CPLX) {
#pragma unroll
      for (int r = 0; r < R; ++r) dg[r] = (j + r * T < lim) ? __ldg(a.diag + p0 + r * st) : zero;
    } else if (DK == DG_LUT16) {
      const unsigned short* ix = (const unsigned short*)a.diag_idx;
      unsigned short id[R];
#pragma unroll
      for (int r = 0; r < R; ++r) id[r] = (j + r * T < lim) ? __ldg(ix + p0 + r * st) : (unsigned short)0xFFFF;
#pragma unroll
      for (int r = 0; r < R; ++r) dg[r] = id[r] != 0xFFFF ? __ldg(a.lut + id[r]) : zero;
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) dg[r] = (j + r * T < lim) ? make_double2(1.0, 0.0) : zero;
    }
  }

  // ---- fused middle: last stage of T1, x diag, first stage of T2 (reversed plan)
  template <int Q> __device__ __forceinline__ void mid_stage(int tid) const {
    using P = PlanX<L, false>;
    constexpr int S = nst - 1, R = P::radix(S), Ns = P::ns(S), T = L / R, TASKS = BG * T, TPT = (TASKS + NT - 1) / NT;
    static_assert(T == Ns, "last stage covers j + r*T");
    constexpr int Pr = SQ::P(Q - 1), Cr = SQ::C(Q - 1), Tr = Cr ? T + Cr * (T / Pr) : T;
    static_assert(Cr == 0 || T % Pr == 0, "reader stride spans whole skew blocks");
    double2 v[TPT][LPT][R];
    int bgs[TPT], js[TPT];
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      map(q, T, bgs[t], js[t]);
#pragma unroll
      for (int l = 0; l < LPT; ++l) {
        const double2* p = buf(Q) + (bgs[t] + l * BG) * LS + pb(js[t]) + skew<Pr, Cr>(js[t]);
#pragma unroll
        for (int r = 0; r < R; ++r) v[t][l][r] = p[SQ::ph(r * Tr)];
      }
    }
    if (!G::pp) __syncthreads();
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      const int j = js[t];
      const Pow<R> pw = stage_pow<R, Ns, false, S>(j);
#pragma unroll
      for (int l = 0; l < LPT; ++l) {
        const int b = bgs[t] + l * BG;
        double2 dg[R];
        diag_fetch<R, T>(b, j, dg);
        apply_pow<R, SIGN1>(pw, v[t][l]);
        DFT<R, SIGN1>::run(v[t][l]);
#pragma unroll
        for (int r = 0; r < R; ++r) v[t][l][r] = c_mul(v[t][l][r], dg[r]);
        DFT<R, -SIGN1>::run(v[t][l]);  // stage 0 of the reversed plan (Ns = 1)
        double2* o = buf(Q + 1) + b * LS + pb(j * R);
#pragma unroll
        for (int r = 0; r < R; ++r) o[SQ::ph(r)] = v[t][l][r];
      }
    }
  }

  // ---- last stage of the second transform: smem -> twiddle -> DFT -> four-step -> global
  template <int Q> __device__ __forceinline__ void last_stage(int tid) const {
    using P = PlanX<L, true>;
    constexpr int S = nst - 1, R = P::radix(S), Ns = P::ns(S), T = L / R, TASKS = BG * T, TPT = (TASKS + NT - 1) / NT;
    static_assert(T == Ns && R == G::R0, "last stage of the reversed plan mirrors stage 0");
    constexpr int Pr = SQ::P(Q - 1), Cr = SQ::C(Q - 1), Tr = Cr ? T + Cr * (T / Pr) : T;
    static_assert(Cr == 0 || T % Pr == 0, "reader stride spans whole skew blocks");
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      int bg, j;
      map(q, T, bg, j);
      const Pow<R> pw = stage_pow<R, Ns, true, S>(j);
      const long long st = gstep(T);
#pragma unroll
      for (int l = 0; l < LPT; ++l) {
        double2 v[R];
        const double2* p = buf(Q) + (bg + l * BG) * LS + pb(j) + skew<Pr, Cr>(j);
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = p[SQ::ph(r * Tr)];
        apply_pow<R, -SIGN1>(pw, v);
        DFT<R, -SIGN1>::run(v);
        if (TW) fourstep<R, false>(bg + l * BG, j, v);
        double2* o = gout + gpos(bg + l * BG, j);
#pragma unroll
        for (int r = 0; r < R; ++r) o[r * st] = v[r];
      }
    }
  }

  // ---- single transform (three-level inner passes): last stage of the
  // forward plan, smem -> twiddle -> DFT -> (four-step) -> global
  template <int SIGN, bool POST> __device__ __forceinline__ void final_stage(int tid) const {
    using P = PlanX<L, false>;
    constexpr int Q = nst - 1, S = nst - 1, R = P::radix(S), Ns = P::ns(S), T = L / R, TASKS = BG * T,
                  TPT = (TASKS + NT - 1) / NT;
    static_assert(T == Ns, "last stage covers j + r*T");
    constexpr int Pr = SQ::P(Q - 1), Cr = SQ::C(Q - 1), Tr = Cr ? T + Cr * (T / Pr) : T;
    static_assert(Cr == 0 || T % Pr == 0, "reader stride spans whole skew blocks");
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      const int q = tid + t * NT;
      if (TASKS % NT != 0 && q >= TASKS) break;
      int bg, j;
      map(q, T, bg, j);
      const Pow<R> pw = stage_pow<R, Ns, false, S>(j);
      const long long st = gstep(T);
#pragma unroll
      for (int l = 0; l < LPT; ++l) {
        double2 v[R];
        const double2* p = buf(Q) + (bg + l * BG) * LS + pb(j) + skew<Pr, Cr>(j);
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = p[SQ::ph(r * Tr)];
        apply_pow<R, SIGN>(pw, v);
        DFT<R, SIGN>::run(v);
        if (POST) fourstep<R, false>(bg + l * BG, j, v);
        double2* o = gout + gpos(bg + l * BG, j);
#pragma unroll
        for (int r = 0; r < R; ++r) o[r * st] = v[r];
      }
    }
  }
  template <int SIGN, bool PRE, bool POST> __device__ __forceinline__ void run_single(int tid) const {
    static_assert(SIGN == SIGN1, "single transforms run in the kernel's sign");
    first_stage<PRE>(tid);
    __syncthreads();  // stage buffer written; POST: also the twiddle powers of the output side
    sfor<nst - 2>([&](auto sc) {
      constexpr int s = decltype(sc)::value + 1;
      inner_stage<s, false, SIGN, s>(tid);
      __syncthreads();
    });
    final_stage<SIGN, POST>(tid);
  }

  __device__ __forceinline__ void run(int tid) const {
    first_stage(tid);
    __syncthreads();
    sfor<nst - 2>([&](auto sc) {
      constexpr int s = decltype(sc)::value + 1;
      inner_stage<s, false, SIGN1, s>(tid);
      __syncthreads();
    });
    mid_stage<nst - 1>(tid);
    __syncthreads();
    sfor<nst - 2>([&](auto sc) {
      constexpr int s = decltype(sc)::value + 1;
      inner_stage<s, true, -SIGN1, nst - 1 + s>(tid);
      __syncthreads();
    });
    last_stage<2 * nst - 2>(tid);
  }
};

// One CTA per tile of B lines; blockIdx.y = batch member.
template <int AXIS, int L, int B, int LPT, bool PP, int NT, int SIGN1, bool TW, int DK, int MINB>
__global__ void __launch_bounds__(NT, MINB) fft_pass4_kernel(const __grid_constant__ PassArgs a) {
  using K = Pass4<AXIS, L, B, LPT, PP, NT, SIGN1, TW, DK>;
  using G = typename K::G;
  extern __shared__ double2 lattdse_smem4[];
  const int tid = threadIdx.x;
  const int line0 = (int)blockIdx.x * B;
  const long long bat = blockIdx.y;
  // L2 prefetch of the tile a.pf tiles ahead in launch order (x fastest)
  if (a.pf > 0) {
    long long tl = (long long)blockIdx.y * gridDim.x + blockIdx.x + a.pf;
    const long long by = tl / gridDim.x;
    if (by < (long long)gridDim.y) {
      const int bx = (int)(tl - by * gridDim.x);
      const double2* src = a.in + by * a.in_bstride;
      if (AXIS == AX_ROW) {
        if (tid == 0) {
          const double2* p = src + (long long)bx * B * L;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(B * L * 16) : "memory");
        }
      } else {
        for (int i = tid; i < L; i += NT) {
          const double2* p = src + (long long)i * a.ncols + bx * B;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
          if (B * 16 > 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 8));
        }
      }
    }
  }
  double2* twp = lattdse_smem4 + (G::pp ? 2 : 1) * G::tile;
  K k{a, lattdse_smem4, twp, a.in + bat * a.in_bstride, a.out + bat * a.out_bstride, line0, 1};
  if (TW) {
    // twp[b][r] = W^(col_b * T0 * r): the powers every task of column b needs
    constexpr int R0 = G::R0, T0 = L / R0;
    for (int i = tid; i < B * R0; i += NT) {
      const int b = i / R0, r = i - b * R0;
      twp[i] = k.twid((long long)(a.col_off + line0 + b) * (T0 * r));
    }
  }
  k.run(tid);
}


// Single-transform pass of the plain COL layout with four-step twiddles on
// one side (the three-level inner passes: FFT_Ma then x W_M2, or x conj W_M2
// then IFFT_Ma, inside every row of the M1 x M2 view; blockIdx.y = row).
// PRE: conjugate twiddles at the load (elements j + r T0 of the first
// stage); POST: twiddles at the store (elements j + r T of the last stage).
template <int L, int B, bool PP, int NT, int SIGN, bool PRE, int MINB>
__global__ void __launch_bounds__(NT, MINB) fft_pass4s_kernel(const __grid_constant__ PassArgs a) {
  using K = Pass4<AX_COL, L, B, 1, PP, NT, SIGN, true, DG_NONE>;
  using G = typename K::G;
  extern __shared__ double2 lattdse_smem4[];
  const int tid = threadIdx.x;
  const int line0 = (int)blockIdx.x * B;
  const long long bat = blockIdx.y;
  double2* twp = lattdse_smem4 + (G::pp ? 2 : 1) * G::tile;
  K k{a, lattdse_smem4, twp, a.in + bat * a.in_bstride, a.out + bat * a.out_bstride, line0, a.tw_mul > 1 ? a.tw_mul : 1};
  // powers of the column twiddles for the side that carries them: the first
  // stage's elements j + r T0 (PRE) or the last stage's j + r T (POST)
  constexpr int Rt = PRE ? G::R0 : Plan<L>::radix(Plan<L>::nst - 1), Tt = L / Rt;
  static_assert(B * Rt <= G::tw_slots, "twiddle slots");
  for (int i = tid; i < B * Rt; i += NT) {
    const int b = i / Rt, r = i - b * Rt;
    twp[i] = k.twid((long long)(a.col_off + line0 + b) * k.twm * (Tt * r));
  }
  if (PRE)
    k.template run_single<SIGN, true, false>(tid);
  else
    k.template run_single<SIGN, false, true>(tid);
}

#endif

}  // namespace lattdse_dev
