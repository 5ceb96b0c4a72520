// Minimal ||h||^2 per residue of a rank-1 lattice, built on the device
// (at d = 20, N ~ 2^30 the shell walk visits ~1e10-1e11
// integer vectors, out of reach of the host enumeration).
//
// Same result as AntiAliasSet::build's norm table (antialias.cpp; SPEC.md
// 163-222): norm2[chi] = min ||h||^2 over h in Z^d with z.h == chi (mod N).
// Only the norms enter the step, so no tie-break (and no h) is needed.
//
// Meet in the middle: h = (hA, hB) with hA the first dA = d/2 coordinates.
// The host lists every half vector with ||.||^2 <= S_list together with its
// partial residue, bucketed by norm. Shell s (exact norm s, ascending) is
// the union over t of the pairs A_t x B_{s-t}; a residue first reached in
// shell s gets norm s. Within one launch every writer stores the same value
// s, so plain loads/stores suffice (no atomics); shells are separate
// launches, which orders them. Shells stop once no residue is left; the
// radius cap 4 N^(1/d) + 16 of SPEC.md raises radius_exhausted.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "aaset_dev.hpp"
#include "lattdse/errors.hpp"
#include "lattdse/setup.hpp"

namespace lattdse::dev {

namespace {

#define AA_CK(x)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) raise(Errc::device_error, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr unsigned short kUnset = 0xFFFF;

// Half vectors over coordinates [j0, j1) with ||h||^2 <= S: partial residues
// sum z_j h_j mod N, bucketed by norm (off[t] .. off[t+1]).
struct Half {
  std::vector<unsigned> res;
  std::vector<long long> off;  // S + 2 entries
};

Half half_list(const std::vector<long long>& z, int j0, int j1, long long N, int S) {
  std::vector<std::vector<unsigned>> by(S + 1);
  std::vector<int> h(j1 - j0, 0);
  // iterative depth-first walk with per-level remaining budget
  struct Frame {
    int x, lim;
    long long res;
    int rem;
  };
  const int k = j1 - j0;
  if (k == 0) {
    by[0].push_back(0);
  } else {
    std::vector<Frame> st(k);
    auto isqrt = [](int v) {
      int r = (int)std::sqrt((double)v);
      while ((r + 1) * (r + 1) <= v) ++r;
      while (r * r > v) --r;
      return r;
    };
    int lvl = 0;
    st[0] = {-isqrt(S), isqrt(S), 0, S};
    for (;;) {
      Frame& f = st[lvl];
      if (f.x > f.lim) {
        if (lvl == 0) break;
        --lvl;
        ++st[lvl].x;
        continue;
      }
      const long long zj = z[j0 + lvl] % N;
      long long r = (f.res + (long long)f.x * zj) % N;
      if (r < 0) r += N;
      const int rem = f.rem - f.x * f.x;
      if (lvl + 1 == k) {
        by[S - rem].push_back((unsigned)r);
        ++f.x;
      } else {
        const int m = isqrt(rem);
        st[lvl + 1] = {-m, m, r, rem};
        ++lvl;
      }
    }
  }
  Half out;
  out.off.assign(S + 2, 0);
  for (int t = 0; t <= S; ++t) out.off[t + 1] = out.off[t] + (long long)by[t].size();
  out.res.reserve(out.off[S + 1]);
  for (int t = 0; t <= S; ++t) out.res.insert(out.res.end(), by[t].begin(), by[t].end());
  return out;
}

struct Combo {
  long long a_off, a_cnt, b_off, b_cnt;
};

// one warp per A entry of the shell; lanes stride over the matching B bucket
__global__ void k_aa_shell(const Combo* __restrict__ combos, const long long* __restrict__ item_pref, int ncombo,
                           long long nitems, const unsigned* __restrict__ resA, const unsigned* __restrict__ resB,
                           unsigned N, unsigned short s, unsigned short* __restrict__ table) {
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nitems; w += nw) {
    int lo = 0, hi = ncombo - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (item_pref[mid] <= w) lo = mid;
      else hi = mid - 1;
    }
    const Combo c = combos[lo];
    const unsigned ra = resA[c.a_off + (w - item_pref[lo])];
    for (long long ib = lane; ib < c.b_cnt; ib += 32) {
      unsigned r = ra + resB[c.b_off + ib];
      if (r >= N) r -= N;
      if (table[r] == kUnset) table[r] = s;
    }
  }
}

__global__ void k_aa_count_unset(const unsigned short* __restrict__ table, long long n, unsigned long long* count) {
  unsigned long long c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    c += table[i] == kUnset;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

}  // namespace

std::uint32_t aaset_norms_device(const Lattice& lat, unsigned short* table, cudaStream_t st, double cap_radius) {
  if (lat.rank() != 1) raise(Errc::unsupported, "device anti-aliasing norms: rank-1 lattices only");
  const long long N = lat.n_total();
  if (N >= (1LL << 31)) raise(Errc::unsupported, "device anti-aliasing norms: N must be < 2^31");
  const int d = lat.dim();
  const auto steps = lat.numerator_steps();
  std::vector<long long> z(d);
  for (int j = 0; j < d; ++j) z[j] = steps[0][j];
  if (cap_radius <= 0) cap_radius = 4.0 * std::pow((double)N, 1.0 / d) + 16.0;
  const long long cap2 = (long long)std::floor(cap_radius * cap_radius);
  const long long limit = std::min<long long>(cap2, kUnset - 1);  // uint16 table entries
  const int dA = d / 2;

  AA_CK(cudaMemsetAsync(table, 0xFF, sizeof(unsigned short) * N, st));
  unsigned long long* dcount = nullptr;
  AA_CK(cudaMalloc(&dcount, sizeof(unsigned long long)));
  unsigned *dA_res = nullptr, *dB_res = nullptr;
  Combo* dcombo = nullptr;
  long long* dpref = nullptr;
  auto cleanup = [&] {
    cudaFree(dcount);
    cudaFree(dA_res);
    cudaFree(dB_res);
    cudaFree(dcombo);
    cudaFree(dpref);
  };
  try {
    int dev = 0, sms = 148;
    AA_CK(cudaGetDevice(&dev));
    AA_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    Half A, B;
    int S_list = -1;
    std::vector<Combo> combos;
    std::vector<long long> pref;
    for (long long s = 0;; ++s) {
      if (s > limit) {
        if (limit == cap2) raise(Errc::radius_exhausted, "anti-aliasing radius cap reached with residues uncovered");
        raise(Errc::unsupported, "device anti-aliasing norms: ||h||^2 beyond the uint16 table");
      }
      if (s > S_list) {  // (re)build the half lists up to a larger radius
        S_list = (int)std::min<long long>(limit, std::max<long long>(2 * S_list, std::max<long long>(s, 8)));
        A = half_list(z, 0, dA, N, S_list);
        B = half_list(z, dA, d, N, S_list);
        cudaFree(dA_res);
        cudaFree(dB_res);
        dA_res = dB_res = nullptr;
        AA_CK(cudaMalloc(&dA_res, sizeof(unsigned) * std::max<size_t>(1, A.res.size())));
        AA_CK(cudaMalloc(&dB_res, sizeof(unsigned) * std::max<size_t>(1, B.res.size())));
        AA_CK(cudaMemcpyAsync(dA_res, A.res.data(), sizeof(unsigned) * A.res.size(), cudaMemcpyHostToDevice, st));
        AA_CK(cudaMemcpyAsync(dB_res, B.res.data(), sizeof(unsigned) * B.res.size(), cudaMemcpyHostToDevice, st));
        cudaFree(dcombo);
        cudaFree(dpref);
        dcombo = nullptr;
        dpref = nullptr;
        AA_CK(cudaMalloc(&dcombo, sizeof(Combo) * (S_list + 1)));
        AA_CK(cudaMalloc(&dpref, sizeof(long long) * (S_list + 1)));
      }
      combos.clear();
      pref.clear();
      long long items = 0;
      for (long long t = 0; t <= s; ++t) {
        const long long ac = A.off[t + 1] - A.off[t], bc = B.off[s - t + 1] - B.off[s - t];
        if (ac == 0 || bc == 0) continue;
        combos.push_back({A.off[t], ac, B.off[s - t], bc});
        pref.push_back(items);
        items += ac;
      }
      if (items > 0) {
        // host vectors must outlive the async copies: synchronise before reuse
        AA_CK(cudaMemcpyAsync(dcombo, combos.data(), sizeof(Combo) * combos.size(), cudaMemcpyHostToDevice, st));
        AA_CK(cudaMemcpyAsync(dpref, pref.data(), sizeof(long long) * pref.size(), cudaMemcpyHostToDevice, st));
        const long long warps = std::min<long long>(items, (long long)sms * 64);
        k_aa_shell<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(dcombo, dpref, (int)combos.size(), items, dA_res,
                                                                      dB_res, (unsigned)N, (unsigned short)s, table);
        AA_CK(cudaGetLastError());
      }
      AA_CK(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), st));
      k_aa_count_unset<<<sms * 8, 256, 0, st>>>(table, N, dcount);
      AA_CK(cudaGetLastError());
      unsigned long long left = 0;
      AA_CK(cudaMemcpyAsync(&left, dcount, sizeof(left), cudaMemcpyDeviceToHost, st));
      AA_CK(cudaStreamSynchronize(st));
      if (left == 0) {
        cleanup();
        return (std::uint32_t)s;
      }
    }
  } catch (...) {
    cudaStreamSynchronize(st);
    cleanup();
    throw;
  }
}

}  // namespace lattdse::dev

namespace lattdse {

AntiAliasSet AntiAliasSet::build_norms_device(const Lattice& lat, int device, double cap_radius) {
  AA_CK(cudaSetDevice(device));
  cudaStream_t st = nullptr;
  AA_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  unsigned short* table = nullptr;
  AntiAliasSet aa;
  aa.n_total = lat.n_total();
  aa.dim = lat.dim();
  try {
    AA_CK(cudaMalloc(&table, sizeof(unsigned short) * aa.n_total));
    aa.max_norm2 = dev::aaset_norms_device(lat, table, st, cap_radius);
    std::vector<unsigned short> h(aa.n_total);
    AA_CK(cudaMemcpyAsync(h.data(), table, sizeof(unsigned short) * aa.n_total, cudaMemcpyDeviceToHost, st));
    AA_CK(cudaStreamSynchronize(st));
    aa.norm2.assign(h.begin(), h.end());
  } catch (...) {
    cudaFree(table);
    cudaStreamDestroy(st);
    throw;
  }
  cudaFree(table);
  cudaStreamDestroy(st);
  return aa;
}

}  // namespace lattdse
