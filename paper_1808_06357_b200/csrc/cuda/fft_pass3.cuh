// pass3: the per-step PROG_DOUBLE passes as persistent, TMA-fed kernels.
//
// Why (profiles/r2a, ncu of the config-3 passes): the v1 pass kernels load
// stage 0 straight from global into registers, so a CTA has its tile in
// flight only during stage 0 and is compute-only afterwards; with 2-3 CTAs
// per SM the HBM queue drains while every CTA is in its butterfly stages
// (long-scoreboard stalls, ~0.3 of HBM peak on the streaming COL pass).
// Here every CTA owns two tile buffers: while tile t is transformed, tile
// t+gridDim is already on its way into the other buffer, issued by ONE
// thread as TMA copies that complete on an mbarrier -- no per-thread
// address registers (what made the round-1 cp.async variant spill).
//
//  COL (strided lines): 3-D tensor map over the work buffer
//     {2*M2 doubles, M1 rows, batch}; box {2B doubles, BOXR rows, 1};
//     L/BOXR copies per tile, landing densely as [row][B] complex.
//  ROW (contiguous lines): one 1-D bulk copy of B*L*16 bytes per tile.
//
// Shared memory per CTA: two tile buffers (+ one stage buffer when the
// stages ping-pong: the tile's own buffer becomes the even stage buffer
// once stage 0 has consumed it), two mbarriers.
#pragma once

#include <cuda.h>

#include "fft_pass.cuh"

namespace lattdse_dev {

constexpr int pass3_boxr(int L) {
  for (int r = 256; r >= 1; --r)
    if (L % r == 0) return r;
  return 1;
}

template <int AXIS, int L, int B> struct Pass3Geom {
  using SG = SmemGeom<L, B>;
  static constexpr int boxr = pass3_boxr(L);
  static constexpr int tile_slots = SG::tile > B * L ? SG::tile : B * L;
  static constexpr int buf_bytes = ((tile_slots * 16 + 127) / 128) * 128;
  static constexpr int nbuf = SG::pp ? 3 : 2;
  static constexpr int bytes = 128 + nbuf * buf_bytes;
  static constexpr unsigned tx_bytes = (unsigned)(B * L * 16);
};

#if defined(__CUDACC__)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses of shared memory before async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int AXIS, int L, int B>
__device__ __forceinline__ void pass3_issue(const PassArgs& a, const CUtensorMap* map, double2* dst,
                                            unsigned long long* bar, int t) {
  using G = Pass3Geom<AXIS, L, B>;
  const int blk = t % a.nblk;
  const int bat = t / a.nblk;
  if (AXIS == AX_COL) {
    // columns beyond the view are zero-filled and still count as transaction bytes
    mbar_arrive_expect_tx(bar, G::tx_bytes);
#pragma unroll 1
    for (int r0 = 0; r0 < L; r0 += G::boxr) tma_load_3d(dst + r0 * B, map, 2 * B * blk, r0, bat, bar);
  } else {
    // contiguous lines; the dead lines of a partial last block stay unloaded
    // (their results are never stored)
    const int live = min(B, a.nlines - blk * B);
    const unsigned bytes = (unsigned)(live * L * 16);
    mbar_arrive_expect_tx(bar, bytes);
    bulk_load(dst, a.in + (long long)bat * a.in_bstride + (long long)blk * B * L, bytes, bar);
  }
}

template <int AXIS, int L, int B, int NT, int SIGN1, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    fft_pass3_kernel(const __grid_constant__ PassArgs a, const __grid_constant__ CUtensorMap map) {
  using G = Pass3Geom<AXIS, L, B>;
  extern __shared__ __align__(128) unsigned char lattdse_smem3[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(lattdse_smem3);
  double2* tb[2] = {reinterpret_cast<double2*>(lattdse_smem3 + 128),
                    reinterpret_cast<double2*>(lattdse_smem3 + 128 + G::buf_bytes)};
  double2* wb = G::nbuf == 3 ? reinterpret_cast<double2*>(lattdse_smem3 + 128 + 2 * G::buf_bytes) : nullptr;
  int t = blockIdx.x;
  if (t >= a.ntiles) return;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pass3_issue<AXIS, L, B>(a, &map, tb[0], &bar[0], t);
  }
  __syncthreads();
  for (int k = 0; t < a.ntiles; t += gridDim.x, ++k) {
    const int cur = k & 1;
    const int tn = t + (int)gridDim.x;
    if (threadIdx.x == 0 && tn < a.ntiles) {
      // the other buffer was last touched (generic proxy) by tile k-1, whose
      // closing barrier every thread has passed
      fence_proxy_async_smem();
      pass3_issue<AXIS, L, B>(a, &map, tb[cur ^ 1], &bar[cur ^ 1], tn);
    }
    mbar_wait(&bar[cur], (unsigned)((k >> 1) & 1));
    Ctx<AXIS, L, B, PROG_DOUBLE> c{tb[cur], a, (t % a.nblk) * B, (long long)(t / a.nblk), tb[cur], wb};
    run_pass<DevExec, AXIS, L, B, NT, PROG_DOUBLE, SIGN1, SRC_TMA>(c);
    __syncthreads();
  }
}
#endif

}  // namespace lattdse_dev
