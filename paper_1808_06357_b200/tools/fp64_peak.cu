// Microbenchmark: FP64 (DFMA / DADD) issue throughput and shared-memory
// bandwidth of one B200, the two in-SM co-limits of the pass kernels
// (DESIGN.md §4). Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// fp64_peak.cu -o fp64_peak ; prints TFLOP/s (DFMA = 2 flops) and TB/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_smem(double* out, int iters) {
  extern __shared__ double2 sm[];
  const int n = 4096;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double2 v = sm[(idx + u * 128) & (n - 1)];
      acc.x += v.x;
      acc.y += v.y;
    }
    idx += 1;
  }
  if (acc.x == 1.2345) out[0] = acc.y;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096, nt = warps * 32, grid = sms;
    k_dfma<8><<<grid, nt>>>(d, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k_dfma<8><<<grid, nt>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 8 * iters * (double)nt * grid;
    printf("dfma warps/SM=%d ILP=8: %.2f TFLOP/s (%.1f DFMA lanes/clk/SM at 1965 MHz)\n", warps, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
  }
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int warps : {8, 16, 32}) {
    const int iters = 8192, nt = warps * 32, grid = sms;
    k_smem<<<grid, nt, 65536>>>(d, 16);
    cudaEventRecord(e0);
    k_smem<<<grid, nt, 65536>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double by = 16.0 * 8 * iters * (double)nt * grid;
    printf("lds.128 warps/SM=%d: %.2f TB/s (%.1f B/clk/SM at 1965 MHz)\n", warps, by / ms / 1e9,
           by / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
