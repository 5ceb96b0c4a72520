// Cluster COL pass (cluster_col.inl): host-side entry points.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "fft_pass.cuh"

namespace lattdse::dev {
// rows per CTA for a column length L over ncols columns when the cluster COL
// pass handles it (0: use the plain pass kernel; LATTDSE_CLUSTER_COL = 0/4/8)
int cluster_col_lloc(int L, long long ncols);
// device table layout the launcher expects: exp(-2 pi i t / L) for t < L,
// then the Plan<L / C> stage twiddles
std::vector<double2> cluster_col_tables(int L, int lloc);
// PROG_DOUBLE (FFT_L sign, x diag, IFFT_L) on every column, in place allowed
cudaError_t launch_cluster_col(int L, int lloc, int sign, const lattdse_dev::PassArgs& a, const double2* tables, long long ncols,
                               long long nbatch, cudaStream_t s);
}  // namespace lattdse::dev
