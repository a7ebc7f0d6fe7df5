// diag_kernels.cuh — on-device volume diagnostics (O-24, O-25).
//
//   diag_kernel<T>      per-cell terms of E_k, enstrophy, |omega|^2, (div U)^2, p div U and the
//                       conservation monitors, summed per block in a fixed order (fp64 for either
//                       precision)
//   diag_final_kernel   one block: fixed-order sum of the block partials -> NDIAG doubles
//
// Deterministic: a fixed grid (DIAG_BLOCKS x DIAG_TPB), a fixed grid-stride cell order per thread
// and fixed tree reductions, so repeated calls on the same state return identical bits.
#pragma once
#include "hgks_kernels.cuh"

namespace hgks {

constexpr int DIAG_BLOCKS = 148 * 4;

template <typename T>
__global__ void __launch_bounds__(DIAG_TPB) diag_kernel(const T* __restrict__ q, Geo<T> g, DiagGeo dg, double gamma,
                                                        double* __restrict__ partial) {
  __shared__ double sh[NDIAG * DIAG_TPB];
  double acc[NDIAG];
#pragma unroll
  for (int n = 0; n < NDIAG; ++n) acc[n] = 0.0;
  const int nx = g.n[0], ny = g.n[1];
  const long long ncell = (long long)nx * ny * g.n[2];
  for (long long e = blockIdx.x * (long long)DIAG_TPB + threadIdx.x; e < ncell; e += (long long)gridDim.x * DIAG_TPB) {
    const int i = (int)(e % nx), j = (int)((e / nx) % ny), k = (int)(e / ((long long)nx * ny));
    diag_cell(q, g, dg, gamma, i, j, k, acc);
  }
  block_sum_fixed(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int n = 0; n < NDIAG; ++n) partial[blockIdx.x * NDIAG + n] = acc[n];
  }
}

template <int N>
__global__ void __launch_bounds__(DIAG_TPB) diag_final_kernel(const double* __restrict__ partial, int nblocks,
                                                              double* __restrict__ out) {
  __shared__ double sh[N * DIAG_TPB];
  double acc[N];
#pragma unroll
  for (int n = 0; n < N; ++n) acc[n] = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += DIAG_TPB) {
#pragma unroll
    for (int n = 0; n < N; ++n) acc[n] += partial[b * N + n];
  }
  block_sum_fixed(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int n = 0; n < N; ++n) out[n] = acc[n];
  }
}

// ---- x-z plane statistics (channel, O-28) -------------------------------------------
// One block per y plane j: thread t sums the plane's cells t, t + DIAG_TPB, ... in that order, then
// a fixed tree; out[j][s] = plane mean of moment s (order of HGKS_STAT_*).
constexpr int NSTAT = 16;

template <typename T>
__global__ void __launch_bounds__(DIAG_TPB) plane_stats_kernel(const T* __restrict__ q, Geo<T> g, double gamma,
                                                               double* __restrict__ out) {
  __shared__ double sh[NSTAT * DIAG_TPB];
  const int j = blockIdx.x, nx = g.n[0], nz = g.n[2];
  const long long nplane = (long long)nx * nz;
  double acc[NSTAT];
#pragma unroll
  for (int s = 0; s < NSTAT; ++s) acc[s] = 0.0;
  for (long long e = threadIdx.x; e < nplane; e += DIAG_TPB) {
    const int i = (int)(e % nx), k = (int)(e / nx);
    const double rho = (double)q[qidx(g, 0, i, j, k)];
    const double U = (double)q[qidx(g, 1, i, j, k)] / rho, V = (double)q[qidx(g, 2, i, j, k)] / rho,
                 W = (double)q[qidx(g, 3, i, j, k)] / rho;
    const double u2 = U * U + V * V + W * W;
    const double p = (gamma - 1.0) * ((double)q[qidx(g, 4, i, j, k)] - 0.5 * rho * u2);
    const double c = sqrt(gamma * p / rho);
    const double M = sqrt(u2) / c;
    const double v[NSTAT] = {rho, U, V, W, U * U, V * V, W * W, U * V, rho * U, rho * V, rho * U * V, c, M, M * M, p / rho, p};
#pragma unroll
    for (int s = 0; s < NSTAT; ++s) acc[s] += v[s];
  }
  block_sum_fixed(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NSTAT; ++s) out[(long long)j * NSTAT + s] = acc[s];
  }
}

}  // namespace hgks
