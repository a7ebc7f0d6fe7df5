// LDS.64 throughput: 32 distinct words per warp vs 16 distinct words shared by the two half-warps
// (lane l and l+16 read the same address) vs the mirrored pattern of the flux kernel.
#include <cstdio>
#include <cuda_runtime.h>

template <int PAT>
__global__ void __launch_bounds__(256) lds_kernel(double* out, int iters, long long* cyc) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int idx;
  if (PAT == 0) idx = lane;                                   // 32 distinct consecutive
  else if (PAT == 1) idx = lane & 15;                         // half-warps share
  else idx = (lane & 15) + (lane >> 4) * 152;                 // two distinct row streams (flux fp64)
  idx += w * 256;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int off = (it & 7) * 16;
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += sm[(idx + off + u * 320) & 4095];
  }
  long long t1 = clock64();
  double s = 0;
  for (int u = 0; u < 8; ++u) s += acc[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int PAT>
void run(const char* name) {
  const int blocks = 148 * 4, iters = 4096;
  double* out;
  long long* cyc;
  cudaMalloc(&out, blocks * 256 * sizeof(double));
  cudaMalloc(&cyc, blocks * sizeof(long long));
  lds_kernel<PAT><<<blocks, 256>>>(out, iters, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  lds_kernel<PAT><<<blocks, 256>>>(out, iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double warp_lds = double(blocks) * 8 * iters * 8;
  // cycles per warp-LDS per SM at the measured clock
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double sm_cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s %.3f ms  %.3f SM-cycles per warp-LDS.64 (per SM)\n", name, ms, sm_cyc * 148 / warp_lds);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("32 distinct");
  run<1>("16 distinct, halves share");
  run<2>("two row streams");
  return 0;
}
