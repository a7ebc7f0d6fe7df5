// Microbenchmark: FP64 vector (DFMA) vs FP64 tensor (DMMA m8n8k4) throughput on sm_100a, alone and
// concurrently (half the warps each), to learn whether the two share execution units.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int MODE>  // 0: DFMA only, 1: DMMA only, 2: even warps DFMA, odd warps DMMA
__global__ void bench(double* out, int iters, double seed) {
  const int warp = threadIdx.x >> 5;
  const bool use_mma = MODE == 1 || (MODE == 2 && (warp & 1));
  double acc = 0.0;
  if (!use_mma) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = seed + k + threadIdx.x;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999999, 1e-7);
    for (int k = 0; k < 8; ++k) acc += x[k];
  } else {
    double c[8][2];
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = seed + k;
    const double a = 0.999, b = 1e-3 * threadIdx.x;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b, c[k][0], c[k][1]);
    for (int k = 0; k < 8; ++k) acc += c[k][0] + c[k][1];
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, threads = 256, blocks = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) bench<0><<<blocks, threads>>>(out, iters, 1.0);
      if (mode == 1) bench<1><<<blocks, threads>>>(out, iters, 1.0);
      if (mode == 2) bench<2><<<blocks, threads>>>(out, iters, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // flops: DFMA thread-op = 2 flop; DMMA m8n8k4 per warp = 2*8*8*4 = 512 flop
      double warps = blocks * threads / 32.0;
      double fl_dfma = (mode == 0 ? warps : (mode == 2 ? warps / 2 : 0)) * 32.0 * iters * 8 * 2;
      double fl_dmma = (mode == 1 ? warps : (mode == 2 ? warps / 2 : 0)) * iters * 8 * 512.0;
      if (rep == 1)
        printf("mode %d: %.3f ms  DFMA %.2f TF  DMMA %.2f TF  total %.2f TF\n", mode, ms, fl_dfma / ms / 1e9,
               fl_dmma / ms / 1e9, (fl_dfma + fl_dmma) / ms / 1e9);
    }
  }
  return 0;
}
