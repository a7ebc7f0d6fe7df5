// Microbenchmark: the ALU peaks bench.py divides by (roofline.peak for the FP64 and FP32 flux).
// Dependent-chain-free FMA loops (8 independent chains per thread, 4 blocks x 256 threads per SM)
// for DFMA (fp64) and FFMA (fp32); prints one JSON object.  Build + run on a B200:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/alu_peaks tools/microbench/alu_peaks.cu && /tmp/alu_peaks
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_loop(T* out, int iters, T seed) {
  T x[8];
  for (int k = 0; k < 8; ++k) x[k] = seed + T(k) + T(threadIdx.x);
  const T a = T(0.999999), b = T(1e-7);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  T acc = T(0);
  for (int k = 0; k < 8; ++k) acc += x[k];
  if (acc == T(12345.678)) out[0] = acc;
}

// packed FP32 (FFMA2): 8 independent float2 chains per thread
__global__ void ffma2_loop(float* out, int iters, float seed) {
  float2 x[8];
  for (int k = 0; k < 8; ++k) x[k] = make_float2(seed + k + threadIdx.x, seed - k);
  const float2 a = make_float2(0.999999f, 0.999998f), b = make_float2(1e-7f, 2e-7f);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], a, b);
  float acc = 0.f;
  for (int k = 0; k < 8; ++k) acc += x[k].x + x[k].y;
  if (acc == 12345.678f) out[0] = acc;
}

// issue test: FFMA (MIX=0) or FFMA2 (MIX=1) chains interleaved with as many independent integer ops;
// if the packed form leaves issue slots free, MIX=1 runs at its pure FMA rate despite the integer ops
template <int MIX>
__global__ void mixed_loop(float* out, int iters, float seed) {
  float2 x[8];
  unsigned u[8];
  for (int k = 0; k < 8; ++k) {
    x[k] = make_float2(seed + k + threadIdx.x, seed - k);
    u[k] = threadIdx.x * (k + 3);
  }
  const float2 a = make_float2(0.999999f, 0.999998f), b = make_float2(1e-7f, 2e-7f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MIX == 1) {
        x[k] = __ffma2_rn(x[k], a, b);
      } else {
        x[k].x = fmaf(x[k].x, a.x, b.x);
        x[k].y = fmaf(x[k].y, a.y, b.y);
      }
      u[k] = (u[k] ^ 0x9e3779b9u) + (u[k] >> 3);  // LOP3 + SHF + IADD3: ALU pipe, not the FMA pipe
    }
  }
  float acc = 0.f;
  unsigned uu = 0;
  for (int k = 0; k < 8; ++k) {
    acc += x[k].x + x[k].y;
    uu ^= u[k];
  }
  if (acc == 12345.678f || uu == 7u) out[0] = acc + uu;
}

template <int MIX>
static double mixed_tflops(int blocks, int threads, int iters) {
  float* out;
  cudaMalloc(&out, sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    mixed_loop<MIX><<<blocks, threads>>>(out, iters, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)blocks * threads * iters * 8 * 4;
    if (rep > 0 && fl / ms / 1e9 > best) best = fl / ms / 1e9;
  }
  cudaFree(out);
  return best;
}

static double ffma2_tflops(int blocks, int threads, int iters) {
  float* out;
  cudaMalloc(&out, sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    ffma2_loop<<<blocks, threads>>>(out, iters, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)blocks * threads * iters * 8 * 4;
    if (rep > 0 && fl / ms / 1e9 > best) best = fl / ms / 1e9;
  }
  cudaFree(out);
  return best;
}

template <typename T>
static double tflops(int blocks, int threads, int iters) {
  T* out;
  cudaMalloc(&out, sizeof(T));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma_loop<T><<<blocks, threads>>>(out, iters, T(1));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)blocks * threads * iters * 8 * 2;
    if (rep > 0 && fl / ms / 1e9 > best) best = fl / ms / 1e9;
  }
  cudaFree(out);
  return best;
}

int main() {
  int sms, clk_khz;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double d = tflops<double>(sms * 4, 256, 20000);
  const double f = tflops<float>(sms * 4, 256, 40000);
  const double f2 = ffma2_tflops(sms * 4, 256, 20000);
  const double m1 = mixed_tflops<0>(sms * 4, 256, 10000), m2 = mixed_tflops<1>(sms * 4, 256, 10000);
  printf("{\"dfma_tflops\": %.3f, \"ffma_tflops\": %.3f, \"ffma2_tflops\": %.3f, \"ffma_plus_int_tflops\": %.3f, "
         "\"ffma2_plus_int_tflops\": %.3f, \"sms\": %d, \"clock_rate_mhz_attr\": %.0f, "
         "\"how\": \"tools/microbench/alu_peaks.cu: 8 independent FMA chains per thread, %d blocks x 256, best of 4\"}\n",
         d, f, f2, m1, m2, sms, clk_khz / 1000.0, sms * 4);
  return 0;
}
