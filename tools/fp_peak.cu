// Measured FP64 / FP32 FMA peak of this GPU (the roofline denominator for
// the K6 kernel's arithmetic): every thread runs 8 independent FMA chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_peak fp_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = (T)(threadIdx.x + j);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  T s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == (T)-1.2345) out[0] = s;
}

template <typename T>
double run(int blocks_per_sm) {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  T* out;
  cudaMalloc(&out, sizeof(T));
  const int iters = 1 << 16, threads = 256, blocks = nsm * blocks_per_sm;
  fma_loop<T><<<blocks, threads>>>(out, 16, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return 2.0 * 8.0 * iters * (double)threads * blocks / (ms * 1e-3) / 1e12;   // TFLOP/s (FMA = 2 flops)
}

int main() {
  double f64 = 0, f32 = 0;
  for (int b = 2; b <= 8; b *= 2) {
    const double x = run<double>(b), y = run<float>(b);
    f64 = x > f64 ? x : f64;
    f32 = y > f32 ? y : f32;
  }
  printf("{\"fp64_fma_tflops\": %.2f, \"fp32_fma_tflops\": %.2f}\n", f64, f32);
  return 0;
}
