// FP64 / FP32 FMA peak of this GPU (roofline denominators for the compute side):
// every thread runs 16 independent FMA chains; flops = 2 per FMA. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_kernel(T* out, int iters, T a, T b) {
  T x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = T(threadIdx.x + j);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = x[j] * a + b;
  T s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  if (s == T(-1)) out[threadIdx.x] = s;  // keep the chains alive
}

template <typename T>
double run(int sms) {
  T* out;
  cudaMalloc(&out, 1024 * sizeof(T));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  fma_kernel<T><<<blocks, threads>>>(out, 16, T(0.999), T(0.001));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) fma_kernel<T><<<blocks, threads>>>(out, iters, T(0.999), T(0.001));
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  const double flops = 5.0 * blocks * threads * double(iters) * 16 * 2;
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double f64 = run<double>(sms), f32 = run<float>(sms);
  printf("{\"fp64_fma_tflops\": %.2f, \"fp32_fma_tflops\": %.2f, \"sms\": %d}\n", f64, f32, sms);
  return 0;
}
