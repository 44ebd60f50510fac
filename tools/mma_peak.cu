// Throughput of the legacy warp-level tensor path (mma.sync) on sm_100a: m16n8k8 TF32 and
// m16n8k16 F16 (fp32 accumulate), and FP32 FFMA for reference. One launch, independent accumulators.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_tf32(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f16(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u + threadIdx.x;
  for (int i = 0; i < 2; ++i) b[i] = 0x38003800u;
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 1024 * sizeof(float));
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int w = 4; w <= 16; w *= 2) {
    for (int kind = 0; kind < 2; ++kind) {
      auto run = [&]() {
        if (kind == 0) k_tf32<<<sms * 2, w * 32>>>(d, iters);
        else k_f16<<<sms * 2, w * 32>>>(d, iters);
      };
      run();
      cudaEventRecord(a);
      run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double flop = 2.0 * sms * 2 * w * (double)iters * 8 * (kind == 0 ? 16 * 8 * 8 : 16 * 8 * 16);
      printf("%s warps/CTA %2d (2 CTAs/SM): %.1f TFLOP/s\n", kind == 0 ? "mma.sync m16n8k8 tf32 " : "mma.sync m16n8k16 f16", w,
             flop / ms / 1e9);
    }
  }
  return 0;
}
