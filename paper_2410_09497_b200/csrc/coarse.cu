// Level-0 pseudo-inverse on the device (coarse_solve SPEC.md:468-476): the bordered system
// [[A_0, e],[e^T, 0]] (e = constant pressure, ker A_0 = span(e)) is LU-factorised by cuSOLVER
// (getrf, partial pivoting) and solved against the identity (getrs); the leading nf x nf block of the
// inverse, symmetrised, is A_0^+. A setup-time library factorisation: the O(nf^3) host Gauss-Jordan
// it replaces limited the multigrid to k <= 4 (nf = 4300 at k = 4, 17152 at k = 7).
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <string>

#include "smg_internal.cuh"

namespace smg {
namespace {

#define SMG_CUSOLVER(call)                                                                         \
  do {                                                                                             \
    cusolverStatus_t s_ = (call);                                                                  \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                             \
      throw ::smg::cuda_error(std::string(#call) + " failed (" + std::to_string(static_cast<int>(s_)) + ")"); \
  } while (0)

__global__ void identity_kernel(double* a, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    a[i] = (i / n == i % n) ? 1.0 : 0.0;
}

// pinv(i, j) = (Ki(i, j) + Ki(j, i)) / 2 for i, j < nf (Ki column-major, leading dimension ld)
__global__ void symmetrise_kernel(const double* __restrict__ ki, int64_t ld, int nf, double* __restrict__ p64,
                                  float* __restrict__ p32) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < static_cast<int64_t>(nf) * nf;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / nf, j = t % nf;
    const double v = 0.5 * (ki[j * ld + i] + ki[i * ld + j]);
    p64[t] = v;
    p32[t] = static_cast<float>(v);
  }
}

}  // namespace

void coarse_inverse_device(Context& c, const Dense& K, int nf, void** pinv64, void** pinv32) {
  const int n = K.r;  // nf + 1 (bordered)
  const size_t bytes = static_cast<size_t>(n) * n * sizeof(double);
  double *dA = nullptr, *dB = nullptr, *work = nullptr;
  int *ipiv = nullptr, *info = nullptr;
  cusolverDnHandle_t h = nullptr;
  struct Guard {
    double **a, **b, **w;
    int **p, **i;
    cusolverDnHandle_t* h;
    ~Guard() {
      cudaFree(*a); cudaFree(*b); cudaFree(*w); cudaFree(*p); cudaFree(*i);
      if (*h) cusolverDnDestroy(*h);
    }
  } g{&dA, &dB, &work, &ipiv, &info, &h};
  SMG_CUDA(cudaMalloc(&dA, bytes));
  SMG_CUDA(cudaMalloc(&dB, bytes));
  SMG_CUDA(cudaMalloc(&ipiv, sizeof(int) * n));
  SMG_CUDA(cudaMalloc(&info, sizeof(int)));
  // K is symmetric: its row-major storage is its column-major storage
  SMG_CUDA(cudaMemcpyAsync(dA, K.a.data(), bytes, cudaMemcpyHostToDevice, c.stream));
  identity_kernel<<<1184, 256, 0, c.stream>>>(dB, n);
  SMG_CUDA(cudaGetLastError());
  SMG_CUSOLVER(cusolverDnCreate(&h));
  SMG_CUSOLVER(cusolverDnSetStream(h, c.stream));
  int lwork = 0;
  SMG_CUSOLVER(cusolverDnDgetrf_bufferSize(h, n, n, dA, n, &lwork));
  SMG_CUDA(cudaMalloc(&work, sizeof(double) * std::max(lwork, 1)));
  SMG_CUSOLVER(cusolverDnDgetrf(h, n, n, dA, n, work, ipiv, info));
  SMG_CUSOLVER(cusolverDnDgetrs(h, CUBLAS_OP_N, n, n, dA, n, ipiv, dB, n, info));
  int hinfo = 0;
  SMG_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SMG_CUDA(cudaStreamSynchronize(c.stream));
  if (hinfo != 0) throw cuda_error("coarse solve: LU of the bordered level-0 system failed (info " +
                                   std::to_string(hinfo) + ")");
  void *p64 = nullptr, *p32 = nullptr;
  SMG_CUDA(cudaMalloc(&p64, static_cast<size_t>(nf) * nf * sizeof(double)));
  c.allocations.push_back(p64);
  SMG_CUDA(cudaMalloc(&p32, static_cast<size_t>(nf) * nf * sizeof(float)));
  c.allocations.push_back(p32);
  symmetrise_kernel<<<1184, 256, 0, c.stream>>>(dB, n, nf, static_cast<double*>(p64), static_cast<float*>(p32));
  SMG_CUDA(cudaGetLastError());
  SMG_CUDA(cudaStreamSynchronize(c.stream));
  *pinv64 = p64;
  *pinv32 = p32;
}

}  // namespace smg
