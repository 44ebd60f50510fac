// K5: BLAS-1 on level vectors (block_vector.hpp:52-93). Grid-stride, vectorised where aligned;
// dots accumulate in fp64 (block_vector.hpp:53-61) with a fixed-shape two-pass reduction, so results
// are deterministic run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "smg_internal.cuh"

namespace smg {
namespace {

constexpr int kThreads = 256;

template <typename T>
__global__ void dot_partial_kernel(const T* __restrict__ a, const T* __restrict__ b, int64_t n,
                                   double* __restrict__ partial) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s += static_cast<double>(a[i]) * static_cast<double>(b[i]);
  __shared__ double red[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

__global__ void dot_final_kernel(const double* __restrict__ partial, int nparts, double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[i];
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[0] = s;
  }
}

template <typename T>
__global__ void axpby_kernel(int64_t n, T alpha, const T* __restrict__ x, T beta, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = alpha * x[i] + beta * y[i];
}

template <typename T>
__global__ void axpy_kernel(int64_t n, T alpha, const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] += alpha * x[i];
}

template <typename T>
__global__ void scale_kernel(int64_t n, T alpha, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] *= alpha;
}

template <typename T>
__global__ void add_scalar_kernel(int64_t n, T alpha, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] += alpha;
}

template <typename D, typename S>
__global__ void convert_kernel(int64_t n, D* __restrict__ dst, const S* __restrict__ src) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<D>(src[i]);
}

// mass-weighted pressure mean: sum_i w(i) p_i with w separable per node
template <typename T>
__global__ void pmean_partial_kernel(const T* __restrict__ p, int n, int nb, const double* __restrict__ w1,
                                     double* __restrict__ partial) {
  double s = 0.0;
  const int64_t total = static_cast<int64_t>(n) * n * n;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int x = static_cast<int>(i % n), y = static_cast<int>((i / n) % n), z = static_cast<int>(i / (int64_t(n) * n));
    s += w1[x % nb] * w1[y % nb] * w1[z % nb] * static_cast<double>(p[i]);
  }
  __shared__ double red[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

template <typename T>
__global__ void sub_scalar_kernel(int64_t n, T* __restrict__ p, const double* __restrict__ sum, double inv_w) {
  const T mean = static_cast<T>(sum[0] * inv_w);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] -= mean;
}

// pressure block: global lexicographic (device layout) <-> cell-local lexicographic (the reference's
// DoFLayout: cells x-fastest, (k+1)^3 nodes per cell x-fastest). One thread per DoF,
// indexed by the global lexicographic position (coalesced on that side).
template <typename T, bool TO_CELL>
__global__ void pressure_permute_kernel(T* __restrict__ dst, const T* __restrict__ src, int m, int H, int64_t begin,
                                        int64_t end) {
  const int n = m * H;
  for (int64_t i = begin + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < end;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int gx = static_cast<int>(i % n), gy = static_cast<int>((i / n) % n), gz = static_cast<int>(i / (int64_t(n) * n));
    const int64_t cell = (static_cast<int64_t>(gz / H) * m + gy / H) * m + gx / H;
    const int64_t c = cell * H * H * H + ((gz % H) * H + gy % H) * H + gx % H;
    if (TO_CELL) dst[c] = src[i];
    else dst[i] = src[c];
  }
}

// out[i] = <V_i, w> for i < nv (fp64), blockIdx.y = i: one launch + one final reduction for all the
// Gram-Schmidt coefficients of an FGMRES iteration
__global__ void multidot_partial_kernel(const double* const* __restrict__ V, const double* __restrict__ w, int64_t n,
                                        double* __restrict__ partial) {
  const double* v = V[blockIdx.y];
  double s = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s += v[i] * w[i];
  __shared__ double red[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}
__global__ void multidot_final_kernel(const double* __restrict__ partial, int nparts, double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[blockIdx.x * nparts + i];
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
  }
}
// w -= sum_i coef[i] V_i (coefficients on the device: no host round trip between the passes)
__global__ void multi_axpy_kernel(const double* const* __restrict__ V, const double* __restrict__ coef, int nv,
                                  int64_t n, double* __restrict__ w) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = w[i];
    for (int j = 0; j < nv; ++j) s -= coef[j] * V[j][i];
    w[i] = s;
  }
}

int grid_for(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return static_cast<int>(g < kDotBlocks ? (g < 1 ? 1 : g) : kDotBlocks);
}

}  // namespace

size_t elem_size(int precision) { return precision == SMG_F64 ? 8 : 4; }

double dot(Context& c, int64_t n, int prec, const void* a, const void* b) {
  const int g = grid_for(n);
  double* part = static_cast<double*>(c.dot_partials);
  if (prec == SMG_F64)
    dot_partial_kernel<double><<<g, kThreads, 0, c.stream>>>(static_cast<const double*>(a),
                                                              static_cast<const double*>(b), n, part);
  else
    dot_partial_kernel<float><<<g, kThreads, 0, c.stream>>>(static_cast<const float*>(a),
                                                             static_cast<const float*>(b), n, part);
  dot_final_kernel<<<1, 1024, 0, c.stream>>>(part, g, part + kDotBlocks);
  c.launches += 2;
  SMG_CUDA(cudaGetLastError());
  double* h = static_cast<double*>(c.dot_host);
  SMG_CUDA(cudaMemcpyAsync(h, part + kDotBlocks, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  SMG_CUDA(cudaStreamSynchronize(c.stream));
  return h[0];
}

// dot over several contiguous index ranges of the same two vectors (the owned part of a z-slab)
double dot_ranges(Context& c, int prec, const void* a, const void* b, const int64_t* begin, const int64_t* len,
                  int nranges) {
  double* part = static_cast<double*>(c.dot_partials);
  const size_t es = elem_size(prec);
  const int per = kDotBlocks / 4;
  int used = 0;
  for (int r = 0; r < nranges && r < 4; ++r) {
    if (len[r] <= 0) continue;
    const int g = std::min(grid_for(len[r]), per);
    const char* pa = static_cast<const char*>(a) + begin[r] * es;
    const char* pb = static_cast<const char*>(b) + begin[r] * es;
    if (prec == SMG_F64)
      dot_partial_kernel<double><<<g, kThreads, 0, c.stream>>>(reinterpret_cast<const double*>(pa),
                                                                reinterpret_cast<const double*>(pb), len[r], part + used);
    else
      dot_partial_kernel<float><<<g, kThreads, 0, c.stream>>>(reinterpret_cast<const float*>(pa),
                                                               reinterpret_cast<const float*>(pb), len[r], part + used);
    used += g;
    ++c.launches;
  }
  if (used == 0) return 0.0;
  dot_final_kernel<<<1, 1024, 0, c.stream>>>(part, used, part + kDotBlocks);
  ++c.launches;
  SMG_CUDA(cudaGetLastError());
  double* h = static_cast<double*>(c.dot_host);
  SMG_CUDA(cudaMemcpyAsync(h, part + kDotBlocks, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  SMG_CUDA(cudaStreamSynchronize(c.stream));
  return h[0];
}

void launch_multidot(Context& c, int64_t n, const double* const* V_dev, int nv, const double* w, double* out_dev) {
  const int per = std::max(1, std::min(grid_for(n), kDotBlocks / std::max(nv, 1)));
  double* part = static_cast<double*>(c.multidot_partials);
  multidot_partial_kernel<<<dim3(per, nv), kThreads, 0, c.stream>>>(V_dev, w, n, part);
  multidot_final_kernel<<<nv, 1024, 0, c.stream>>>(part, per, out_dev);
  c.launches += 2;
  SMG_CUDA(cudaGetLastError());
}

void launch_multi_axpy(Context& c, int64_t n, const double* const* V_dev, int nv, const double* coef_dev, double* w) {
  multi_axpy_kernel<<<grid_for(n), kThreads, 0, c.stream>>>(V_dev, coef_dev, nv, n, w);
  ++c.launches;
  SMG_CUDA(cudaGetLastError());
}

void launch_axpy(Context& c, int64_t n, int prec, double alpha, const void* x, void* y) {
  if (prec == SMG_F64)
    axpy_kernel<double><<<grid_for(n), kThreads, 0, c.stream>>>(n, alpha, static_cast<const double*>(x),
                                                                static_cast<double*>(y));
  else
    axpy_kernel<float><<<grid_for(n), kThreads, 0, c.stream>>>(n, static_cast<float>(alpha),
                                                               static_cast<const float*>(x), static_cast<float*>(y));
  ++c.launches;
  SMG_CUDA(cudaGetLastError());
}

void launch_axpby(Context& c, int64_t n, int prec, double alpha, const void* x, double beta, void* y) {
  if (prec == SMG_F64)
    axpby_kernel<double><<<grid_for(n), kThreads, 0, c.stream>>>(n, alpha, static_cast<const double*>(x), beta,
                                                                 static_cast<double*>(y));
  else
    axpby_kernel<float><<<grid_for(n), kThreads, 0, c.stream>>>(n, static_cast<float>(alpha),
                                                                static_cast<const float*>(x),
                                                                static_cast<float>(beta), static_cast<float*>(y));
  ++c.launches;
  SMG_CUDA(cudaGetLastError());
}

void launch_scale(Context& c, int64_t n, int prec, double alpha, void* x) {
  if (prec == SMG_F64)
    scale_kernel<double><<<grid_for(n), kThreads, 0, c.stream>>>(n, alpha, static_cast<double*>(x));
  else
    scale_kernel<float><<<grid_for(n), kThreads, 0, c.stream>>>(n, static_cast<float>(alpha), static_cast<float*>(x));
  ++c.launches;
  SMG_CUDA(cudaGetLastError());
}

void launch_add_scalar(Context& c, int64_t n, int prec, double alpha, void* x) {
  if (prec == SMG_F64)
    add_scalar_kernel<double><<<grid_for(n), kThreads, 0, c.stream>>>(n, alpha, static_cast<double*>(x));
  else
    add_scalar_kernel<float><<<grid_for(n), kThreads, 0, c.stream>>>(n, static_cast<float>(alpha),
                                                                      static_cast<float*>(x));
  ++c.launches;
  SMG_CUDA(cudaGetLastError());
}

void launch_zero(Context& c, int64_t n, int prec, void* x) {
  SMG_CUDA(cudaMemsetAsync(x, 0, static_cast<size_t>(n) * elem_size(prec), c.stream));
}

void launch_convert(Context& c, int64_t n, int dst_prec, void* dst, int src_prec, const void* src) {
  const int g = grid_for(n);
  if (dst_prec == src_prec) {
    SMG_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(n) * elem_size(dst_prec), cudaMemcpyDeviceToDevice,
                             c.stream));
    return;
  }
  if (dst_prec == SMG_F32)
    convert_kernel<float, double><<<g, kThreads, 0, c.stream>>>(n, static_cast<float*>(dst),
                                                                 static_cast<const double*>(src));
  else
    convert_kernel<double, float><<<g, kThreads, 0, c.stream>>>(n, static_cast<double*>(dst),
                                                                 static_cast<const float*>(src));
  ++c.launches;
  SMG_CUDA(cudaGetLastError());
}

void launch_pressure_permute(Context& c, int level, int prec, void* dst, const void* src, bool to_cell_local, int z0,
                             int z1, cudaStream_t stream) {
  const LevelLayout& lay = c.dev[0][level].lay;
  const int H = c.cfg.degree + 1;
  if (z1 < 0) z1 = lay.m;
  // the pressure of the cells [z0, z1) is the global-lexicographic range of their node planes (and a
  // contiguous range of the cell-local numbering as well)
  const int64_t plane = static_cast<int64_t>(lay.n) * lay.n;
  const int64_t begin = static_cast<int64_t>(z0) * H * plane, end = static_cast<int64_t>(z1) * H * plane;
  const int g = grid_for(end - begin);
  if (stream == nullptr) stream = c.stream;
  auto go = [&](auto* d, auto* s) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(s)>>;
    if (to_cell_local) pressure_permute_kernel<T, true><<<g, kThreads, 0, stream>>>(d, s, lay.m, H, begin, end);
    else pressure_permute_kernel<T, false><<<g, kThreads, 0, stream>>>(d, s, lay.m, H, begin, end);
  };
  if (prec == SMG_F64) go(static_cast<double*>(dst), static_cast<const double*>(src));
  else go(static_cast<float*>(dst), static_cast<const float*>(src));
  ++c.launches;
  SMG_CUDA(cudaGetLastError());
}

void launch_sub_pressure_mean(Context& c, int level, int prec, void* x) {
  const DevLevel& dl = c.dev[prec][level];
  const int n = dl.lay.n, nb = c.cfg.degree + 1;
  const int64_t np = dl.lay.size[3];
  const int g = grid_for(np);
  double* part = static_cast<double*>(c.dot_partials);
  const double* w1 = static_cast<const double*>(c.dev[0][level].pweights);
  char* p = static_cast<char*>(x) + dl.lay.off[3] * elem_size(prec);
  if (prec == SMG_F64)
    pmean_partial_kernel<double><<<g, kThreads, 0, c.stream>>>(reinterpret_cast<const double*>(p), n, nb, w1, part);
  else
    pmean_partial_kernel<float><<<g, kThreads, 0, c.stream>>>(reinterpret_cast<const float*>(p), n, nb, w1, part);
  dot_final_kernel<<<1, 1024, 0, c.stream>>>(part, g, part + kDotBlocks);
  // total weight: (sum_a w_a)^3 per cell times m^3 cells, in reference-cell units
  double ws = 0.0;
  for (double v : pressure_node_weights(c.cfg.degree)) ws += v;
  const double wtot = ws * ws * ws * double(dl.lay.m) * dl.lay.m * dl.lay.m;
  if (prec == SMG_F64)
    sub_scalar_kernel<double><<<g, kThreads, 0, c.stream>>>(np, reinterpret_cast<double*>(p), part + kDotBlocks,
                                                            1.0 / wtot);
  else
    sub_scalar_kernel<float><<<g, kThreads, 0, c.stream>>>(np, reinterpret_cast<float*>(p), part + kDotBlocks,
                                                           1.0 / wtot);
  c.launches += 3;
  SMG_CUDA(cudaGetLastError());
}

}  // namespace smg
