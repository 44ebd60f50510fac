// K1/K2: matrix-free Stokes operator y = A x and residual r = b - A x on sm_100a.
//
// Reference: apply_stokes evaluated by Alg. 1. On the uniform
// Cartesian unit cube the cell/face loops of Alg. 1 equal a Kronecker sum of banded 1D operators
// (verified here against the quadrature-based CPU oracle to 1e-13). Per velocity
// component c with orthogonal axes o1, o2:
//   S  = M_o1 M_o2 u_c                      (DG mass, block diagonal)
//   Tt = L_o1 (M_o2 u_c) + M_o1 (L_o2 u_c)  (DG SIPG, block tridiagonal)
//   y_c = L_c S + M_c Tt + D_c^T (M_o1 M_o2 p)   (C0 stiffness/mass, divergence transpose)
//   y_p += D_c S
// One CTA owns a brick of TX x TY x TZ cells. It stages the input brick plus the halo each banded
// operator needs in shared memory once, performs the seven sum-factorised 1D contractions per
// component in shared memory, and writes each output DoF exactly once: HBM traffic is one read of x
// and one write of y (16 B/DoF in fp64); halo re-reads are served from L2.
#include <cuda_runtime.h>

#include "smg_internal.cuh"

namespace smg {
namespace {

struct Box {
  int lo[3];
  int n[3];
  __device__ int size() const { return n[0] * n[1] * n[2]; }
  __device__ int idx(int x, int y, int z) const { return ((z - lo[2]) * n[1] + (y - lo[1])) * n[0] + (x - lo[0]); }
};

__device__ __forceinline__ int floor_div(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

// Banded 1D contraction along axis AX in shared memory:
//   dst(q) (+)= sum_{delta, b} W[var][delta][a][b] * src(q with q[AX] = (e+delta)(K+1)+b)
// where q[AX] = e (K+1) + a, var = first/interior/last of the global cell e + cell0.
template <typename T, int K, int NB, int AX, int DMIN, int DMAX, bool ACC>
__device__ __forceinline__ void contract(const T* __restrict__ src, const Box& sb, T* __restrict__ dst,
                                         const Box& db, const T* __restrict__ W, int cell0, int m) {
  constexpr int H = K + 1;
  const int total = db.size();
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    int q[3];
    q[0] = db.lo[0] + i % db.n[0];
    q[1] = db.lo[1] + (i / db.n[0]) % db.n[1];
    q[2] = db.lo[2] + i / (db.n[0] * db.n[1]);
    const int g = q[AX];
    const int e = floor_div(g, H);
    const int a = g - e * H;
    const int E = cell0 + e;
    T sum = T(0);
    if (E >= 0 && E < m) {
      const int var = (E == 0) ? 0 : (E == m - 1 ? 2 : 1);
      int sq[3] = {q[0], q[1], q[2]};
#pragma unroll
      for (int d = DMIN; d <= DMAX; ++d) {
        const T* w = W + ((var * 3 + d + 1) * H + a) * (K + 2);
        const int base = (e + d) * H;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int s = base + b;
          if (s >= sb.lo[AX] && s < sb.lo[AX] + sb.n[AX]) {
            sq[AX] = s;
            sum += w[b] * src[sb.idx(sq[0], sq[1], sq[2])];
          }
        }
      }
    }
    const int o = db.idx(q[0], q[1], q[2]);
    dst[o] = ACC ? dst[o] + sum : sum;
  }
}

template <int K, int TX, int TY, int TZ>
struct Plan {
  static constexpr int H = K + 1;
  static constexpr int Nax(int a) { return (a == 0 ? TX : (a == 1 ? TY : TZ)) * H; }
  static constexpr int o1(int c) { return c == 0 ? 1 : 0; }
  static constexpr int o2(int c) { return c == 2 ? 1 : 2; }
  static constexpr int par_n(int c) { return Nax(c) + K + 2; }  // [-H, N_c]
  static constexpr int halo_n(int a) { return Nax(a) + 2 * H; }  // [-H, N+H)
  static constexpr int sizeU(int c) { return par_n(c) * halo_n(o1(c)) * halo_n(o2(c)); }
  static constexpr int sizeA1(int c) { return par_n(c) * halo_n(o1(c)) * Nax(o2(c)); }
  static constexpr int sizeB1(int c) { return par_n(c) * Nax(o1(c)) * Nax(o2(c)); }
  static constexpr int sizeQ(int c) { return (Nax(c) + H) * Nax(o1(c)) * Nax(o2(c)); }
  static constexpr int mx(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
  static constexpr int U = mx(sizeU(0), sizeU(1), sizeU(2));
  static constexpr int A1 = mx(mx(sizeA1(0), sizeA1(1), sizeA1(2)), sizeQ(0), mx(sizeQ(1), sizeQ(2), 0));
  static constexpr int B1 = mx(sizeB1(0), sizeB1(1), sizeB1(2));
  static constexpr int Q = mx(sizeQ(0), sizeQ(1), sizeQ(2));
  static constexpr int P = (Nax(0) + H) * (Nax(1) + H) * (Nax(2) + H);
  static constexpr int YP = Nax(0) * Nax(1) * Nax(2);
  static constexpr int TAB = N_OPS * 9 * (K + 1) * (K + 2);
  static constexpr bool ALIAS = 2 * B1 <= U;  // S, Tt live in the dead U buffer when they fit
  static constexpr int TOTAL = TAB + P + YP + Q + U + A1 + B1 + (ALIAS ? 0 : 2 * B1);
};

template <typename T, int K, int TX, int TY, int TZ, bool RESID>
__global__ void __launch_bounds__(256) stokes_vmult_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                           const T* __restrict__ b, const T* __restrict__ ops,
                                                           int m) {
  using PL = Plan<K, TX, TY, TZ>;
  constexpr int H = K + 1;
  constexpr int OPS = 9 * (K + 1) * (K + 2);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* W = reinterpret_cast<T*>(smem_raw);
  T* sP = W + PL::TAB;
  T* sYP = sP + PL::P;
  T* sQ = sYP + PL::YP;
  T* sU = sQ + PL::Q;
  T* sA1 = sU + PL::U;
  T* sB1 = sA1 + PL::A1;
  T* sS = PL::ALIAS ? sU : sB1 + PL::B1;  // U is dead once A1, B1 exist
  T* sT = sS + PL::B1;

  const int n = m * H;
  const int c0[3] = {static_cast<int>(blockIdx.x) * TX, static_cast<int>(blockIdx.y) * TY,
                     static_cast<int>(blockIdx.z) * TZ};
  const int g0[3] = {c0[0] * H, c0[1] * H, c0[2] * H};
  const int64_t sizeV = static_cast<int64_t>(n + 1) * n * n;
  const int64_t offP = 3 * sizeV;

  for (int i = threadIdx.x; i < PL::TAB; i += blockDim.x) W[i] = ops[i];
  // pressure box with a one-cell halo on the low side of every axis
  Box bP;
  for (int a = 0; a < 3; ++a) { bP.lo[a] = -H; bP.n[a] = PL::Nax(a) + H; }
  for (int i = threadIdx.x; i < PL::P; i += blockDim.x) {
    const int lx = i % bP.n[0] - H, ly = (i / bP.n[0]) % bP.n[1] - H, lz = i / (bP.n[0] * bP.n[1]) - H;
    const int gx = g0[0] + lx, gy = g0[1] + ly, gz = g0[2] + lz;
    T v = T(0);
    if (gx >= 0 && gx < n && gy >= 0 && gy < n && gz >= 0 && gz < n)
      v = x[offP + (static_cast<int64_t>(gz) * n + gy) * n + gx];
    sP[i] = v;
  }
  for (int i = threadIdx.x; i < PL::YP; i += blockDim.x) sYP[i] = T(0);
  __syncthreads();

#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    const int o1 = PL::o1(c), o2 = PL::o2(c);
    const int64_t offc = c * sizeV;
    int64_t gd[3] = {n, n, n};
    gd[c] = n + 1;
    // ---- stage U (x_c with halos; constrained boundary-normal entries read as 0) ----
    Box bU;
    bU.lo[c] = -H; bU.n[c] = PL::Nax(c) + K + 2;
    bU.lo[o1] = -H; bU.n[o1] = PL::Nax(o1) + 2 * H;
    bU.lo[o2] = -H; bU.n[o2] = PL::Nax(o2) + 2 * H;
    for (int i = threadIdx.x; i < bU.size(); i += blockDim.x) {
      int l[3] = {i % bU.n[0] + bU.lo[0], (i / bU.n[0]) % bU.n[1] + bU.lo[1], i / (bU.n[0] * bU.n[1]) + bU.lo[2]};
      int g[3] = {g0[0] + l[0], g0[1] + l[1], g0[2] + l[2]};
      bool ok = g[0] >= 0 && g[1] >= 0 && g[2] >= 0 && g[0] < gd[0] && g[1] < gd[1] && g[2] < gd[2];
      ok = ok && g[c] != 0 && g[c] != n;
      sU[i] = ok ? x[offc + (static_cast<int64_t>(g[2]) * gd[1] + g[1]) * gd[0] + g[0]] : T(0);
    }
    // ---- Q = M_o1 M_o2 p over [-H, N_c) x owned x owned ----
    Box bQ2;
    bQ2.lo[c] = -H; bQ2.n[c] = PL::Nax(c) + H;
    bQ2.lo[o1] = 0; bQ2.n[o1] = PL::Nax(o1);
    bQ2.lo[o2] = 0; bQ2.n[o2] = PL::Nax(o2);
    T* sQ2 = sA1;
    if (o2 == 1) contract<T, K, K + 1, 1, 0, 0, false>(sP, bP, sQ2, bQ2, W + OP_MO * OPS, c0[1], m);
    else contract<T, K, K + 1, 2, 0, 0, false>(sP, bP, sQ2, bQ2, W + OP_MO * OPS, c0[2], m);
    __syncthreads();
    if (o1 == 0) contract<T, K, K + 1, 0, 0, 0, false>(sQ2, bQ2, sQ, bQ2, W + OP_MO * OPS, c0[0], m);
    else contract<T, K, K + 1, 1, 0, 0, false>(sQ2, bQ2, sQ, bQ2, W + OP_MO * OPS, c0[1], m);
    __syncthreads();
    // ---- A1 = M_o2 U (o1 keeps its halo), B1 = L_o2 U ----
    Box bA1 = bU;
    bA1.lo[o2] = 0; bA1.n[o2] = PL::Nax(o2);
    Box bB1 = bA1;
    bB1.lo[o1] = 0; bB1.n[o1] = PL::Nax(o1);
    if (o2 == 1) {
      contract<T, K, K + 1, 1, 0, 0, false>(sU, bU, sA1, bA1, W + OP_MO * OPS, c0[1], m);
      contract<T, K, K + 1, 1, -1, 1, false>(sU, bU, sB1, bB1, W + OP_LO * OPS, c0[1], m);
    } else {
      contract<T, K, K + 1, 2, 0, 0, false>(sU, bU, sA1, bA1, W + OP_MO * OPS, c0[2], m);
      contract<T, K, K + 1, 2, -1, 1, false>(sU, bU, sB1, bB1, W + OP_LO * OPS, c0[2], m);
    }
    __syncthreads();
    // ---- S = M_o1 A1 ; Tt = L_o1 A1 + M_o1 B1 ----
    if (o1 == 0) {
      contract<T, K, K + 1, 0, 0, 0, false>(sA1, bA1, sS, bB1, W + OP_MO * OPS, c0[0], m);
      contract<T, K, K + 1, 0, -1, 1, false>(sA1, bA1, sT, bB1, W + OP_LO * OPS, c0[0], m);
    } else {
      contract<T, K, K + 1, 1, 0, 0, false>(sA1, bA1, sS, bB1, W + OP_MO * OPS, c0[1], m);
      contract<T, K, K + 1, 1, -1, 1, false>(sA1, bA1, sT, bB1, W + OP_LO * OPS, c0[1], m);
    }
    __syncthreads();
    if (o1 == 0) contract<T, K, K + 1, 0, 0, 0, true>(sB1, bB1, sT, bB1, W + OP_MO * OPS, c0[0], m);
    else contract<T, K, K + 1, 1, 0, 0, true>(sB1, bB1, sT, bB1, W + OP_MO * OPS, c0[1], m);
    __syncthreads();
    // ---- y_c = L_c S + M_c Tt + D_c^T Q over the owned box; y_p += D_c S ----
    Box bY;
    for (int a = 0; a < 3; ++a) { bY.lo[a] = 0; bY.n[a] = PL::Nax(a); }
    // reuse sA1 (dead) for the three contributions, then write out
    T* sY = sA1;
    if (c == 0) {
      contract<T, K, K + 2, 0, -1, 0, false>(sS, bB1, sY, bY, W + OP_LP * OPS, c0[0], m);
      contract<T, K, K + 2, 0, -1, 0, true>(sT, bB1, sY, bY, W + OP_MP * OPS, c0[0], m);
      contract<T, K, K + 1, 0, -1, 0, true>(sQ, bQ2, sY, bY, W + OP_DT * OPS, c0[0], m);
      contract<T, K, K + 2, 0, 0, 0, true>(sS, bB1, sYP, bY, W + OP_D * OPS, c0[0], m);
    } else if (c == 1) {
      contract<T, K, K + 2, 1, -1, 0, false>(sS, bB1, sY, bY, W + OP_LP * OPS, c0[1], m);
      contract<T, K, K + 2, 1, -1, 0, true>(sT, bB1, sY, bY, W + OP_MP * OPS, c0[1], m);
      contract<T, K, K + 1, 1, -1, 0, true>(sQ, bQ2, sY, bY, W + OP_DT * OPS, c0[1], m);
      contract<T, K, K + 2, 1, 0, 0, true>(sS, bB1, sYP, bY, W + OP_D * OPS, c0[1], m);
    } else {
      contract<T, K, K + 2, 2, -1, 0, false>(sS, bB1, sY, bY, W + OP_LP * OPS, c0[2], m);
      contract<T, K, K + 2, 2, -1, 0, true>(sT, bB1, sY, bY, W + OP_MP * OPS, c0[2], m);
      contract<T, K, K + 1, 2, -1, 0, true>(sQ, bQ2, sY, bY, W + OP_DT * OPS, c0[2], m);
      contract<T, K, K + 2, 2, 0, 0, true>(sS, bB1, sYP, bY, W + OP_D * OPS, c0[2], m);
    }
    // (each thread reads back exactly the sY / sYP entries it wrote: no barrier needed here)
    for (int i = threadIdx.x; i < bY.size(); i += blockDim.x) {
      int l[3] = {i % bY.n[0], (i / bY.n[0]) % bY.n[1], i / (bY.n[0] * bY.n[1])};
      int g[3] = {g0[0] + l[0], g0[1] + l[1], g0[2] + l[2]};
      if (g[0] >= n || g[1] >= n || g[2] >= n) continue;  // partial brick beyond the mesh
      const int64_t gi = offc + (static_cast<int64_t>(g[2]) * gd[1] + g[1]) * gd[0] + g[0];
      T v = sY[i];
      if (g[c] == 0) v = T(0);  // constrained
      else if (RESID) v = b[gi] - v;
      y[gi] = v;
    }
    // the constrained plane g_c = n belongs to the last brick along c
    if (c0[c] + (c == 0 ? TX : (c == 1 ? TY : TZ)) >= m) {
      const int na = PL::Nax(o1), nb = PL::Nax(o2);
      for (int i = threadIdx.x; i < na * nb; i += blockDim.x) {
        int g[3];
        g[c] = n;
        g[o1] = g0[o1] + i % na;
        g[o2] = g0[o2] + i / na;
        if (g[o1] >= n || g[o2] >= n) continue;
        y[offc + (static_cast<int64_t>(g[2]) * gd[1] + g[1]) * gd[0] + g[0]] = T(0);
      }
    }
    __syncthreads();
  }
  // ---- pressure rows ----
  for (int i = threadIdx.x; i < PL::YP; i += blockDim.x) {
    const int lx = i % PL::Nax(0), ly = (i / PL::Nax(0)) % PL::Nax(1), lz = i / (PL::Nax(0) * PL::Nax(1));
    const int gx = g0[0] + lx, gy = g0[1] + ly, gz = g0[2] + lz;
    if (gx >= n || gy >= n || gz >= n) continue;
    const int64_t gi = offP + (static_cast<int64_t>(gz) * n + gy) * n + gx;
    y[gi] = RESID ? b[gi] - sYP[i] : sYP[i];
  }
}

template <typename T, int K, int TX, int TY, int TZ>
void launch_t(Context& ctx, int level, void* y, const void* x, const void* b) {
  using PL = Plan<K, TX, TY, TZ>;
  const DevLevel& dl = ctx.dev[sizeof(T) == 8 ? 0 : 1][level];
  const int m = dl.lay.m;
  dim3 grid((m + TX - 1) / TX, (m + TY - 1) / TY, (m + TZ - 1) / TZ);
  const size_t smem = sizeof(T) * PL::TOTAL;
  if (b) {
    auto kern = stokes_vmult_kernel<T, K, TX, TY, TZ, true>;
    SMG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, 256, smem, ctx.stream>>>(static_cast<const T*>(x), static_cast<T*>(y), static_cast<const T*>(b),
                                          static_cast<const T*>(dl.ops), m);
  } else {
    auto kern = stokes_vmult_kernel<T, K, TX, TY, TZ, false>;
    SMG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, 256, smem, ctx.stream>>>(static_cast<const T*>(x), static_cast<T*>(y), nullptr,
                                          static_cast<const T*>(dl.ops), m);
  }
  SMG_CUDA(cudaGetLastError());
  ++ctx.launches;
}

template <typename T>
void launch_prec(Context& ctx, int level, void* y, const void* x, const void* b) {
  switch (ctx.cfg.degree) {
    case 1: launch_t<T, 1, 8, 4, 4>(ctx, level, y, x, b); break;
    case 2: launch_t<T, 2, 4, 4, 4>(ctx, level, y, x, b); break;
    case 3: launch_t<T, 3, 4, 2, 2>(ctx, level, y, x, b); break;
    case 4: launch_t<T, 4, 2, 2, 2>(ctx, level, y, x, b); break;
    case 5: launch_t<T, 5, 2, 2, 1>(ctx, level, y, x, b); break;
    case 6: launch_t<T, 6, 2, 1, 1>(ctx, level, y, x, b); break;
    case 7: launch_t<T, 7, 2, 1, 1>(ctx, level, y, x, b); break;
    default: throw std::invalid_argument("degree not supported by the vmult kernel (1..7)");
  }
}

}  // namespace

void launch_vmult(Context& ctx, int level, int prec, void* y, const void* x, const void* b) {
  if (prec == SMG_F64) launch_prec<double>(ctx, level, y, x, b);
  else launch_prec<float>(ctx, level, y, x, b);
}

}  // namespace smg
