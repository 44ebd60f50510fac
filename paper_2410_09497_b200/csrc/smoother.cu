// K3: vertex-patch multiplicative Schwarz smoother, one colour per launch (smooth SPEC.md:400-408,
// Alg. 2). One CTA owns one patch (the 8 cells around an interior vertex) of the
// colour; it gathers the patch residual into shared memory, runs the local Schur-complement solve
// (schur_solve SPEC.md:356-364) entirely in shared memory —
//   S P = B A^-1 F - G,  S = B A^-1 B^T (fast diagonalisation, Eq. 9), projected CG with
//   the pressure-mass preconditioner —
// and adds R^T (U, P) into x. Same-colour patches write disjoint DoFs, so the update is
// race-free and independent of CTA order. The residual r = b - A x is refreshed per colour by the
// vmult kernel in residual mode.
#include <cuda_runtime.h>

#include "smg_internal.cuh"

namespace smg {
namespace {

constexpr int kPatchThreads = 128;

template <int K>
struct PatchDims {
  static constexpr int NP = 2 * K + 1;  // parallel (C0, interior nodes)
  static constexpr int NO = 2 * K + 2;  // orthogonal (DG) / pressure
  static constexpr int NV = NP * NO * NO;
  static constexpr int NPR = NO * NO * NO;
  // packed table offsets
  static constexpr int PAR_S = 0;
  static constexpr int PAR_L = PAR_S + NP * NP;
  static constexpr int ORTH_S = PAR_L + NP;
  static constexpr int ORTH_L = ORTH_S + 4 * NO * NO;
  static constexpr int DM = ORTH_L + 4 * NO;
  static constexpr int MP = DM + NO * NP;
  static constexpr int MPI = MP + NO * NO;
  static constexpr int TAB = MPI + NO * NO;
};

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // protect red from a previous use
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  T s = T(0);
#pragma unroll
  for (int w = 0; w < kPatchThreads / 32; ++w) s += red[w];
  return s;
}

// out (dims with axis ax replaced by R) = M applied along axis ax of in (dims d)
// M(i,j) = trans ? A[j*lda + i] : A[i*lda + j], j < C = d[ax]
template <typename T>
__device__ void axis_apply(const T* __restrict__ in, int d0, int d1, int d2, int ax, const T* __restrict__ A, int lda,
                           int R, bool trans, T* __restrict__ out) {
  int din[3] = {d0, d1, d2};
  int dout[3] = {d0, d1, d2};
  const int C = din[ax];
  dout[ax] = R;
  const int sin_ax = ax == 0 ? 1 : (ax == 1 ? d0 : d0 * d1);
  const int total = dout[0] * dout[1] * dout[2];
  for (int o = threadIdx.x; o < total; o += blockDim.x) {
    const int x = o % dout[0], y = (o / dout[0]) % dout[1], z = o / (dout[0] * dout[1]);
    const int q[3] = {x, y, z};
    const int i = q[ax];
    int base[3] = {x, y, z};
    base[ax] = 0;
    const T* src = in + (base[2] * din[1] + base[1]) * din[0] + base[0];
    T s = T(0);
    if (trans)
      for (int j = 0; j < C; ++j) s += A[j * lda + i] * src[j * sin_ax];
    else
      for (int j = 0; j < C; ++j) s += A[i * lda + j] * src[j * sin_ax];
    out[o] = s;
  }
}

template <typename T, int K>
struct PatchSolver {
  using PD = PatchDims<K>;
  const T* tab;
  int var[3];  // orthogonal-axis variant per axis
  T* red;

  __device__ const T* S(int c, int a) const {
    return a == c ? tab + PD::PAR_S : tab + PD::ORTH_S + var[a] * PD::NO * PD::NO;
  }
  __device__ const T* L(int c, int a) const { return a == c ? tab + PD::PAR_L : tab + PD::ORTH_L + var[a] * PD::NO; }
  __device__ int dim(int c, int a) const { return a == c ? PD::NP : PD::NO; }

  // out = A_c^-1 in (fast diagonalisation); t is scratch of NV. in may alias out.
  __device__ void ainv(int c, const T* in, T* out, T* t) const {
    const int d0 = dim(c, 0), d1 = dim(c, 1), d2 = dim(c, 2);
    axis_apply(in, d0, d1, d2, 0, S(c, 0), d0, d0, true, t);
    __syncthreads();
    axis_apply(t, d0, d1, d2, 1, S(c, 1), d1, d1, true, out);
    __syncthreads();
    axis_apply(out, d0, d1, d2, 2, S(c, 2), d2, d2, true, t);
    __syncthreads();
    const T* l0 = L(c, 0);
    const T* l1 = L(c, 1);
    const T* l2 = L(c, 2);
    for (int o = threadIdx.x; o < PD::NV; o += blockDim.x) {
      const int x = o % d0, y = (o / d0) % d1, z = o / (d0 * d1);
      t[o] /= (l0[x] + l1[y] + l2[z]);
    }
    __syncthreads();
    axis_apply(t, d0, d1, d2, 2, S(c, 2), d2, d2, false, out);
    __syncthreads();
    axis_apply(out, d0, d1, d2, 1, S(c, 1), d1, d1, false, t);
    __syncthreads();
    axis_apply(t, d0, d1, d2, 0, S(c, 0), d0, d0, false, out);
    __syncthreads();
  }
  // p (NPR) = B_c u ; t scratch of max(NV,NPR)*... two buffers t1,t2 of NPR
  __device__ void bmul(int c, const T* u, T* p, T* t1) const {
    // along c: D (NO x NP); others: Mp (NO x NO)
    int d[3] = {dim(c, 0), dim(c, 1), dim(c, 2)};
    const T* Dm = tab + PD::DM;
    const T* Mp = tab + PD::MP;
    axis_apply(u, d[0], d[1], d[2], 0, c == 0 ? Dm : Mp, c == 0 ? PD::NP : PD::NO, PD::NO, false, t1);
    d[0] = PD::NO;
    __syncthreads();
    axis_apply(t1, d[0], d[1], d[2], 1, c == 1 ? Dm : Mp, c == 1 ? PD::NP : PD::NO, PD::NO, false, p);
    d[1] = PD::NO;
    __syncthreads();
    axis_apply(p, d[0], d[1], d[2], 2, c == 2 ? Dm : Mp, c == 2 ? PD::NP : PD::NO, PD::NO, false, t1);
    __syncthreads();
    for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) p[o] = t1[o];
    __syncthreads();
  }
  // u (NV) = B_c^T p
  __device__ void btmul(int c, const T* p, T* u, T* t1) const {
    const T* Dm = tab + PD::DM;
    const T* Mp = tab + PD::MP;
    int d[3] = {PD::NO, PD::NO, PD::NO};
    axis_apply(p, d[0], d[1], d[2], 2, c == 2 ? Dm : Mp, c == 2 ? PD::NP : PD::NO, dim(c, 2), true, t1);
    d[2] = dim(c, 2);
    __syncthreads();
    axis_apply(t1, d[0], d[1], d[2], 1, c == 1 ? Dm : Mp, c == 1 ? PD::NP : PD::NO, dim(c, 1), true, u);
    d[1] = dim(c, 1);
    __syncthreads();
    axis_apply(u, d[0], d[1], d[2], 0, c == 0 ? Dm : Mp, c == 0 ? PD::NP : PD::NO, dim(c, 0), true, t1);
    __syncthreads();
    for (int o = threadIdx.x; o < PD::NV; o += blockDim.x) u[o] = t1[o];
    __syncthreads();
  }
  __device__ void project(T* p) const {
    T s = T(0);
    for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) s += p[o];
    s = block_sum(s, red) / T(PD::NPR);
    for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) p[o] -= s;
    __syncthreads();
  }
  __device__ T dotp(const T* a, const T* b) const {
    T s = T(0);
    for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) s += a[o] * b[o];
    return block_sum(s, red);
  }
};

template <typename T, int K>
__global__ void __launch_bounds__(kPatchThreads) patch_smooth_kernel(T* __restrict__ x, const T* __restrict__ r,
                                                                     const T* __restrict__ ptab, int m, int colour,
                                                                     int cg_max_iter, T cg_tol, int cg_fixed,
                                                                     int cg_precond) {
  using PD = PatchDims<K>;
  constexpr int H = K + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tab = reinterpret_cast<T*>(smem_raw);
  T* F = tab + ((PD::TAB + 1) / 2) * 2;  // 3 x NV
  constexpr int BIG = PD::NV > PD::NPR ? PD::NV : PD::NPR;
  T* V1 = F + 3 * PD::NV;  // velocity scratch (holds NO^3 intermediates of B^T)
  T* V2 = V1 + BIG;        // scratch
  T* Pr = V2 + BIG;       // rhs / residual
  T* Pz = Pr + PD::NPR;   // preconditioned residual
  T* Pd = Pz + PD::NPR;   // search direction
  T* Pq = Pd + PD::NPR;   // S d
  T* Px = Pq + PD::NPR;   // solution
  T* Pt = Px + PD::NPR;   // scratch
  T* red = Pt + PD::NPR;  // 32

  const int v[3] = {((colour & 1) ? 1 : 2) + 2 * static_cast<int>(blockIdx.x),
                    (((colour >> 1) & 1) ? 1 : 2) + 2 * static_cast<int>(blockIdx.y),
                    (((colour >> 2) & 1) ? 1 : 2) + 2 * static_cast<int>(blockIdx.z)};
  const int n = m * H;
  const int64_t sizeV = static_cast<int64_t>(n + 1) * n * n;

  for (int i = threadIdx.x; i < PD::TAB; i += blockDim.x) tab[i] = ptab[i];
  PatchSolver<T, K> ps;
  ps.tab = tab;
  ps.red = red;
  for (int a = 0; a < 3; ++a) ps.var[a] = 2 * (v[a] == 1) + (v[a] == m - 1);

  // ---- gather R_j r ----
  for (int c = 0; c < 3; ++c) {
    const int d0 = ps.dim(c, 0), d1 = ps.dim(c, 1);
    int64_t gd[3] = {n, n, n};
    gd[c] = n + 1;
    int base[3];
    for (int a = 0; a < 3; ++a) base[a] = (v[a] - 1) * H + (a == c ? 1 : 0);
    for (int o = threadIdx.x; o < PD::NV; o += blockDim.x) {
      const int xx = o % d0, yy = (o / d0) % d1, zz = o / (d0 * d1);
      F[c * PD::NV + o] =
          r[c * sizeV + (static_cast<int64_t>(base[2] + zz) * gd[1] + base[1] + yy) * gd[0] + base[0] + xx];
    }
  }
  for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) {
    const int xx = o % PD::NO, yy = (o / PD::NO) % PD::NO, zz = o / (PD::NO * PD::NO);
    const int gx = (v[0] - 1) * H + xx, gy = (v[1] - 1) * H + yy, gz = (v[2] - 1) * H + zz;
    Pt[o] = r[3 * sizeV + (static_cast<int64_t>(gz) * n + gy) * n + gx];  // G
    Pr[o] = T(0);
  }
  __syncthreads();
  // ---- rhs = B A^-1 F - G (projected) ----
  for (int c = 0; c < 3; ++c) {
    ps.ainv(c, F + c * PD::NV, V1, V2);
    ps.bmul(c, V1, Pq, V2);
    for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) Pr[o] += Pq[o];
    __syncthreads();
  }
  for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) Pr[o] -= Pt[o];
  __syncthreads();
  ps.project(Pr);
  auto precond = [&](const T* rr, T* zz) {
    if (cg_precond) {
      const T* Mi = tab + PD::MPI;
      axis_apply(rr, PD::NO, PD::NO, PD::NO, 0, Mi, PD::NO, PD::NO, false, zz);
      __syncthreads();
      axis_apply(zz, PD::NO, PD::NO, PD::NO, 1, Mi, PD::NO, PD::NO, false, Pt);
      __syncthreads();
      axis_apply(Pt, PD::NO, PD::NO, PD::NO, 2, Mi, PD::NO, PD::NO, false, zz);
      __syncthreads();
    } else {
      for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) zz[o] = rr[o];
      __syncthreads();
    }
    ps.project(zz);
  };
  precond(Pr, Pz);
  for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) {
    Pd[o] = Pz[o];
    Px[o] = T(0);
  }
  __syncthreads();
  T rz = ps.dotp(Pr, Pz);
  const T r0 = sqrt(ps.dotp(Pr, Pr));
  for (int it = 0; it < cg_max_iter; ++it) {
    if (!cg_fixed) {
      const T rr = sqrt(ps.dotp(Pr, Pr));
      if (rr <= cg_tol * r0) break;
    }
    // q = S d = sum_c B_c A_c^-1 B_c^T d
    for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) Pq[o] = T(0);
    __syncthreads();
    for (int c = 0; c < 3; ++c) {
      ps.btmul(c, Pd, V1, V2);
      ps.ainv(c, V1, V1, V2);
      ps.bmul(c, V1, Pt, V2);
      for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) Pq[o] += Pt[o];
      __syncthreads();
    }
    const T dq = ps.dotp(Pd, Pq);
    if (!(dq > T(0)) || rz == T(0)) break;
    const T alpha = rz / dq;
    for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) {
      Px[o] += alpha * Pd[o];
      Pr[o] -= alpha * Pq[o];
    }
    __syncthreads();
    ps.project(Pr);
    precond(Pr, Pz);
    const T rzn = ps.dotp(Pr, Pz);
    const T beta = rzn / rz;
    rz = rzn;
    for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) Pd[o] = Pz[o] + beta * Pd[o];
    __syncthreads();
  }
  ps.project(Px);
  // ---- U_c = A_c^-1 (F_c - B_c^T P); x += R^T (U, P) ----
  for (int c = 0; c < 3; ++c) {
    ps.btmul(c, Px, V1, V2);
    T* Fc = F + c * PD::NV;
    for (int o = threadIdx.x; o < PD::NV; o += blockDim.x) Fc[o] -= V1[o];
    __syncthreads();
    ps.ainv(c, Fc, Fc, V2);
    const int d0 = ps.dim(c, 0), d1 = ps.dim(c, 1);
    int64_t gd[3] = {n, n, n};
    gd[c] = n + 1;
    int base[3];
    for (int a = 0; a < 3; ++a) base[a] = (v[a] - 1) * H + (a == c ? 1 : 0);
    for (int o = threadIdx.x; o < PD::NV; o += blockDim.x) {
      const int xx = o % d0, yy = (o / d0) % d1, zz = o / (d0 * d1);
      x[c * sizeV + (static_cast<int64_t>(base[2] + zz) * gd[1] + base[1] + yy) * gd[0] + base[0] + xx] += Fc[o];
    }
  }
  for (int o = threadIdx.x; o < PD::NPR; o += blockDim.x) {
    const int xx = o % PD::NO, yy = (o / PD::NO) % PD::NO, zz = o / (PD::NO * PD::NO);
    const int gx = (v[0] - 1) * H + xx, gy = (v[1] - 1) * H + yy, gz = (v[2] - 1) * H + zz;
    x[3 * sizeV + (static_cast<int64_t>(gz) * n + gy) * n + gx] += Px[o];
  }
}

template <typename T, int K>
void launch_k(Context& ctx, int level, int colour, void* x, const void* r) {
  using PD = PatchDims<K>;
  const DevLevel& dl = ctx.dev[sizeof(T) == 8 ? 0 : 1][level];
  const int m = dl.lay.m;
  auto cnt = [&](int bit) { return bit ? m / 2 : m / 2 - 1; };
  dim3 grid(cnt(colour & 1), cnt((colour >> 1) & 1), cnt((colour >> 2) & 1));
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  constexpr int BIG = PD::NV > PD::NPR ? PD::NV : PD::NPR;
  const size_t smem = sizeof(T) * (((PD::TAB + 1) / 2) * 2 + 3 * PD::NV + 2 * BIG + 6 * PD::NPR + 32);
  auto kern = patch_smooth_kernel<T, K>;
  SMG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<grid, kPatchThreads, smem, ctx.stream>>>(static_cast<T*>(x), static_cast<const T*>(r),
                                                 static_cast<const T*>(dl.patch), m, colour, ctx.cfg.cg_max_iter,
                                                 static_cast<T>(ctx.cfg.cg_tol), ctx.cfg.cg_fixed,
                                                 ctx.cfg.cg_precond);
  SMG_CUDA(cudaGetLastError());
  ++ctx.launches;
}

template <typename T>
void launch_prec(Context& ctx, int level, int colour, void* x, const void* r) {
  switch (ctx.cfg.degree) {
    case 1: launch_k<T, 1>(ctx, level, colour, x, r); break;
    case 2: launch_k<T, 2>(ctx, level, colour, x, r); break;
    case 3: launch_k<T, 3>(ctx, level, colour, x, r); break;
    case 4: launch_k<T, 4>(ctx, level, colour, x, r); break;
    default: throw std::invalid_argument("degree not supported by the patch smoother kernel (1..4)");
  }
}

}  // namespace

void launch_smooth_colour(Context& ctx, int level, int prec, int colour, void* x, const void* r) {
  if (prec == SMG_F64) launch_prec<double>(ctx, level, colour, x, r);
  else launch_prec<float>(ctx, level, colour, x, r);
}

// packed patch table (same order as PatchDims offsets)
std::vector<double> pack_patch_tables(const PatchTables& P) {
  const int k = P.k, NP = 2 * k + 1, NO = 2 * k + 2;
  std::vector<double> t;
  for (int i = 0; i < NP; ++i)
    for (int j = 0; j < NP; ++j) t.push_back(P.par_S(i, j));
  for (int i = 0; i < NP; ++i) t.push_back(P.par_lam[i]);
  for (int v = 0; v < 4; ++v)
    for (int i = 0; i < NO; ++i)
      for (int j = 0; j < NO; ++j) t.push_back(P.orth_S[v](i, j));
  for (int v = 0; v < 4; ++v)
    for (int i = 0; i < NO; ++i) t.push_back(P.orth_lam[v][i]);
  for (int i = 0; i < NO; ++i)
    for (int j = 0; j < NP; ++j) t.push_back(P.D(i, j));
  for (int i = 0; i < NO; ++i)
    for (int j = 0; j < NO; ++j) t.push_back(P.Mp(i, j));
  for (int i = 0; i < NO; ++i)
    for (int j = 0; j < NO; ++j) t.push_back(P.Mpinv(i, j));
  return t;
}

}  // namespace smg
