// K4/K6: intergrid transfer and the coarse solve (prolongate / restrict SPEC.md:441-458,
// coarse_solve SPEC.md:468-476).
// Prolongation is the canonical embedding of the coarse finite element function into the fine
// space: per velocity component the continuous two-child embedding along its own axis and the
// discontinuous one along the others; pressure discontinuous in all three (fem1d.hpp:243-264).
// Restriction is its exact transpose on coefficient vectors. Both are one thread
// per output DoF, reading the (k+2)(k+1)^2 / 2(k+1)-stencil from L1/L2; HBM-bound by construction.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "smg_internal.cuh"

namespace smg {
namespace {

constexpr int kThreads = 256;

// per-block base pointers in the global index space (z-slab vectors: shifted back by their first plane)
template <typename T>
struct TBlocks {
  T* c[4];
};

template <typename T>
TBlocks<T> tblocks(const LevelLayout& lay, T* v) {
  TBlocks<T> B;
  const int H = lay.k + 1;
  for (int c = 0; c < 4; ++c) B.c[c] = v + lay.off[c] - static_cast<int64_t>(lay.zlo) * H * lay.plane[c];
  return B;
}

// 1D stencils. Continuous (par): fine node gf of a coarse mesh with mc cells, H = k+1:
//   cell E = gf / 2H, row r = gf - 2HE (last node: E = mc-1, r = 2H); coarse nodes E*H + j, j<=H.
// Discontinuous: E = gf / 2H, r = gf % 2H; coarse nodes E*H + j, j < H.
// fine rows of the fine cells [f0, f1) (all rows: f0 = 0, f1 = 2 mc)
template <typename T, int K>
__global__ void prolongate_kernel(const TBlocks<T> xf, const TBlocks<const T> xc, const T* __restrict__ tab, int mc,
                                  int f0, int f1) {
  constexpr int H = K + 1;
  constexpr int EC_R = 2 * H + 1, EC_C = H + 1, ED_R = 2 * H, ED_C = H;
  __shared__ T Ec[EC_R * EC_C], Ed[ED_R * ED_C];
  for (int i = threadIdx.x; i < EC_R * EC_C; i += blockDim.x) Ec[i] = tab[i];
  for (int i = threadIdx.x; i < ED_R * ED_C; i += blockDim.x) Ed[i] = tab[EC_R * EC_C + i];
  __syncthreads();
  const int comp = blockIdx.y;
  const int nc = mc * H, nf = 2 * nc;
  int64_t fd[3] = {nf, nf, nf}, cd[3] = {nc, nc, nc};
  if (comp < 3) { fd[comp] = nf + 1; cd[comp] = nc + 1; }
  const int64_t pl = fd[0] * fd[1];
  const int64_t ibeg = static_cast<int64_t>(f0) * H * pl;
  const int64_t iend = (static_cast<int64_t>(f1) * H + (comp == 2 && f1 == 2 * mc ? 1 : 0)) * pl;
  T* out = xf.c[comp];
  const T* in = xc.c[comp];
  for (int64_t i = ibeg + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < iend;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g[3] = {static_cast<int>(i % fd[0]), static_cast<int>((i / fd[0]) % fd[1]),
                      static_cast<int>(i / (fd[0] * fd[1]))};
    int base[3], row[3], cnt[3];
    const T* W[3];
    for (int a = 0; a < 3; ++a) {
      if (a == comp) {
        int E = g[a] / (2 * H), r = g[a] - 2 * H * E;
        if (E == mc) { E = mc - 1; r = 2 * H; }
        base[a] = E * H; row[a] = r; cnt[a] = EC_C; W[a] = Ec + r * EC_C;
      } else {
        const int E = g[a] / (2 * H);
        base[a] = E * H; row[a] = g[a] - 2 * H * E; cnt[a] = ED_C; W[a] = Ed + row[a] * ED_C;
      }
    }
    T s = T(0);
    for (int j2 = 0; j2 < cnt[2]; ++j2) {
      const T w2 = W[2][j2];
      if (w2 == T(0)) continue;
      const int c2 = base[2] + j2;
      if (comp == 2 && (c2 == 0 || c2 == nc)) continue;
      for (int j1 = 0; j1 < cnt[1]; ++j1) {
        const T w12 = w2 * W[1][j1];
        if (w12 == T(0)) continue;
        const int c1 = base[1] + j1;
        if (comp == 1 && (c1 == 0 || c1 == nc)) continue;
        const T* src = in + (static_cast<int64_t>(c2) * cd[1] + c1) * cd[0] + base[0];
        for (int j0 = 0; j0 < cnt[0]; ++j0) {
          const int c0 = base[0] + j0;
          if (comp == 0 && (c0 == 0 || c0 == nc)) continue;
          s += w12 * W[0][j0] * src[j0];
        }
      }
    }
    out[i] += s;
  }
}

// Restriction = P^T: coarse node gc collects fine rows r < 2H of every coarse cell containing it
// (the fine vertex at r = 2H of cell E is row 0 of cell E+1, counted once).
// coarse rows of the coarse cells [c0, c1) (all rows: c0 = 0, c1 = mc); reads fine cells [2 c0 - 2, 2 c1): a
// u_z node on the bottom plane of coarse cell c0 (j = 0) also lies in coarse cell c0 - 1 and collects its
// fine rows (fine cells 2 c0 - 2, 2 c0 - 1)
template <typename T, int K>
__global__ void restrict_kernel(const TBlocks<T> rc, const TBlocks<const T> rf, const T* __restrict__ tab, int mc,
                                int c0, int c1) {
  constexpr int H = K + 1;
  constexpr int EC_R = 2 * H + 1, EC_C = H + 1, ED_R = 2 * H, ED_C = H;
  __shared__ T Ec[EC_R * EC_C], Ed[ED_R * ED_C];
  for (int i = threadIdx.x; i < EC_R * EC_C; i += blockDim.x) Ec[i] = tab[i];
  for (int i = threadIdx.x; i < ED_R * ED_C; i += blockDim.x) Ed[i] = tab[EC_R * EC_C + i];
  __syncthreads();
  const int comp = blockIdx.y;
  const int nc = mc * H, nf = 2 * nc;
  int64_t fd[3] = {nf, nf, nf}, cd[3] = {nc, nc, nc};
  if (comp < 3) { fd[comp] = nf + 1; cd[comp] = nc + 1; }
  const int64_t pl = cd[0] * cd[1];
  const int64_t ibeg = static_cast<int64_t>(c0) * H * pl;
  const int64_t iend = (static_cast<int64_t>(c1) * H + (comp == 2 && c1 == mc ? 1 : 0)) * pl;
  T* out = rc.c[comp];
  const T* in = rf.c[comp];
  for (int64_t i = ibeg + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < iend;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g[3] = {static_cast<int>(i % cd[0]), static_cast<int>((i / cd[0]) % cd[1]),
                      static_cast<int>(i / (cd[0] * cd[1]))};
    if (comp < 3 && (g[comp] == 0 || g[comp] == nc)) {
      out[i] = T(0);  // constrained coarse DoF
      continue;
    }
    // per axis up to two (cell, local index) pairs
    int ncell[3], fbase[3][2], jj[3][2];
    bool par[3];
    for (int a = 0; a < 3; ++a) {
      par[a] = (a == comp);
      const int E = g[a] / H, j = g[a] - E * H;
      ncell[a] = 0;
      if (E < mc) { fbase[a][ncell[a]] = 2 * H * E; jj[a][ncell[a]] = j; ++ncell[a]; }
      if (par[a] && j == 0 && E > 0) { fbase[a][ncell[a]] = 2 * H * (E - 1); jj[a][ncell[a]] = H; ++ncell[a]; }
    }
    T s = T(0);
    for (int p2 = 0; p2 < ncell[2]; ++p2)
      for (int r2 = 0; r2 < 2 * H; ++r2) {
        const T w2 = par[2] ? Ec[r2 * EC_C + jj[2][p2]] : Ed[r2 * ED_C + jj[2][p2]];
        if (w2 == T(0)) continue;
        const int f2 = fbase[2][p2] + r2;
        for (int p1 = 0; p1 < ncell[1]; ++p1)
          for (int r1 = 0; r1 < 2 * H; ++r1) {
            const T w12 = w2 * (par[1] ? Ec[r1 * EC_C + jj[1][p1]] : Ed[r1 * ED_C + jj[1][p1]]);
            if (w12 == T(0)) continue;
            const int f1 = fbase[1][p1] + r1;
            const T* src = in + (static_cast<int64_t>(f2) * fd[1] + f1) * fd[0];
            for (int p0 = 0; p0 < ncell[0]; ++p0)
              for (int r0 = 0; r0 < 2 * H; ++r0) {
                const T w0 = par[0] ? Ec[r0 * EC_C + jj[0][p0]] : Ed[r0 * ED_C + jj[0][p0]];
                const int f0 = fbase[0][p0] + r0;
                if (comp == 0 && (f0 == 0 || f0 == nf)) continue;
                if (comp == 1 && (f1 == 0 || f1 == nf)) continue;
                if (comp == 2 && (f2 == 0 || f2 == nf)) continue;
                s += w12 * w0 * src[f0];
              }
          }
      }
    out[i] = s;
  }
}

// ---- round 2: one thread per (x cell, row) of the output, compile-time stencils ----
// The per-DoF kernels above decoded every index with 64-bit division, looped over runtime stencil
// extents with zero-weight branches and, for restriction, re-read up to (4H)(2H)^2 fine values per
// coarse DoF: 3.7 % / 4.7 % of the HBM bandwidth at C2 (bench transfer_fp32, round 2). Here a thread
// owns the 2H fine x nodes (prolongation) or the H coarse x nodes (restriction) of one coarse x cell at
// one (y, z) row: the y / z weights are combined once per tap pair and the x contraction is shared by
// the thread's outputs.
template <int COMP, int H>
struct Tap {  // 1D stencil of a fine node g (prolongation): coarse base node, row in the cell table
  __device__ static void fine(int g, int mc, bool par, int& base, int& row) {
    int E = g / (2 * H), r = g - 2 * H * E;
    if (par && E == mc) {
      E = mc - 1;
      r = 2 * H;
    }
    base = E * H;
    row = r;
  }
};

template <typename T, int K, int COMP>
__device__ __forceinline__ void prolong_row(const TBlocks<T>& xf, const TBlocks<const T>& xc, const T* Ec, const T* Ed,
                                            int mc, int ex, int gy, int gz) {
  constexpr int H = K + 1, EC_C = H + 1, ED_C = H;
  constexpr bool PX = COMP == 0, PY = COMP == 1, PZ = COMP == 2;
  constexpr int NX = PX ? H + 1 : H, NY = PY ? H + 1 : H, NZ = PZ ? H + 1 : H;
  const int nc = mc * H, nf = 2 * nc;
  const int cd0 = nc + PX, cd1 = nc + PY, fd0 = nf + PX, fd1 = nf + PY;
  int by, ry, bz, rz;
  Tap<COMP, H>::fine(gy, mc, PY, by, ry);
  Tap<COMP, H>::fine(gz, mc, PZ, bz, rz);
  const T* in = xc.c[COMP];
  T t[NX];
#pragma unroll
  for (int j = 0; j < NX; ++j) t[j] = T(0);
#pragma unroll
  for (int jz = 0; jz < NZ; ++jz) {
    const int cz = bz + jz;
    T wz = PZ ? Ec[rz * EC_C + jz] : Ed[rz * ED_C + jz];
    if (PZ && (cz == 0 || cz == nc)) wz = T(0);  // constrained coarse nodes (input ignored)
#pragma unroll
    for (int jy = 0; jy < NY; ++jy) {
      const int cy = by + jy;
      T w = wz * (PY ? Ec[ry * EC_C + jy] : Ed[ry * ED_C + jy]);
      if (PY && (cy == 0 || cy == nc)) w = T(0);
      const T* src = in + (static_cast<int64_t>(cz) * cd1 + cy) * cd0 + ex * H;
#pragma unroll
      for (int jx = 0; jx < NX; ++jx) {
        const int cx = ex * H + jx;
        const T v = (PX && (cx == 0 || cx == nc)) ? T(0) : src[jx];
        t[jx] += w * v;
      }
    }
  }
  T* out = xf.c[COMP] + (static_cast<int64_t>(gz) * fd1 + gy) * fd0 + 2 * H * ex;
  const int rows = (PX && ex == mc - 1) ? 2 * H + 1 : 2 * H;
#pragma unroll
  for (int r = 0; r <= 2 * H; ++r) {
    if (r >= rows) break;
    T s = T(0);
#pragma unroll
    for (int jx = 0; jx < NX; ++jx) s += (PX ? Ec[r * EC_C + jx] : Ed[r * ED_C + jx]) * t[jx];
    const int gx = 2 * H * ex + r;
    if (!(PX && (gx == 0 || gx == nf))) out[r] += s;
  }
}

// fine rows of the fine cells [f0, f1) along z; grid: x = (x cell, fine y) pairs, y = fine z plane,
// z = component
template <typename T, int K>
__global__ void prolongate_kernel2(const TBlocks<T> xf, const TBlocks<const T> xc, const T* __restrict__ tab, int mc,
                                   int f0, int f1) {
  constexpr int H = K + 1;
  constexpr int EC_R = 2 * H + 1, EC_C = H + 1, ED_R = 2 * H, ED_C = H;
  __shared__ T Ec[EC_R * EC_C], Ed[ED_R * ED_C];
  for (int i = threadIdx.x; i < EC_R * EC_C; i += blockDim.x) Ec[i] = tab[i];
  for (int i = threadIdx.x; i < ED_R * ED_C; i += blockDim.x) Ed[i] = tab[EC_R * EC_C + i];
  __syncthreads();
  const int comp = blockIdx.z;
  const int nf = 2 * mc * H;
  const int fy = nf + (comp == 1);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= mc * fy) return;
  const int ex = t % mc, gy = t / mc;
  const int gz = f0 * H + blockIdx.y;
  if (gz >= f1 * H + (comp == 2 && f1 == 2 * mc ? 1 : 0)) return;
  switch (comp) {
    case 0: prolong_row<T, K, 0>(xf, xc, Ec, Ed, mc, ex, gy, gz); break;
    case 1: prolong_row<T, K, 1>(xf, xc, Ec, Ed, mc, ex, gy, gz); break;
    case 2: prolong_row<T, K, 2>(xf, xc, Ec, Ed, mc, ex, gy, gz); break;
    default: prolong_row<T, K, 3>(xf, xc, Ec, Ed, mc, ex, gy, gz); break;
  }
}

template <typename T, int K, int COMP>
__device__ __forceinline__ void restrict_row(const TBlocks<T>& rc, const TBlocks<const T>& rf, const T* Ec, const T* Ed,
                                             int mc, int ex, int cy, int cz) {
  constexpr int H = K + 1, EC_C = H + 1, ED_C = H;
  constexpr bool PX = COMP == 0, PY = COMP == 1, PZ = COMP == 2;
  constexpr int NXC = PX ? 2 : 1;  // fine x cells read (C0: the previous cell for the shared node j = 0)
  const int nc = mc * H, nf = 2 * nc;
  const int cd0 = nc + PX, cd1 = nc + PY, fd0 = nf + PX, fd1 = nf + PY;
  T* out = rc.c[COMP] + (static_cast<int64_t>(cz) * cd1 + cy) * cd0 + ex * H;
  const bool zero_row = (PY && (cy == 0 || cy == nc)) || (PZ && (cz == 0 || cz == nc));
  // fine x rows of cell ex (and ex - 1) summed over the (y, z) taps with their combined weights
  T acc[NXC][2 * H];
#pragma unroll
  for (int c = 0; c < NXC; ++c)
#pragma unroll
    for (int r = 0; r < 2 * H; ++r) acc[c][r] = T(0);
  if (!zero_row) {
    // per axis: up to two (fine cell base, local coarse index) pairs (C0: the node on a cell boundary
    // belongs to both cells)
    const int Ey = cy / H, jy = cy - Ey * H, Ez = cz / H, jz = cz - Ez * H;
#pragma unroll
    for (int pz = 0; pz < (PZ ? 2 : 1); ++pz) {
      const int E = pz == 0 ? Ez : Ez - 1, j = pz == 0 ? jz : H;
      if (E < 0 || E >= mc || (pz == 1 && jz != 0)) continue;
#pragma unroll
      for (int rz = 0; rz < 2 * H; ++rz) {
        const T wz = PZ ? Ec[rz * EC_C + j] : Ed[rz * ED_C + j];
        const int fz = 2 * H * E + rz;
        if (PZ && fz == 0) continue;
#pragma unroll
        for (int py = 0; py < (PY ? 2 : 1); ++py) {
          const int Ey2 = py == 0 ? Ey : Ey - 1, j2 = py == 0 ? jy : H;
          if (Ey2 < 0 || Ey2 >= mc || (py == 1 && jy != 0)) continue;
#pragma unroll
          for (int ry = 0; ry < 2 * H; ++ry) {
            const T w = wz * (PY ? Ec[ry * EC_C + j2] : Ed[ry * ED_C + j2]);
            const int fyy = 2 * H * Ey2 + ry;
            if (PY && fyy == 0) continue;
            const T* src = rf.c[COMP] + (static_cast<int64_t>(fz) * fd1 + fyy) * fd0;
#pragma unroll
            for (int c = 0; c < NXC; ++c) {
              const int exc = ex - c;
              if (exc < 0) continue;
#pragma unroll
              for (int r = 0; r < 2 * H; ++r) {
                const int fx = 2 * H * exc + r;
                const T v = (PX && fx == 0) ? T(0) : src[fx];
                acc[c][r] += w * v;
              }
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < H; ++j) {
    T s = T(0);
#pragma unroll
    for (int r = 0; r < 2 * H; ++r) s += (PX ? Ec[r * EC_C + j] : Ed[r * ED_C + j]) * acc[0][r];
    if (PX && j == 0) {
#pragma unroll
      for (int r = 0; r < 2 * H; ++r) s += Ec[r * EC_C + H] * acc[NXC - 1][r];
    }
    const int gx = ex * H + j;
    out[j] = (zero_row || (PX && gx == 0)) ? T(0) : s;
  }
  if (PX && ex == mc - 1) out[H] = T(0);  // constrained last coarse node x = nc
}

// coarse rows of the coarse cells [c0, c1) along z; grid: x = (x cell, coarse y) pairs, y = coarse z
// plane, z = component
template <typename T, int K>
__global__ void restrict_kernel2(const TBlocks<T> rc, const TBlocks<const T> rf, const T* __restrict__ tab, int mc,
                                 int c0, int c1) {
  constexpr int H = K + 1;
  constexpr int EC_R = 2 * H + 1, EC_C = H + 1, ED_R = 2 * H, ED_C = H;
  __shared__ T Ec[EC_R * EC_C], Ed[ED_R * ED_C];
  for (int i = threadIdx.x; i < EC_R * EC_C; i += blockDim.x) Ec[i] = tab[i];
  for (int i = threadIdx.x; i < ED_R * ED_C; i += blockDim.x) Ed[i] = tab[EC_R * EC_C + i];
  __syncthreads();
  const int comp = blockIdx.z;
  const int nc = mc * H;
  const int cyn = nc + (comp == 1);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= mc * cyn) return;
  const int ex = t % mc, cy = t / mc;
  const int cz = c0 * H + blockIdx.y;
  if (cz >= c1 * H + (comp == 2 && c1 == mc ? 1 : 0)) return;
  switch (comp) {
    case 0: restrict_row<T, K, 0>(rc, rf, Ec, Ed, mc, ex, cy, cz); break;
    case 1: restrict_row<T, K, 1>(rc, rf, Ec, Ed, mc, ex, cy, cz); break;
    case 2: restrict_row<T, K, 2>(rc, rf, Ec, Ed, mc, ex, cy, cz); break;
    default: restrict_row<T, K, 3>(rc, rf, Ec, Ed, mc, ex, cy, cz); break;
  }
}

// x_free = Pinv b_free, one warp per row (level 0: at most a few thousand free DoFs)
template <typename T>
__global__ void coarse_kernel(T* __restrict__ x, const T* __restrict__ b, const T* __restrict__ pinv,
                              const int64_t* __restrict__ free_idx, int nf) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nf) return;
  const T* row = pinv + static_cast<int64_t>(warp) * nf;
  T s = T(0);
  for (int j = lane; j < nf; j += 32) s += row[j] * b[free_idx[j]];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) x[free_idx[warp]] = s;
}

int grid_for(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return static_cast<int>(g < 4 * kDotBlocks ? (g < 1 ? 1 : g) : 4 * kDotBlocks);
}

// held ranges: fine vectors hold fine cells [fzlo, fzhi), coarse ones [czlo, czhi); rows computed for
// fine cells [r0, r1) (prolongation) or coarse cells [r0, r1) (restriction)
// A/B switch: the round-1 per-DoF kernels (SMG_LEGACY_TRANSFER=1)
bool legacy_transfer() {
  static const bool v = std::getenv("SMG_LEGACY_TRANSFER") != nullptr;
  return v;
}

struct TransferRange {
  int fzlo, fzhi, czlo, czhi, r0, r1;
};

template <typename T, int K>
void transfer_k(Context& ctx, int coarse_level, void* out, const void* in, bool prolong, const TransferRange& t) {
  const int p = sizeof(T) == 8 ? 0 : 1;
  const DevLevel& fine = ctx.dev[p][coarse_level + 1];
  const DevLevel& coarse = ctx.dev[p][coarse_level];
  const int mc = coarse.lay.m;
  const LevelLayout fl(K, coarse_level + 1, t.fzlo, t.fzhi), cl(K, coarse_level, t.czlo, t.czhi);
  if (prolong) {
    // fine cells [r0, r1) read coarse cells [r0 / 2, (r1 + 1) / 2)
    if (t.r0 < t.fzlo || t.r1 > t.fzhi || t.r0 / 2 < t.czlo || (t.r1 + 1) / 2 > t.czhi)
      throw std::invalid_argument("prolongate: held ranges do not cover the rows");
    const int H = K + 1, nf = 2 * mc * H;
    const int planes = (t.r1 - t.r0) * H + 1;
    const dim3 grid((mc * (nf + 1) + kThreads - 1) / kThreads, planes, 4);
    if (legacy_transfer()) {
      const int64_t rows = (static_cast<int64_t>(t.r1 - t.r0) * (K + 1) + 1) * fl.plane[0];
      prolongate_kernel<T, K><<<dim3(grid_for(rows), 4), kThreads, 0, ctx.stream>>>(
          tblocks(fl, static_cast<T*>(out)), tblocks(cl, static_cast<const T*>(in)),
          static_cast<const T*>(fine.transfer), mc, t.r0, t.r1);
    } else {
      prolongate_kernel2<T, K><<<grid, kThreads, 0, ctx.stream>>>(tblocks(fl, static_cast<T*>(out)),
                                                                 tblocks(cl, static_cast<const T*>(in)),
                                                                 static_cast<const T*>(fine.transfer), mc, t.r0, t.r1);
    }
  } else {
    // coarse cells [r0, r1) read fine cells [2 r0 - 2, 2 r1) (within the domain), see restrict_kernel
    if (t.r0 < t.czlo || t.r1 > t.czhi || std::max(2 * t.r0 - 2, 0) < t.fzlo || std::min(2 * t.r1, 2 * mc) > t.fzhi)
      throw std::invalid_argument("restrict: held ranges do not cover the rows");
    const int H = K + 1, nc = mc * H;
    const int planes = (t.r1 - t.r0) * H + 1;
    const dim3 grid((mc * (nc + 1) + kThreads - 1) / kThreads, planes, 4);
    if (legacy_transfer()) {
      const int64_t rows = (static_cast<int64_t>(t.r1 - t.r0) * (K + 1) + 1) * cl.plane[0];
      restrict_kernel<T, K><<<dim3(grid_for(rows), 4), kThreads, 0, ctx.stream>>>(
          tblocks(cl, static_cast<T*>(out)), tblocks(fl, static_cast<const T*>(in)),
          static_cast<const T*>(fine.transfer), mc, t.r0, t.r1);
    } else {
      restrict_kernel2<T, K><<<grid, kThreads, 0, ctx.stream>>>(tblocks(cl, static_cast<T*>(out)),
                                                               tblocks(fl, static_cast<const T*>(in)),
                                                               static_cast<const T*>(fine.transfer), mc, t.r0, t.r1);
    }
  }
  SMG_CUDA(cudaGetLastError());
  ++ctx.launches;
}

template <typename T>
void transfer_prec(Context& ctx, int coarse_level, void* out, const void* in, bool prolong, const TransferRange& t) {
  switch (ctx.cfg.degree) {
    case 1: transfer_k<T, 1>(ctx, coarse_level, out, in, prolong, t); break;
    case 2: transfer_k<T, 2>(ctx, coarse_level, out, in, prolong, t); break;
    case 3: transfer_k<T, 3>(ctx, coarse_level, out, in, prolong, t); break;
    case 4: transfer_k<T, 4>(ctx, coarse_level, out, in, prolong, t); break;
    case 5: transfer_k<T, 5>(ctx, coarse_level, out, in, prolong, t); break;
    case 6: transfer_k<T, 6>(ctx, coarse_level, out, in, prolong, t); break;
    case 7: transfer_k<T, 7>(ctx, coarse_level, out, in, prolong, t); break;
    default: throw std::invalid_argument("degree not supported by the transfer kernels (1..7)");
  }
}

}  // namespace

void launch_prolongate_add(Context& ctx, int coarse_level, int prec, void* xf, const void* xc) {
  const int mc = ctx.dev[0][coarse_level].lay.m;
  const TransferRange t{0, 2 * mc, 0, mc, 0, 2 * mc};
  if (prec == SMG_F64) transfer_prec<double>(ctx, coarse_level, xf, xc, true, t);
  else transfer_prec<float>(ctx, coarse_level, xf, xc, true, t);
}

void launch_restrict(Context& ctx, int coarse_level, int prec, void* rc, const void* rf) {
  const int mc = ctx.dev[0][coarse_level].lay.m;
  const TransferRange t{0, 2 * mc, 0, mc, 0, mc};
  if (prec == SMG_F64) transfer_prec<double>(ctx, coarse_level, rc, rf, false, t);
  else transfer_prec<float>(ctx, coarse_level, rc, rf, false, t);
}

void launch_prolongate_add_held(Context& ctx, int coarse_level, int prec, void* xf, const void* xc, int fzlo, int fzhi,
                                int czlo, int czhi, int f0, int f1) {
  const TransferRange t{fzlo, fzhi, czlo, czhi, f0, f1};
  if (prec == SMG_F64) transfer_prec<double>(ctx, coarse_level, xf, xc, true, t);
  else transfer_prec<float>(ctx, coarse_level, xf, xc, true, t);
}

void launch_restrict_held(Context& ctx, int coarse_level, int prec, void* rc, const void* rf, int fzlo, int fzhi,
                          int czlo, int czhi, int c0, int c1) {
  const TransferRange t{fzlo, fzhi, czlo, czhi, c0, c1};
  if (prec == SMG_F64) transfer_prec<double>(ctx, coarse_level, rc, rf, false, t);
  else transfer_prec<float>(ctx, coarse_level, rc, rf, false, t);
}

void launch_coarse_apply(Context& ctx, int prec, void* x, const void* b) {
  const int nf = static_cast<int>(ctx.coarse_free.size());
  const DevLevel& dl = ctx.dev[prec][0];
  SMG_CUDA(cudaMemsetAsync(x, 0, dl.lay.total * elem_size(prec), ctx.stream));
  const int blocks = (nf * 32 + kThreads - 1) / kThreads;
  if (prec == SMG_F64)
    coarse_kernel<double><<<blocks, kThreads, 0, ctx.stream>>>(
        static_cast<double*>(x), static_cast<const double*>(b), static_cast<const double*>(ctx.coarse_pinv[0]),
        static_cast<const int64_t*>(ctx.coarse_free_dev), nf);
  else
    coarse_kernel<float><<<blocks, kThreads, 0, ctx.stream>>>(
        static_cast<float*>(x), static_cast<const float*>(b), static_cast<const float*>(ctx.coarse_pinv[1]),
        static_cast<const int64_t*>(ctx.coarse_free_dev), nf);
  SMG_CUDA(cudaGetLastError());
  ++ctx.launches;
}

}  // namespace smg
