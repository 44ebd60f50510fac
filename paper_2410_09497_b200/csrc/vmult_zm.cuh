#pragma once
// K1z: the Stokes operator y = A x / residual r = b - A x as a z-MARCH ("2.5D") kernel for k <= 2.
//
// Reference: apply_stokes, Alg. 1 of PAPER.md:115-151, evaluated in the exact
// Kronecker form of vmult_kernel.cuh. What changes is the data flow, chosen to cut
// shared-memory traffic, which ncu showed to be the limiter of the brick kernel (profiles/r01: 57 M
// SMEM wavefronts per C2 apply, ~21 accesses per DoF, plus 2.8-3.3-way bank conflicts):
//
//   * A CTA owns a TX x TY cell tile in (x, y) and walks a range of z cell layers. Per layer and per
//     z node plane b (0..k) it processes the four blocks p, u_x, u_y, u_z in turn ("steps").
//   * Stage A (x direction, shared memory -> shared memory): the plane's staged box (TMA / bulk copy
//     into a 4-slot ring, prefetched 3 steps ahead) is contracted along x by cell work items:
//       u_x (C0 in x): A = M_x u, B = L_x u, E = D_x u       u_y, u_z: A = M_x u, B = L_x u
//       p: PX = M_x p, P1 = D_x^T p
//   * Stage B (y direction, shared memory -> registers): thread (x node, y cell) contracts its
//     column along y:  S = M_y A, T = M_y B + L_y A (+ R = M_y E or D_y A for y_p, + PB from PX/P1).
//   * Stage C (z direction, registers only): S, T, PB, R of plane b are folded immediately into
//     per-thread accumulators -- the current cell's rows, the previous cell's rows that still wait for
//     this cell's face values, and the face terms carried to the next cell -- so the z contractions
//     never touch shared memory and the outputs leave from registers (coalesced along x).
// Shared-memory accesses per DoF drop to ~10 (stage A ~5.5 incl. the y halo, stage B ~5), the z halo
// disappears (one extra layer per z range), and there are 4 CTA barriers per z plane (1 per step).
// Pitches are chosen bank-conflict free for the work-item shapes (x pitches = 8 mod 16 doubles /
// 8 mod 32 floats). Boundary Nitsche rows, constrained boundary-normal rows (output 0, input ignored),
// z slabs (held / computed cell ranges) and the residual variant follow vmult_kernel.cuh.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "smg_internal.cuh"
#include "vmult.cuh"

namespace smg {

static __constant__ double zm_ref_d[kRefTotal];
static __constant__ float zm_ref_f[kRefTotal];

namespace zm {

template <typename T>
__device__ __forceinline__ T cr(int i);
template <>
__device__ __forceinline__ double cr<double>(int i) { return zm_ref_d[i]; }
template <>
__device__ __forceinline__ float cr<float>(int i) { return zm_ref_f[i]; }

// offsets of the reference-cell blocks of degree K in the constant table (setup1d.hpp ref_layout)
template <int K>
struct Ref {
  static constexpr int H = K + 1, P = K + 2;
  static constexpr int MO = ref_base(K);
  static constexpr int LO0 = MO + H * H;
  static constexpr int LOM = LO0 + H * H;
  static constexpr int LOP = LOM + H * H;
  static constexpr int DLF = LOP + H * H;
  static constexpr int DLL = DLF + H * H;
  static constexpr int MP = DLL + H * H;
  static constexpr int LP = MP + P * P;
  static constexpr int D = LP + P * P;
};
// element accessors (compile-time indices after unrolling -> constant-bank operands)
template <typename T, int K> __device__ __forceinline__ T mo(int a, int b) { return cr<T>(Ref<K>::MO + a * (K + 1) + b); }
template <typename T, int K> __device__ __forceinline__ T lo0(int a, int b) { return cr<T>(Ref<K>::LO0 + a * (K + 1) + b); }
template <typename T, int K> __device__ __forceinline__ T lom(int a, int b) { return cr<T>(Ref<K>::LOM + a * (K + 1) + b); }
template <typename T, int K> __device__ __forceinline__ T lop(int a, int b) { return cr<T>(Ref<K>::LOP + a * (K + 1) + b); }
template <typename T, int K> __device__ __forceinline__ T dlf(int a, int b) { return cr<T>(Ref<K>::DLF + a * (K + 1) + b); }
template <typename T, int K> __device__ __forceinline__ T dll(int a, int b) { return cr<T>(Ref<K>::DLL + a * (K + 1) + b); }
template <typename T, int K> __device__ __forceinline__ T mp(int a, int b) { return cr<T>(Ref<K>::MP + a * (K + 2) + b); }
template <typename T, int K> __device__ __forceinline__ T lp(int a, int b) { return cr<T>(Ref<K>::LP + a * (K + 2) + b); }
// D (H x P): DG row i from C0 node b of the cell
template <typename T, int K> __device__ __forceinline__ T dd(int i, int b) { return cr<T>(Ref<K>::D + i * (K + 2) + b); }
// cross-shaped SIPG face blocks of the Gauss-Lobatto basis: LOM[a][b] != 0 only if a == 0 or b == K,
// LOP[a][b] != 0 only if a == K or b == 0 (face value: node K of the left / node 0 of the right cell)
template <int K> __host__ __device__ constexpr bool lom_nz(int a, int b) { return a == 0 || b == K; }
template <int K> __host__ __device__ constexpr bool lop_nz(int a, int b) { return a == K || b == 0; }

constexpr int pitch8(int v, int vec, int mod) {
  int p = v;
  while (p % vec != 0 || p % mod != 8) ++p;
  return p;
}

template <typename T, int K, int TX, int TY, int OCC>
struct Cfg {
  static constexpr int H = K + 1, P = K + 2;
  static constexpr int XN = TX * H;                   // owned x nodes of a tile (C0 for u_x, DG otherwise)
  static constexpr int NT = XN * TY;                  // one thread per (x node, y cell)
  static constexpr int YE = TY * H + 2 * H + 1;       // stage-A rows: y0 - H .. y0 + TY H + H
  static constexpr int VEC = 16 / static_cast<int>(sizeof(T));
  static constexpr int PADF = 128 / static_cast<int>(sizeof(T));
  static constexpr int MODB = sizeof(T) == 8 ? 16 : 32;  // 64-bit: 16 bank pairs per half warp
  static constexpr int XNEED = XN + 2 * H + 1 + VEC - 1;  // x0 - H .. x0 + XN + H, + 16-B alignment slack
  static constexpr int XB = pitch8(XNEED, VEC, MODB);     // staged box row pitch
  static constexpr int AP = pitch8(XN, 1, MODB);          // stage-A output pitch
  static constexpr int BOX = YE * XB;
  static constexpr int SLOT = (PADF + BOX + VEC + PADF - 1) / PADF * PADF;  // 128-B aligned ring slots
  static constexpr int RING = 4;
  static constexpr int ARR = YE * AP;
  static constexpr int OFF_V = RING * SLOT;        // velocity stage-A outputs: 2 buffers x (A, B, E)
  static constexpr int OFF_P = OFF_V + 6 * ARR;    // pressure stage-A outputs: 2 buffers x (PX, P1)
  static constexpr int END_C0 = OFF_P + 4 * ARR;  // per-thread layer carries: 4 x H x H per thread
  static constexpr int END = END_C0 + 4 * H * H * NT;
  static constexpr size_t BYTES = (static_cast<size_t>(END) * sizeof(T) + 7) / 8 * 8 + RING * 8;
};

struct ZMaps {
  CUtensorMap u1, u2, p;  // 3D plane boxes of u_y, u_z, p (u_x rows are non-tensor bulk copies)
};

template <typename T>
struct ZBlocks {
  T* c[4];
};

// the (<= 2) contiguous (tile, z-layer range) segments of a persistent CTA
struct Seg {
  int tile, zs, ze;  // computed cells [zs, ze) of the tile's column
  int l0, nl;        // processed layers [l0, l0 + nl): zs-1 .. ze, clipped to the domain and the held range
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ int floor_to(int v, int q) { return v & -q; }

struct Geo {
  int m, n, H;
  int lnx, lny;  // log2 of the tile counts along x / y
  int zoff;      // first z node plane held by the vector (TMA maps are slab-local)
  int zlo, zhi;  // held cells
};

template <typename T, int K, int TX, int TY, int OCC>
struct Kern {
  using C = Cfg<T, K, TX, TY, OCC>;
  static constexpr int H = K + 1, XN = C::XN, NT = C::NT, YE = C::YE, XB = C::XB, AP = C::AP, VEC = C::VEC;

  // ---- staging of one (block, plane) box into a ring slot; thread 0 (TMA) or warp 0 (u_x rows) ----
  // box rows: global y = y0 - H + r (r < YE); columns from the 16-B aligned position at or below
  // x0 - H (clamped to 0; u_x: per row); consumers add the shift returned by col0().
  __device__ static void issue(T* slot, uint64_t* bar, int blk, int gz, int x0, int y0, const ZBlocks<const T>& X,
                               const ZMaps& M, const Geo& G) {
    const int tid = threadIdx.x;
    const int n = G.n;
    if (blk == 3 && gz == 0) {  // constrained plane z = 0 of u_z: never read (stage A writes zeros)
      if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
      return;
    }
    if (blk == 1) {  // u_x: one bulk copy per row (pitch n + 1 is no legal TMA stride)
      if (tid < 32) {
        unsigned bytes = 0;
        for (int r = tid; r < YE; r += 32) {
          const int y = y0 - H + r;
          T* dst = slot + C::PADF + r * XB;
          if (y >= 0 && y < n) {
            const int64_t start = (static_cast<int64_t>(gz) * n + y) * (n + 1) + x0 - H;
            const int64_t sal = start & -static_cast<int64_t>(VEC);
            const int64_t row0 = static_cast<int64_t>(gz) * n * (n + 1);  // never reach into plane gz - 1
            const int64_t ss = (y == 0 && sal < row0) ? row0 : sal;
            const unsigned nb = static_cast<unsigned>((XB - (ss - sal)) * sizeof(T));
            bulk_load(dst + (ss - sal), X.c[0] + ss, nb, bar);
            bytes += nb;
          } else {
            for (int i = 0; i < XB; ++i) dst[i] = T(0);
          }
        }
        bytes = __reduce_add_sync(0xffffffffu, bytes);
        if (tid == 0) mbar_expect(bar, bytes);
      }
      return;
    }
    if (tid == 0) {
      mbar_expect(bar, static_cast<unsigned>(C::BOX * sizeof(T)));
      const int xs = max(floor_to(x0 - H, VEC), 0);
      if (blk == 0) tma_load_3d(slot + C::PADF, &M.p, xs, y0 - H, gz - G.zoff, bar);
      else if (blk == 2) tma_load_3d(slot + C::PADF, &M.u1, xs, y0 - H - 1, gz - G.zoff, bar);  // map starts at row 1
      else tma_load_3d(slot + C::PADF, &M.u2, xs, y0 - H, gz - G.zoff, bar);
    }
  }
  // smem column of global x node x0 - H in box row r (relative to slot + PADF + r XB)
  __device__ static int col0(int blk, int x0, int y0, int r, int n, int gz) {
    if (blk == 1) {
      const int y = y0 - H + r;
      return static_cast<int>(((static_cast<int64_t>(gz) * n + y) * (n + 1) + x0 - H) & (VEC - 1));
    }
    return x0 - H - max(floor_to(x0 - H, VEC), 0);
  }

  // ---- stage A: x contractions of one plane box into the stage-A arrays ----
  // work item = (x cell ex of the tile, box row r); DG windows read cells ex-1, ex, ex+1 (zero outside
  // the domain by selection -- never by multiplication, the slack may hold anything)
  __device__ static void stage_a(int blk, const T* box, T* o0, T* o1, T* o2, int x0, int y0, const Geo& G, int gz,
                                 bool zero_plane) {
    const int n = G.n, m = G.m;
    const int cx0 = x0 / H;
    for (int it = threadIdx.x; it < TX * YE; it += NT) {
      const int ex = it % TX, r = it / TX;
      const T* row = box + C::PADF + r * XB + col0(blk, x0, y0, r, n, gz);  // row[j] = node x0 - H + j
      const int gcell = cx0 + ex;
      const bool lz = gcell == 0, rzc = gcell == m - 1;
      T* d0 = o0 + r * AP + ex * H;
      T* d1 = o1 + r * AP + ex * H;
      if (blk == 1) {
        // u_x, C0 along x: window nodes (ex-1)H .. ex H + H -> w[0 .. 2H]; node 0 and n are constrained
        T w[2 * H + 1];
#pragma unroll
        for (int j = 0; j < 2 * H + 1; ++j) {
          const int gx = x0 + (ex - 1) * H + j;
          const T v = row[ex * H + j];
          w[j] = (zero_plane || gx <= 0 || gx >= n) ? T(0) : v;
        }
        T* d2 = o2 + r * AP + ex * H;
#pragma unroll
        for (int a = 0; a < H; ++a) {
          T sa = T(0), sb = T(0);
#pragma unroll
          for (int b = 0; b <= H; ++b) {
            sa += mp<T, K>(a, b) * w[H + b];
            sb += lp<T, K>(a, b) * w[H + b];
          }
          if (a == 0) {
#pragma unroll
            for (int b = 0; b <= H; ++b) {
              sa += mp<T, K>(H, b) * w[b];
              sb += lp<T, K>(H, b) * w[b];
            }
          }
          T se = T(0);
#pragma unroll
          for (int b = 0; b <= H; ++b) se += dd<T, K>(a, b) * w[H + b];
          d0[a] = sa;
          d1[a] = sb;
          d2[a] = se;
        }
      } else if (blk == 0) {
        // p: PX = M p (own cell), P1 = D^T p (C0 rows of cell ex from cells ex-1, ex)
        T w[2 * H];
#pragma unroll
        for (int j = 0; j < 2 * H; ++j) {
          const T v = row[ex * H + j];
          w[j] = (j < H && lz) ? T(0) : v;
        }
#pragma unroll
        for (int a = 0; a < H; ++a) {
          T sx = T(0), s1 = T(0);
#pragma unroll
          for (int i = 0; i < H; ++i) {
            sx += mo<T, K>(a, i) * w[H + i];
            s1 += dd<T, K>(i, a) * w[H + i];
          }
          if (a == 0) {
#pragma unroll
            for (int i = 0; i < H; ++i) s1 += dd<T, K>(i, H) * w[i];
          }
          d0[a] = sx;
          d1[a] = s1;
        }
      } else {
        // u_y, u_z: DG along x, A = M u, B = L u (SIPG with Nitsche rows at the domain ends)
        T w[3 * H];
#pragma unroll
        for (int j = 0; j < 3 * H; ++j) {
          const T v = row[ex * H + j];
          w[j] = (zero_plane || (j < H && lz) || (j >= 2 * H && rzc)) ? T(0) : v;
        }
#pragma unroll
        for (int a = 0; a < H; ++a) {
          T sa = T(0), sb = T(0);
#pragma unroll
          for (int b = 0; b < H; ++b) {
            sa += mo<T, K>(a, b) * w[H + b];
            sb += lo0<T, K>(a, b) * w[H + b];
            if (lom_nz<K>(a, b)) sb += lom<T, K>(a, b) * w[b];
            if (lop_nz<K>(a, b)) sb += lop<T, K>(a, b) * w[2 * H + b];
          }
          if (lz) {
#pragma unroll
            for (int b = 0; b < H; ++b) sb += dlf<T, K>(a, b) * w[H + b];
          }
          if (rzc) {
#pragma unroll
            for (int b = 0; b < H; ++b) sb += dll<T, K>(a, b) * w[H + b];
          }
          d0[a] = sa;
          d1[a] = sb;
        }
      }
    }
  }
};

template <bool V>
using bc_ = std::integral_constant<bool, V>;
template <int V>
using ic_ = std::integral_constant<int, V>;

// segments of CTA `cta` among `ncta`: the flattened (tile, z cell) sequence of the computed cells is cut
// into equal consecutive ranges; a range covers at most two tiles. Processed layers: zs-1 (face terms
// only) .. ze, where layer ze = m is a virtual all-zero layer that closes the last cell's rows.
__device__ __forceinline__ int make_segs(Seg* sg, int cta, int ncta, int ntiles, int z0, int z1) {
  const int nz = z1 - z0;
  const int64_t total = static_cast<int64_t>(ntiles) * nz;
  const int64_t beg = total * cta / ncta, end = total * (cta + 1) / ncta;
  int ns = 0;
  for (int64_t p = beg; p < end && ns < 2;) {
    const int tile = static_cast<int>(p / nz);
    const int zs = z0 + static_cast<int>(p % nz);
    const int64_t stop = std::min<int64_t>(end, static_cast<int64_t>(tile + 1) * nz);
    const int ze = z0 + static_cast<int>(stop - static_cast<int64_t>(tile) * nz);
    Seg& s = sg[ns++];
    s.tile = tile;
    s.zs = zs;
    s.ze = ze;
    s.l0 = max(zs - 1, 0);
    s.nl = ze - s.l0 + 1;
    p = stop;
  }
  return ns;
}

template <typename T, int K, int TX, int TY, int OCC, bool RESID>
__global__ void __launch_bounds__(Cfg<T, K, TX, TY, OCC>::NT, OCC)
    zm_vmult_kernel(const ZBlocks<const T> X, const ZBlocks<T> Y, const ZBlocks<const T> Bv, int m, int z0, int z1,
                    int zlo, int zhi, T h, const ZMaps* __restrict__ mapsp) {
  using C = Cfg<T, K, TX, TY, OCC>;
  using KN = Kern<T, K, TX, TY, OCC>;
  constexpr int H = K + 1, XN = C::XN, AP = C::AP, NT = C::NT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (C::BYTES - C::RING * 8));
  const ZMaps& maps = *mapsp;
  Geo G;
  G.m = m;
  G.n = m * H;
  G.H = H;
  G.zoff = zlo * H;
  G.zlo = zlo;
  G.zhi = zhi;
  const int n = G.n;
  const int ntx = m / TX, nty = m / TY;
  Seg sg[2];
  const int nseg = make_segs(sg, blockIdx.x, gridDim.x, ntx * nty, z0, z1);
  if (nseg == 0) return;
  int total = 0;
  for (int s = 0; s < nseg; ++s) total += sg[s].nl * H * 4;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int r = 0; r < C::RING; ++r) mbar_init(&bars[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // producer: step -> (segment, layer, plane, block) -> box (the virtual layer m: arrival only)
  auto issue_step = [&](int st) {
    int s = 0, j = st;
    if (nseg > 1 && j >= sg[0].nl * H * 4) {
      j -= sg[0].nl * H * 4;
      s = 1;
    }
    const int blk = j & 3, pl = (j >> 2) % H, lay = sg[s].l0 + (j >> 2) / H;
    const int tile = sg[s].tile;
    const int tx = tile % ntx, ty = tile / ntx;
    uint64_t* bar = &bars[st % C::RING];
    if (lay >= m) {
      if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
      return;
    }
    KN::issue(sm + (st % C::RING) * C::SLOT, bar, blk, lay * H + pl, tx * TX * H, ty * TY * H, X, maps, G);
  };
  for (int st = 0; st < C::RING - 1 && st < total; ++st) issue_step(st);

  // per-thread layer carries in shared memory (thread-major, conflict free): rows of the previous cell
  // that wait for this cell's planes -- u_x, u_y (DG in z), u_z (C0 in z) and p -- H x H each
  T* cs = sm + C::END_C0;
  auto cslot = [&](int blockv, int q, int a) -> T& { return cs[((blockv * H + q) * H + a) * NT + tid]; };

  const int xi = tid % XN, yj = tid / XN;
  int step = 0;
  for (int s = 0; s < nseg; ++s) {
    const Seg S = sg[s];
    const int tx = S.tile % ntx, ty = S.tile / ntx;
    const int x0 = tx * TX * H, y0 = ty * TY * H;
    const int cy = ty * TY + yj;  // global y cell of this thread
    const int gx = x0 + xi;
    const bool ylo = cy == 0, yhi = cy == m - 1;
    // per-thread 32-bit row offsets within a node plane of each block, and plane strides
    const int gy0 = y0 + yj * H;
    const int plx = n * (n + 1), ply = (n + 1) * n, plz = n * n;
    int ox[H], oy[H], oz[H];
#pragma unroll
    for (int q = 0; q < H; ++q) {
      ox[q] = (gy0 + q) * (n + 1) + gx;
      oy[q] = (gy0 + q) * n + gx;
      oz[q] = (gy0 + q) * n + gx;
    }
    // register carries across layers: face terms of the previous cell (DG blocks: c0 = row-0 coupling
    // summed over its planes, sK = S of its last plane) and u_z's row-H partial of the previous cell
    T c0[2][H], sK[2][H], zcl[H];
#pragma unroll
    for (int q = 0; q < H; ++q) {
      c0[0][q] = c0[1][q] = sK[0][q] = sK[1][q] = zcl[q] = T(0);
#pragma unroll
      for (int a = 0; a < H; ++a)
#pragma unroll
        for (int v = 0; v < 4; ++v) cslot(v, q, a) = T(0);
    }
    for (int li = 0; li < S.nl; ++li) {
      const int e = S.l0 + li;
      const bool virt = e >= m;                             // closing all-zero layer
      const bool in_prev = e - 1 >= S.zs && e - 1 < S.ze;  // rows of cell e-1 are ours to store
      const bool zlo_c = e == 0, zhi_c = e == m - 1;
      // global pointers of the previous cell's first node plane per block
      const int64_t pz0 = static_cast<int64_t>(e - 1) * H;
      T* yx = Y.c[0] + pz0 * plx;
      T* yy = Y.c[1] + pz0 * ply;
      T* yz = Y.c[2] + pz0 * plz;
      T* yp = Y.c[3] + pz0 * plz;
      const T* bx = RESID ? Bv.c[0] + pz0 * plx : nullptr;
      const T* by = RESID ? Bv.c[1] + pz0 * ply : nullptr;
      const T* bz = RESID ? Bv.c[2] + pz0 * plz : nullptr;
      const T* bp = RESID ? Bv.c[3] + pz0 * plz : nullptr;
      auto put = [&](T* y, const T* bb, int off, T v, bool constrained) {
        T r = constrained ? T(0) : v;
        if (RESID && !constrained) r = bb[off] - r;
        y[off] = r;
      };
      T acc[3][H][H];  // rows of cell e per velocity block (u_x, u_y, u_z), y node q
      T pacc[H][H];    // pressure rows of cell e
      T pK[2][H];      // DG blocks: row K of cell e-1 (pending until the last plane)
#pragma unroll
      for (int q = 0; q < H; ++q)
#pragma unroll
        for (int a = 0; a < H; ++a) pacc[q][a] = T(0);
      auto plane = [&](auto btag) {
        constexpr int b = decltype(btag)::value;
        const int gzp = e * H + b;  // global node plane
        T* pbuf = sm + C::OFF_P + ((gzp & 1) ? 2 * C::ARR : 0);  // PX, P1 of this plane
        auto blockstep = [&](auto ktag) {
          constexpr int blk = decltype(ktag)::value;
          T* slot = sm + (step % C::RING) * C::SLOT;
          mbar_wait(&bars[step % C::RING], (step / C::RING) & 1);
          T* vb = sm + C::OFF_V + (blk & 1) * 3 * C::ARR;
          const bool zp = virt || (blk == 3 && gzp == 0);
          if (blk == 0) KN::stage_a(0, slot, pbuf, pbuf + C::ARR, nullptr, x0, y0, G, gzp, virt);
          else KN::stage_a(blk, slot, vb, vb + C::ARR, vb + 2 * C::ARR, x0, y0, G, gzp, zp);
          fence_proxy_async();
          __syncthreads();
          if (step + C::RING - 1 < total) issue_step(step + C::RING - 1);
          ++step;
          if constexpr (blk != 0) {
            // ---- stage B: y contractions of this thread's column (x node xi, y cell yj) ----
            const T* A = vb;
            const T* Bb = vb + C::ARR;
            const T* E = vb + 2 * C::ARR;
            const T* PX = pbuf;
            const T* P1 = pbuf + C::ARR;
            const int ro = (H + yj * H) * AP + xi;      // own row 0
            const int rl = (yj * H) * AP + xi;          // left cell row 0
            const int rr = (2 * H + yj * H) * AP + xi;  // right cell row 0
            T Sq[H], Tq[H], Rq[H], PBq[H];
            if constexpr (blk == 2) {
              // u_y: C0 along y (rows = C0 nodes of cell yj), R = D_y A, PB = D_y^T PX
              T al[H + 1], ao[H + 1], bl[H + 1], bo[H + 1], pxo[H], pxl[H];
#pragma unroll
              for (int j = 0; j <= H; ++j) {
                ao[j] = A[ro + j * AP];
                bo[j] = Bb[ro + j * AP];
              }
#pragma unroll
              for (int j = 0; j < H; ++j) {
                al[j] = A[rl + j * AP];
                bl[j] = Bb[rl + j * AP];
              }
              al[H] = ao[0];
              bl[H] = bo[0];
#pragma unroll
              for (int i = 0; i < H; ++i) {
                pxo[i] = PX[ro + i * AP];
                pxl[i] = ylo ? T(0) : PX[rl + i * AP];
              }
#pragma unroll
              for (int q = 0; q < H; ++q) {
                T sv = T(0), tv = T(0), pv = T(0);
#pragma unroll
                for (int j = 0; j <= H; ++j) {
                  sv += mp<T, K>(q, j) * ao[j];
                  tv += mp<T, K>(q, j) * bo[j] + lp<T, K>(q, j) * ao[j];
                }
                if (q == 0) {
#pragma unroll
                  for (int j = 0; j <= H; ++j) {
                    sv += mp<T, K>(H, j) * al[j];
                    tv += mp<T, K>(H, j) * bl[j] + lp<T, K>(H, j) * al[j];
                  }
                }
#pragma unroll
                for (int i = 0; i < H; ++i) pv += dd<T, K>(i, q) * pxo[i];
                if (q == 0) {
#pragma unroll
                  for (int i = 0; i < H; ++i) pv += dd<T, K>(i, H) * pxl[i];
                }
                T rv = T(0);
#pragma unroll
                for (int j = 0; j <= H; ++j) rv += dd<T, K>(q, j) * ao[j];
                Sq[q] = sv;
                Tq[q] = tv;
                PBq[q] = pv;
                Rq[q] = rv;
              }
            } else {
              // u_x, u_z: DG along y (SIPG with Nitsche rows at y cells 0, m-1)
              T al[H], ao[H], ar[H], bo[H], xo[H];
#pragma unroll
              for (int j = 0; j < H; ++j) {
                ao[j] = A[ro + j * AP];
                al[j] = ylo ? T(0) : A[rl + j * AP];
                ar[j] = yhi ? T(0) : A[rr + j * AP];
                bo[j] = Bb[ro + j * AP];
                xo[j] = blk == 1 ? P1[ro + j * AP] : PX[ro + j * AP];
              }
              T eo[H];
              if constexpr (blk == 1) {
#pragma unroll
                for (int j = 0; j < H; ++j) eo[j] = E[ro + j * AP];
              }
#pragma unroll
              for (int q = 0; q < H; ++q) {
                T sv = T(0), tv = T(0), pv = T(0), rv = T(0);
#pragma unroll
                for (int j = 0; j < H; ++j) {
                  sv += mo<T, K>(q, j) * ao[j];
                  tv += mo<T, K>(q, j) * bo[j] + lo0<T, K>(q, j) * ao[j];
                  if (lom_nz<K>(q, j)) tv += lom<T, K>(q, j) * al[j];
                  if (lop_nz<K>(q, j)) tv += lop<T, K>(q, j) * ar[j];
                  pv += mo<T, K>(q, j) * xo[j];
                  if constexpr (blk == 1) rv += mo<T, K>(q, j) * eo[j];
                }
                if (ylo) {
#pragma unroll
                  for (int j = 0; j < H; ++j) tv += dlf<T, K>(q, j) * ao[j];
                }
                if (yhi) {
#pragma unroll
                  for (int j = 0; j < H; ++j) tv += dll<T, K>(q, j) * ao[j];
                }
                Sq[q] = sv;
                Tq[q] = tv;
                PBq[q] = pv;
                Rq[q] = rv;
              }
            }
            // ---- stage C: z contractions folded into the register accumulators ----
            if constexpr (blk == 1 || blk == 2) {
              constexpr int v = blk - 1;  // DG-in-z block slot
#pragma unroll
              for (int q = 0; q < H; ++q) {
                const T sv = Sq[q], tv = Tq[q] + h * PBq[q];
                if (b == 0) {
                  // the previous cell's face terms open this cell's rows; its own pending rows get the
                  // plane-0 coupling (LOP is cross shaped) and all but row K are complete
                  acc[v][q][0] = c0[v][q];
#pragma unroll
                  for (int a = 1; a < H; ++a) acc[v][q][a] = lom<T, K>(a, K) * sK[v][q];
#pragma unroll
                  for (int a = 0; a < H; ++a) {
                    const T pv = cslot(v, q, a) + lop<T, K>(a, 0) * sv;
                    if (a < K) {
                      if (in_prev) {
                        if (v == 0) put(yx, bx, a * plx + ox[q], h * pv, gx == 0);
                        else put(yy, by, a * ply + oy[q], h * pv, gy0 + q == 0);
                      }
                    } else {
                      pK[v][q] = pv;
                    }
                  }
                } else {
                  pK[v][q] += lop<T, K>(K, b) * sv;
                }
#pragma unroll
                for (int a = 0; a < H; ++a) {
                  T w = mo<T, K>(a, b) * tv + lo0<T, K>(a, b) * sv;
                  if (zlo_c) w += dlf<T, K>(a, b) * sv;
                  if (zhi_c) w += dll<T, K>(a, b) * sv;
                  acc[v][q][a] += w;
                }
                // face term of this cell for the next one: row 0 collects all planes, the others S[K]
                if (b == 0) c0[v][q] = lom<T, K>(0, b) * sv;
                else c0[v][q] += lom<T, K>(0, b) * sv;
#pragma unroll
                for (int i = 0; i < H; ++i) pacc[q][i] += mo<T, K>(i, b) * Rq[q];
                if (b == K) {
                  sK[v][q] = sv;
                  if (in_prev) {
                    if (v == 0) put(yx, bx, K * plx + ox[q], h * pK[v][q], gx == 0);
                    else put(yy, by, K * ply + oy[q], h * pK[v][q], gy0 + q == 0);
                  }
#pragma unroll
                  for (int a = 0; a < H; ++a) cslot(v, q, a) = acc[v][q][a];
                }
              }
            } else {
              // u_z: C0 along z; plane b is node e H + b
#pragma unroll
              for (int q = 0; q < H; ++q) {
                const T sv = Sq[q], tv = Tq[q], pbv = h * PBq[q];
                if (b == 0) {
                  // node e H is node H of cell e-1: completes its rows and the pressure rows of cell e-1
#pragma unroll
                  for (int a = 0; a < H; ++a) {
                    const T zv = cslot(2, q, a) + mp<T, K>(a, H) * tv + lp<T, K>(a, H) * sv;
                    const T pvv = cslot(3, q, a) + dd<T, K>(a, H) * sv;
                    if (in_prev) {
                      put(yz, bz, a * plz + oz[q], h * zv, e - 1 == 0 && a == 0);
                      put(yp, bp, a * plz + oz[q], h * h * pvv, false);
                    }
                  }
                  acc[2][q][0] = zcl[q] + mp<T, K>(H, H) * tv + lp<T, K>(H, H) * sv;
#pragma unroll
                  for (int a = 1; a < H; ++a) acc[2][q][a] = T(0);
                  zcl[q] = T(0);
                  // constrained top plane z = n of u_z (row 0 of the virtual layer)
                  if (virt && in_prev) put(yz, bz, H * plz + oz[q], T(0), true);
                }
#pragma unroll
                for (int a = 0; a < H; ++a)
                  acc[2][q][a] += mp<T, K>(a, b) * tv + lp<T, K>(a, b) * sv + dd<T, K>(b, a) * pbv;
                zcl[q] += mp<T, K>(H, b) * tv + lp<T, K>(H, b) * sv + dd<T, K>(b, H) * pbv;
#pragma unroll
                for (int i = 0; i < H; ++i) pacc[q][i] += dd<T, K>(i, b) * sv;
                if (b == K) {
#pragma unroll
                  for (int a = 0; a < H; ++a) {
                    cslot(2, q, a) = acc[2][q][a];
                    cslot(3, q, a) = pacc[q][a];
                  }
                }
              }
            }
          }
        };
        blockstep(ic_<0>());
        blockstep(ic_<1>());
        blockstep(ic_<2>());
        blockstep(ic_<3>());
      };
      plane(ic_<0>());
      if constexpr (K >= 1) plane(ic_<1>());
      if constexpr (K >= 2) plane(ic_<2>());
    }
    // constrained planes x = n (u_x) and y = n (u_y) of the last tiles, for the computed cells
    if (x0 + XN == n && xi == XN - 1) {
      for (int gz = S.zs * H; gz < S.ze * H; ++gz)
#pragma unroll
        for (int q = 0; q < H; ++q) Y.c[0][(static_cast<int64_t>(gz) * n + gy0 + q) * (n + 1) + n] = T(0);
    }
    if (y0 + TY * H == n && yj == TY - 1) {
      for (int gz = S.zs * H; gz < S.ze * H; ++gz) Y.c[1][(static_cast<int64_t>(gz) * (n + 1) + n) * n + gx] = T(0);
    }
  }
}

}  // namespace zm
// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
namespace zmhost {

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SMG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw cuda_error("cuTensorMapEncodeTiled not available");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <typename T>
void encode(CUtensorMap* map, const void* base, const uint64_t* dims, const uint64_t* strides_bytes,
            const uint32_t* box) {
  const uint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 3, const_cast<void*>(base), dims, strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

// plane boxes (XB x YE x 1) over the held part of u_y (rows 1..n-1: the constrained rows are OOB),
// u_z (all planes incl. the top one) and p
template <typename T, class C>
zm::ZMaps make_maps(const LevelLayout& lay, const T* x) {
  zm::ZMaps M;
  std::memset(&M, 0, sizeof(M));
  const int H = lay.k + 1;
  const uint64_t es = sizeof(T), nn = static_cast<uint64_t>(lay.n);
  const uint64_t nz = static_cast<uint64_t>(lay.zhi - lay.zlo) * H;
  const uint32_t box[3] = {static_cast<uint32_t>(C::XB), static_cast<uint32_t>(C::YE), 1u};
  {
    const uint64_t d[3] = {nn, nn - 1, nz};
    const uint64_t s[2] = {nn * es, nn * (nn + 1) * es};
    encode<T>(&M.u1, x + lay.off[1] + nn, d, s, box);
  }
  {
    const uint64_t d[3] = {nn, nn, nz + 1};
    const uint64_t s[2] = {nn * es, nn * nn * es};
    encode<T>(&M.u2, x + lay.off[2], d, s, box);
  }
  {
    const uint64_t d[3] = {nn, nn, nz};
    const uint64_t s[2] = {nn * es, nn * nn * es};
    encode<T>(&M.p, x + lay.off[3], d, s, box);
  }
  return M;
}

template <typename T>
zm::ZBlocks<T> bases(const LevelLayout& lay, T* v) {
  zm::ZBlocks<T> B;
  const int H = lay.k + 1;
  for (int c = 0; c < 4; ++c) B.c[c] = v ? v + lay.off[c] - static_cast<int64_t>(lay.zlo) * H * lay.plane[c] : nullptr;
  return B;
}

// z-march shapes: (TX, TY) cells per tile, resident CTAs per SM
template <typename T, int K>
struct ZShape;
template <>
struct ZShape<double, 1> { static constexpr int TX = 16, TY = 4, OCC = 2; };
template <>
struct ZShape<float, 1> { static constexpr int TX = 16, TY = 4, OCC = 3; };
template <>
struct ZShape<double, 2> { static constexpr int TX = 8, TY = 4, OCC = 2; };
template <>
struct ZShape<float, 2> { static constexpr int TX = 8, TY = 4, OCC = 3; };

// true if the z-march kernel handles this launch (else the brick kernel runs)
template <typename T, int K>
bool usable(const Context& ctx, int level, const VmultArgs& a) {
  using S = ZShape<T, K>;
  using C = zm::Cfg<T, K, S::TX, S::TY, S::OCC>;
  // opt-in (SMG_ZMARCH=1): measured 2.6x slower than the brick kernel at C2 (K1z)
  static const bool on = std::getenv("SMG_ZMARCH") != nullptr;
  if (!on) return false;
  const LevelLayout& lay = ctx.dev[0][level].lay;
  const int m = lay.m, n = lay.n;
  if (m % S::TX != 0 || m % S::TY != 0) return false;
  if ((static_cast<int64_t>(n) * sizeof(T)) % 16 != 0) return false;
  if (C::XB > n - 1 || C::YE > n - 1) return false;  // boxes within the tensor extents
  for (int c = 0; c < 4; ++c)
    if ((reinterpret_cast<uintptr_t>(a.x) + lay.off[c] * sizeof(T)) % 16 != 0) return false;
  return true;
}

template <typename T, int K>
void launch(Context& ctx, int level, const VmultArgs& a) {
  using S = ZShape<T, K>;
  using C = zm::Cfg<T, K, S::TX, S::TY, S::OCC>;
  static_assert(C::BYTES * S::OCC <= 233472 - 1024 * S::OCC, "z-march tile exceeds the shared memory of its occupancy");
  const int m = ctx.dev[0][level].lay.m;
  const LevelLayout lay = a.slab ? LevelLayout(K, level, a.zlo, a.zhi) : ctx.dev[0][level].lay;
  if (a.slab) {
    if (a.z0 < 0 || a.z1 > m || a.z0 >= a.z1 || a.zlo > std::max(a.z0 - 1, 0) || a.zhi < std::min(a.z1 + 1, m) ||
        a.zlo < 0 || a.zhi > m)
      throw std::invalid_argument("slab: the held cells must cover the computed cells plus one neighbour cell layer");
  }
  const zm::ZBlocks<const T> X = bases(lay, static_cast<const T*>(a.x));
  const zm::ZBlocks<T> Y = bases(lay, static_cast<T*>(a.y));
  const zm::ZBlocks<const T> B = bases(lay, static_cast<const T*>(a.b));
  const T h = static_cast<T>(1.0 / m);
  // tensor maps cached per (vector, layout) in the context's global slots (vmult_kernel.cuh scheme),
  // tagged so the brick kernel's maps of the same vector are not mistaken for these
  const TmapKey key{a.x, level + 1000, static_cast<int>(sizeof(T)), a.zlo, a.zhi};
  auto it = ctx.tmap_slots.find(key);
  if (it == ctx.tmap_slots.end()) {
    const int slot = tmap_alloc_slot(ctx);
    zm::ZMaps mh = make_maps<T, C>(lay, static_cast<const T*>(a.x));
    char* dst = static_cast<char*>(ctx.tmap_dev) + static_cast<size_t>(slot) * kTmapSlotBytes;
    SMG_CUDA(cudaMemcpyAsync(dst, &mh, sizeof(mh), cudaMemcpyHostToDevice, ctx.stream));
    SMG_CUDA(cudaStreamSynchronize(ctx.stream));
    it = ctx.tmap_slots.emplace(key, slot).first;
  }
  static_assert(sizeof(zm::ZMaps) <= kTmapSlotBytes, "tensor-map slot too small");
  const zm::ZMaps* dmaps =
      reinterpret_cast<const zm::ZMaps*>(static_cast<char*>(ctx.tmap_dev) + static_cast<size_t>(it->second) * kTmapSlotBytes);
  if (ctx.tmap_recording) ctx.tmap_recorded.insert(it->second);
  const int units = (m / S::TX) * (m / S::TY) * (a.z1 - a.z0);
  const dim3 grid(std::min(units, S::OCC * ctx.num_sms));
  auto go = [&](auto kern) {
    ensure_smem_attr(reinterpret_cast<const void*>(kern), ctx.device, C::BYTES);
    kern<<<grid, C::NT, C::BYTES, ctx.stream>>>(X, Y, B, m, a.z0, a.z1, lay.zlo, lay.zhi, h, dmaps);
  };
  if (a.b) go(zm::zm_vmult_kernel<T, K, S::TX, S::TY, S::OCC, true>);
  else go(zm::zm_vmult_kernel<T, K, S::TX, S::TY, S::OCC, false>);
  SMG_CUDA(cudaGetLastError());
  ++ctx.launches;
}

}  // namespace zmhost

// entry points (vmult_zm_k<K>.cu): false if the z-march kernel does not handle this launch
template <int K>
bool zm_vmult_launch_k(Context& ctx, int level, int prec, const VmultArgs& a) {
  if (prec == SMG_F64) {
    if (!zmhost::usable<double, K>(ctx, level, a)) return false;
    zmhost::launch<double, K>(ctx, level, a);
  } else {
    if (!zmhost::usable<float, K>(ctx, level, a)) return false;
    zmhost::launch<float, K>(ctx, level, a);
  }
  return true;
}

template <int K>
void zm_upload_k(const double* t, const float* f) {
  SMG_CUDA(cudaMemcpyToSymbol(zm_ref_d, t, sizeof(double) * kRefTotal));
  SMG_CUDA(cudaMemcpyToSymbol(zm_ref_f, f, sizeof(float) * kRefTotal));
}

#define SMG_INSTANTIATE_ZM(K)                                                        \
  template bool zm_vmult_launch_k<K>(Context&, int, int, const VmultArgs&);          \
  template void zm_upload_k<K>(const double*, const float*);

}  // namespace smg
