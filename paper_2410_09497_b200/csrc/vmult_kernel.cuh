#pragma once
// K1/K2: matrix-free Stokes operator y = A x and residual r = b - A x on sm_100a.
//
// Reference: apply_stokes evaluated by Alg. 1. On the uniform
// Cartesian unit cube the cell/face loops of Alg. 1 equal a Kronecker sum of banded 1D operators
// (re-verified by the GPU-vs-Alg.1-oracle parity tests to 1e-13). Per velocity
// component c with orthogonal axes o1, o2 (all 1D blocks at reference size h = 1, see
// setup1d.hpp reference_cell_tables; level scaling applied once at the output):
//   pass 1 (along o2):  A1 = M_o2 u_c,            B1 = L_o2 u_c
//   pass 2 (along o1):  S  = M_o1 A1,             T  = L_o1 A1 + M_o1 B1
//   pass 3 (along c) :  y_c = h (L_c S + M_c T) + h^2 D_c^T Q,   y_p += h^2 D_c S
// with Q = M_o1 M_o2 p. Every pass is "one thread per pencil": a thread loads a 1D line of the
// brick from shared memory into registers, applies the banded cell-block operator with fully
// unrolled loops whose coefficients are compile-time offsets into __constant__ memory (so they are
// DFMA constant-bank operands, no loads), and writes the result line back. Index arithmetic is per
// pencil, never per element. Domain-boundary Nitsche rows are a CTA-uniform correction applied only
// by bricks that touch the boundary; constrained (boundary-normal) rows / inputs are masked.
//
// One CTA owns a brick of BX x BY x BZ cells. HBM traffic is one read of x and one write of y
// (16 B/DoF in fp64); the one-cell halos of neighbouring bricks are re-read from L2. Inputs are
// staged by TMA (cp.async.bulk.tensor) into double-buffered shared memory, see the persistent kernel.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>
#include <type_traits>

#include "smg_internal.cuh"
#include "vmult.cuh"

namespace smg {

// each translation unit (one per degree, vmult_k<K>.cu) holds its own copy of the tables
static __constant__ double c_ref_d[kRefTotal];
static __constant__ float c_ref_f[kRefTotal];

namespace {

template <typename T>
__device__ __forceinline__ T cref(int i);
template <>
__device__ __forceinline__ double cref<double>(int i) { return c_ref_d[i]; }
template <>
__device__ __forceinline__ float cref<float>(int i) { return c_ref_f[i]; }

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

constexpr int odd(int v) { return v | 1; }

// Asynchronous global->shared copy of one element with zero fill (cp.async, LDGSTS): when `ok` is
// false nothing is read and the destination is zeroed -- this implements the halo outside the
// domain and the constrained boundary-normal entries without any masking pass.
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = ok ? static_cast<int>(sizeof(T)) : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(src), "n"(sizeof(T)), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------------------------
// register-pencil banded operators
// ---------------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------------
// brick geometry
// ---------------------------------------------------------------------------------------------
// QDB (default on where it fits): second Q buffer and no CTA barrier after pass 3 (the last warp to
// finish its pass-3 reads issues the next staging into the component's U buffer)
#ifndef SMG_VMULT_QDB
#define SMG_VMULT_QDB 1
#endif
template <typename T, int K, int BX, int BY, int BZ, int OCC>
struct Brick {
  static constexpr int H = K + 1;
  static constexpr int VEC = 16 / static_cast<int>(sizeof(T));  // elements per 16 B (TMA granule)
  static constexpr int ALN = 128 / static_cast<int>(sizeof(T));  // elements per 128 B (TMA smem alignment)
  static constexpr int PADF = ALN;  // front pad of a TMA box buffer: room for the x < 0 halo of clamped boxes
  static constexpr int rup(int v) { return (v + VEC - 1) / VEC * VEC; }
  static constexpr int rupa(int v) { return (v + ALN - 1) / ALN * ALN; }
  static constexpr int B(int a) { return a == 0 ? BX : (a == 1 ? BY : BZ); }
  static constexpr int N(int a) { return B(a) * H; }
  static constexpr int O1(int c) { return c == 0 ? 1 : 0; }
  static constexpr int O2(int c) { return c == 2 ? 1 : 2; }
  static constexpr int LC(int c) { return N(c) + H + 1; }       // c range [-H, N_c]
  static constexpr int PC(int c) { return odd(LC(c)); }         // padded c extent of intermediates
  static constexpr int LO1H(int c) { return N(O1(c)) + 2 * H; }  // o1 range [-H, N + H)
  static constexpr int LO2H(int c) { return N(O2(c)) + 2 * H; }
  // staged input box of component c, TMA box order (x fastest, x pitch UX):
  //   c=0: [z=o2][y=o1][x=c]   c=1: [z=o2][y=c][x=o1]   c=2: [z=c][y=o2][x=o1]
  // TMA (measured on B200, tools/tma_test.cu) needs the x start of a box 16-B aligned and >= 0 and the
  // shared-memory destination 128-B aligned. Every row is loaded from the 16-B aligned position at or
  // below the needed start (clamped to 0); UX carries VEC-1 elements of slack and the consumers add
  // the per-brick shift PADF + x0 - xs (per sub-box shift for the u_x rows, u0_row).
  static constexpr int XEXT(int c) { return c == 0 ? LC(0) : LO1H(c); }
  static constexpr int UX(int c) { return rup(XEXT(c) + VEC - 1); }
  static constexpr int UY(int c) { return c == 0 ? LO1H(0) : (c == 1 ? LC(1) : LO2H(2)); }
  static constexpr int UZ(int c) { return c == 2 ? LC(2) : LO2H(c); }
  // u_x rows have the odd pitch n+1, so the rows y = q (mod VEC) form VEC tensors with a 16-B aligned
  // pitch VEC (n+1) (make_maps): the u_x box is staged as VEC sub-boxes, sub-box s holding the rows
  // y0 + s + VEC i (i < UYS) of every z plane, each sub-box 128-B aligned
  static constexpr int UYS = (LO1H(0) + VEC - 1) / VEC;
  static constexpr int SUB0 = rupa(UX(0) * UYS * UZ(0));
  static constexpr int sizeU(int c) { return c == 0 ? VEC * SUB0 : UX(c) * UY(c) * UZ(c); }  // elements staged
  static constexpr int sizeA1(int c) { return N(O2(c)) * LO1H(c) * PC(c); }
  static constexpr int sizeST(int c) { return N(O2(c)) * N(O1(c)) * PC(c); }
  static constexpr int mx3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
  static constexpr int U = rupa(PADF + mx3(sizeU(0), sizeU(1), sizeU(2)) + VEC);  // + clamp slack
  static constexpr int A1 = mx3(sizeA1(0), sizeA1(1), sizeA1(2));
  static constexpr int ST = mx3(sizeST(0), sizeST(1), sizeST(2));
  static constexpr int PXT = rup(N(0) + H + VEC - 1);  // pressure box [-H, N) per axis, x pitch PXT
  static constexpr int PBOX = (N(2) + H) * (N(1) + H) * PXT;
  static constexpr int PBUF = rupa(PADF + PBOX + VEC);
  static constexpr int YX = odd(N(0));
  static constexpr int YP = N(2) * N(1) * YX;
  static constexpr bool ALIAS = 2 * ST <= U;  // S and T overwrite the dead U buffer of the component
  // layout: [U buffer 0][U buffer 1][P box][A1 (also Q2)][B1][Q][YP][S,T if no alias][mbarriers]
  // two U buffers (staging of the next component overlaps compute) when they fit in the per-CTA share
  // of the 228 KB SM (OCC resident CTAs, 1 KB reserved per CTA), else one
  static constexpr size_t kSmemCap = OCC == 1 ? 232448 : 233472 / OCC - 1024;
  static constexpr size_t rup16(size_t b) { return (b + 15) / 16 * 16 + 3 * 8; }
  // double-buffered layout: [U0][U1][P][A1][B1][Q][YP] (+[S][T] unless they alias the dead U buffer)
  static constexpr size_t bytes_db() {
    return rup16(static_cast<size_t>(2 * U + PBUF + A1 + 2 * ST + YP + (ALIAS ? 0 : 2 * ST)) * sizeof(T));
  }
  // single-buffered "early release" layout: [U][P][A1][B1=T][Q][YP][S]; U is dead after pass 1, so the
  // next component's staging is issued there and overlaps passes 2-3 and the next Q passes
  static constexpr size_t bytes_sb() { return rup16(static_cast<size_t>(U + PBUF + A1 + 3 * ST + YP) * sizeof(T)); }
  // double-buffered layout + a second Q buffer (QDB): pass 3 of component c reads Q while pass 1 of
  // component c+1 writes its Q2 into the other buffer, so no CTA barrier is needed after pass 3
  static constexpr size_t bytes_dbq() {
    return rup16(static_cast<size_t>(2 * U + PBUF + A1 + 3 * ST + YP + (ALIAS ? 0 : 2 * ST)) * sizeof(T));
  }
  static constexpr bool DB = bytes_db() <= kSmemCap;
  // measured (tools/ab_lib.py, profiles/r02/ab_vmult_qdb.jsonl): k = 2 fp64 -2.1 %, k = 3 -1.1 %; k = 1 fp32
  // +3 %, k = 4 fp64 +4 %, k = 5 / 6 fp64 +20 % (ab_vmult_qdb_high_degree.jsonl) -> k = 2, 3 only
  static constexpr bool QDB = SMG_VMULT_QDB && (K == 2 || K == 3) && DB && bytes_dbq() <= kSmemCap;
  static constexpr size_t bytes_for(int nbuf) { return nbuf == 2 ? (QDB ? bytes_dbq() : bytes_db()) : bytes_sb(); }
  static constexpr int OFF_U1 = DB ? U : 0;
  static constexpr int OFF_P = (DB ? 2 : 1) * U;
  static constexpr int OFF_A1 = OFF_P + PBUF;
  static constexpr int OFF_B1 = OFF_A1 + A1;
  static constexpr int OFF_Q = OFF_B1 + ST;
  static constexpr int OFF_YP = OFF_Q + ST;
  static constexpr int OFF_ST = OFF_YP + YP;  // DB && !ALIAS: S, T; SB: S
  static constexpr int OFF_Q2 = OFF_ST + (ALIAS ? 0 : 2 * ST);  // QDB: second Q buffer
  static constexpr int END = DB ? OFF_Q2 + (QDB ? ST : 0) : OFF_YP + YP + ST;
  static constexpr size_t BYTES = (static_cast<size_t>(END) * sizeof(T) + 15) / 16 * 16 + 3 * 8;
  static_assert(BYTES == bytes_for(DB ? 2 : 1), "smem layout");
  static constexpr int stride(int axis, int a0, int a1) { return axis == 0 ? 1 : (axis == 1 ? a0 : a0 * a1); }
};

struct Maps {
  CUtensorMap u1, u2, p;  // 3D boxes of u_y, u_z, p
  CUtensorMap u0[4];      // u_x rows y = q (mod VEC), q < VEC (Brick::SUB0)
};

// per-block base pointers [u_x, u_y, u_z, p] in the GLOBAL index space of the level: for a z-slab
// vector the bases are virtual (shifted back by the slab's first plane), so the kernel
// indexes globally and only ever touches planes the slab holds.
template <typename T>
struct Blocks {
  T* c[4];
};

struct Geo {
  int m, n;
  int nlim[3];  // exclusive node limit of the outputs per axis (n, n, z_end * H)
  int mlim[3];  // exclusive cell limit per axis (m, m, z_end)
  int zoff;     // first z node plane the vector holds (0, or zlo * H for a slab): TMA maps are slab-local
  int zend;     // one past the last z node plane of the held cells (u_z holds one more plane)
  int c0[3];  // brick cell origin
  int g0[3];  // brick node origin
};

// ---------------------------------------------------------------------------------------------
// mbarrier / TMA primitives
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ void tma_load_1d(void* dst, const CUtensorMap* map, int x, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(smem_u32(bar))
      : "memory");
}

// floor to a multiple of the power of two q (two's complement: also right for negative v)
__device__ __forceinline__ int floor_to(int v, int q) { return v & -q; }

// smem origin offsets of the staged rows (element of x = g0x - H relative to the row start)
// smem position of element x0 in a staged 3D box row: PADF + x0 - xs, xs = max(floor16B(x0), 0);
// negative x0 (boxes clamped at the domain start) lands in the front pad / the previous row's unused tail
template <typename T>
__device__ __forceinline__ int brick_shift(const Geo& G, int H) {
  constexpr int VEC = 16 / static_cast<int>(sizeof(T));
  constexpr int PADF = 128 / static_cast<int>(sizeof(T));
  const int x0 = G.g0[0] - H;
  return PADF + x0 - max(floor_to(x0, VEC), 0);
}
// u_x box: smem offset of the element (x = x0 = g0x - H, local row oi, plane 0). Row oi lives in
// sub-box s = oi % VEC (row i = oi / VEC), loaded from the map of rows y = q (mod VEC),
// q = (y0 + s) mod VEC, whose x coordinate is x' = x + q; the box starts at xs = max(floor16B(x0 + q), 0)
template <typename T, int SUB0, int UX>
__device__ __forceinline__ int u0_row(const Geo& G, int H, int oi) {
  constexpr int VEC = 16 / static_cast<int>(sizeof(T));
  constexpr int PADF = 128 / static_cast<int>(sizeof(T));
  const int s = oi & (VEC - 1);
  const int q = (G.g0[1] - H + s) & (VEC - 1);
  const int x0 = G.g0[0] - H;
  return PADF + s * SUB0 + (oi / VEC) * UX + x0 + q - max(floor_to(x0 + q, VEC), 0);
}

// ---------------------------------------------------------------------------------------------
// staging: TMA (default) or cp.async element copies (fallback when a pitch is not 16-B aligned,
// i.e. fp32 on level 0 with even k). Both write the same TMA box layout.
// ---------------------------------------------------------------------------------------------
// SINGLE: called by one thread (QDB: the U barriers then count one arrival, the issuer's expect_tx);
// otherwise called by every thread and thread 0 issues while the other warps arrive once each
template <typename T, int K, int BX, int BY, int BZ, int OCC, int NT, int C, bool TMA, bool SINGLE = false>
__device__ __forceinline__ void issue_u(T* sU, uint64_t* bar, const Blocks<const T>& X, const Maps& M, const Geo& G) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  constexpr int H = K + 1;
  constexpr int UX = BR::UX(C), UY = BR::UY(C), UZ = BR::UZ(C);
  const int n = G.n;
  const int tid = threadIdx.x;
  if constexpr (TMA) {
    if constexpr (C == 0) {
      // VEC sub-boxes from the row-residue maps u0[q] (Brick::SUB0); rows / planes outside the domain
      // are OOB-filled with zeros, the columns x <= 0 and x >= n are zeroed by fix_columns
      if (SINGLE || tid == 0) {
        constexpr int VEC = BR::VEC;
        mbar_expect(bar, static_cast<unsigned>(VEC * UX * BR::UYS * UZ * sizeof(T)));
        const int y0 = G.g0[1] - H, x0 = G.g0[0] - H, zc = G.g0[2] - H - G.zoff;
#pragma unroll
        for (int s = 0; s < VEC; ++s) {
          const int q = (y0 + s) & (VEC - 1);
          // rows y0 + s + VEC i = VEC (j0 + i) + q of map q (exact: y0 + s - q is a multiple of VEC)
          const int j0 = (y0 + s - q) / VEC;
          tma_load_3d(sU + BR::PADF + s * BR::SUB0, &M.u0[q], max(floor_to(x0 + q, VEC), 0), j0, zc, bar);
        }
      } else if ((tid & 31) == 0) {
        mbar_arrive(bar);  // the U barriers count one arrival per warp
      }
    } else {
      if (SINGLE || tid == 0) {
        mbar_expect(bar, static_cast<unsigned>(BR::sizeU(C) * sizeof(T)));
        // the u_y map starts one row in, so its constrained rows 0 and n fall outside
        const int xs = max(floor_to(G.g0[0] - H, BR::VEC), 0);
        if (C == 1) tma_load_3d(sU + BR::PADF, &M.u1, xs, G.g0[1] - H - 1, G.g0[2] - H - G.zoff, bar);
        else tma_load_3d(sU + BR::PADF, &M.u2, xs, G.g0[1] - H, G.g0[2] - H - G.zoff, bar);
      } else if ((tid & 31) == 0) {
        mbar_arrive(bar);  // the U barriers count one arrival per warp
      }
    }
  } else {
    int gd[3] = {n, n, n};
    gd[C] = n + 1;
    const T* xc = X.c[C];
    constexpr int XE = BR::XEXT(C);
    for (int i = tid; i < XE * UY * UZ; i += NT) {
      const int l[3] = {i % XE - H, (i / XE) % UY - H, i / (XE * UY) - H};
      const int g[3] = {G.g0[0] + l[0], G.g0[1] + l[1], G.g0[2] + l[2]};
      bool ok = g[0] >= 0 && g[1] >= 0 && g[2] >= 0 && g[0] < gd[0] && g[1] < gd[1] && g[2] < gd[2];
      ok = ok && g[C] != 0 && g[C] != n && g[2] >= G.zoff && g[2] < G.zend + (C == 2);
      const T* src = ok ? xc + (static_cast<int64_t>(g[2]) * gd[1] + g[1]) * gd[0] + g[0] : xc;
      T* dst = C == 0 ? sU + u0_row<T, BR::SUB0, UX>(G, H, l[1] + H) + (l[2] + H) * BR::UYS * UX
                      : sU + (i / XE) * UX + brick_shift<T>(G, H);
      cp_async_elem(dst + (l[0] + H), src, ok);
    }
  }
}

template <typename T, int K, int BX, int BY, int BZ, int OCC, int NT, bool TMA>
__device__ __forceinline__ void issue_p(T* sP, uint64_t* bar, const Blocks<const T>& X, const Maps& M, const Geo& G) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  constexpr int H = K + 1;
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_expect(bar, static_cast<unsigned>(BR::PBOX * sizeof(T)));
      const int xs = max(floor_to(G.g0[0] - H, BR::VEC), 0);
      tma_load_3d(sP + BR::PADF, &M.p, xs, G.g0[1] - H, G.g0[2] - H - G.zoff, bar);
    }
  } else {
    constexpr int E0 = BR::N(0) + H, E1 = BR::N(1) + H, E2 = BR::N(2) + H;
    const int n = G.n;
    const int sh = brick_shift<T>(G, H);
    const T* xp = X.c[3];
    for (int i = threadIdx.x; i < E0 * E1 * E2; i += NT) {
      const int lx = i % E0, ly = (i / E0) % E1, lz = i / (E0 * E1);
      const int gx = G.g0[0] + lx - H, gy = G.g0[1] + ly - H, gz = G.g0[2] + lz - H;
      const bool ok = gx >= 0 && gy >= 0 && gz >= G.zoff && gx < n && gy < n && gz < G.zend;
      const T* src = ok ? xp + (static_cast<int64_t>(gz) * n + gy) * n + gx : xp;
      cp_async_elem(sP + (lz * E1 + ly) * BR::PXT + sh + lx, src, ok);
    }
  }
}

// CTA-uniform: does fix_columns write anything for these boxes? (interior bricks skip it and the barrier
// after it: every thread waits on the box's mbarrier itself, so the TMA data needs no CTA barrier)
template <typename T, int K, int BX, int BY, int BZ, int OCC>
__device__ __forceinline__ bool fix_needed(bool u0, bool u2, const Geo& G) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  constexpr int H = K + 1;
  const int x0 = G.g0[0] - H, zb = G.g0[2] - H;
  if (x0 < 0) return true;
  if (u0 && !(x0 > 0 && x0 + BR::XEXT(0) <= G.n)) return true;
  return u2 && (zb <= 0 || zb + BR::UZ(2) > G.n);
}

// Boundary fix-ups after a TMA box landed (bricks touching the x ends only):
//  - u_x rows (row-residue maps: the x < 0 columns of a row are the previous row's tail): zero the
//    columns outside [1, n-1] (halo beyond the domain and the constrained boundary-normal nodes x = 0, x = n);
//  - u_y, u_z, p boxes clamped at x = 0 leave the x < 0 halo columns unwritten: zero them.
template <typename T, int K, int BX, int BY, int BZ, int OCC, int NT>
__device__ __forceinline__ void fix_columns(T* sU0, T* sU1, T* sU2, T* sP, const Geo& G) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  constexpr int H = K + 1;
  const int x0 = G.g0[0] - H;
  if (sU2) {
    // u_z boxes hold every z plane of the vector: zero the constrained planes z = 0 and z = n
    constexpr int PL = BR::UY(2) * BR::UX(2);
    const int zb = G.g0[2] - H;  // global plane of box plane 0
    if (zb <= 0)
      for (int i = threadIdx.x; i < PL; i += NT) sU2[BR::PADF + (0 - zb) * PL + i] = T(0);
    if (zb + BR::UZ(2) > G.n)
      for (int i = threadIdx.x; i < PL; i += NT) sU2[BR::PADF + (G.n - zb) * PL + i] = T(0);
  }
  if (x0 > 0 && x0 + BR::XEXT(0) <= G.n) return;
  if (sU0) {
    // only the columns gx <= 0 (left end: x0 <= 0) or gx >= n (right end) of every row
    constexpr int XE = BR::XEXT(0), UY = BR::UY(0), ROWS = BR::UY(0) * BR::UZ(0);
    const int lo = x0 <= 0 ? 1 - x0 : 0;                  // columns [0, lo) have gx <= 0
    const int hi = G.n - x0 < XE ? G.n - x0 : XE;          // columns [hi, XE) have gx >= n
    const int nl = lo, nr = XE - hi, per = nl + nr;
    for (int i = threadIdx.x; i < ROWS * per; i += NT) {
      const int r = i / per, j = i - r * per;
      const int col = j < nl ? j : hi + (j - nl);
      sU0[u0_row<T, BR::SUB0, BR::UX(0)>(G, H, r % UY) + (r / UY) * BR::UYS * BR::UX(0) + col] = T(0);
    }
  }
  if (x0 >= 0) return;
  const int sh = brick_shift<T>(G, H);
  auto zero_low = [&](T* buf, int rows, int pitch) {
    for (int i = threadIdx.x; i < rows * H; i += NT) buf[(i / H) * pitch + sh + i % H] = T(0);
  };
  if (sU1) zero_low(sU1, BR::UY(1) * BR::UZ(1), BR::UX(1));
  if (sU2) zero_low(sU2, BR::UY(2) * BR::UZ(2), BR::UX(2));
  if (sP) zero_low(sP, (BR::N(1) + H) * (BR::N(2) + H), BR::PXT);
}

// ---------------------------------------------------------------------------------------------
// 1D kernels on register arrays: one work item = a segment of NC consecutive cells of one 1D line
// ---------------------------------------------------------------------------------------------
// DG mass, block diagonal: out[e*H+a] = sum_b MO[a][b] in[e*H+b]
template <typename T, int K, int NC>
__device__ __forceinline__ void seg_mass(const T (&in)[NC * (K + 1)], T (&out)[NC * (K + 1)]) {
  constexpr int H = K + 1;
#pragma unroll
  for (int e = 0; e < NC; ++e)
#pragma unroll
    for (int a = 0; a < H; ++a) {
      T s = T(0);
#pragma unroll
      for (int b = 0; b < H; ++b) s += cref<T>(Ref<K>::MO + a * H + b) * in[e * H + b];
      out[e * H + a] = s;
    }
}
// DG SIPG rows of NC cells from NC+2 cells of input (one neighbour cell each side, zero-filled
// outside the domain). The off-diagonal blocks are cross shaped for the Gauss-Lobatto basis
// (LOM[a][b] != 0 only if a == 0 or b == K, LOP only if a == K or b == 0). BND: the segment may hold
// the first / last cell of the global line (local index efirst / elast, -1 if not): Nitsche rows.
template <typename T, int K, int NC, bool BND>
__device__ __forceinline__ void seg_sipg(const T (&in)[(NC + 2) * (K + 1)], T (&out)[NC * (K + 1)], int efirst,
                                         int elast) {
  constexpr int H = K + 1;
  using R = Ref<K>;
#pragma unroll
  for (int e = 0; e < NC; ++e)
#pragma unroll
    for (int a = 0; a < H; ++a) {
      T s = T(0);
#pragma unroll
      for (int b = 0; b < H; ++b) s += cref<T>(R::LO0 + a * H + b) * in[(e + 1) * H + b];
#pragma unroll
      for (int b = 0; b < H; ++b)
        if (a == 0 || b == K) s += cref<T>(R::LOM + a * H + b) * in[e * H + b];
#pragma unroll
      for (int b = 0; b < H; ++b)
        if (a == K || b == 0) s += cref<T>(R::LOP + a * H + b) * in[(e + 2) * H + b];
      if (BND) {
        if (e == efirst) {
#pragma unroll
          for (int b = 0; b < H; ++b) s += cref<T>(R::DLF + a * H + b) * in[(e + 1) * H + b];
        }
        if (e == elast) {
#pragma unroll
          for (int b = 0; b < H; ++b) s += cref<T>(R::DLL + a * H + b) * in[(e + 1) * H + b];
        }
      }
      out[e * H + a] = s;
    }
}
template <bool V>
using bool_c = std::integral_constant<bool, V>;
// u_x outputs (x = the pencil axis of component 0) staged in smem for coalesced x-row stores, or
// stored directly from the pencils
#ifndef SMG_STAGE_UX
#define SMG_STAGE_UX 0
#endif
constexpr bool kStageUx = SMG_STAGE_UX;
#ifndef SMG_VMULT_WIDE_A
#define SMG_VMULT_WIDE_A 1
#endif
constexpr bool kWideA = SMG_VMULT_WIDE_A;  // component(): AWIDE
// cells per work item along a brick axis of nc cells: segments of 2 cells for low degrees (shared
// neighbour loads, fewer index computations), single cells otherwise
constexpr int seg_cells(int nc, int k) { return (nc % 2 == 0 && k <= 3) ? 2 : 1; }
// row groups of the pass-3 items: the smallest divisor d of H with items * d >= threads, for k >= 7
// (few, heavy items); 1 otherwise
constexpr int pass3_groups(int items, int nt, int h, int k) {
  if (k < 7) return 1;  // measured: helps k = 7 (33.3 -> 30.9 ms at level 5), hurts k = 4..6
  for (int d = 1; d <= h && d <= 8; ++d)
    if (h % d == 0 && items * d >= nt) return d;
  int best = 1;
  for (int d = 1; d <= h && d <= 8; ++d)
    if (h % d == 0) best = d;
  return best;
}

// ---------------------------------------------------------------------------------------------
// one velocity component (U already staged in sU); if C == 2 and Gn != nullptr, the next brick's
// pressure box is issued as soon as this brick's P box is dead. Every pass is a loop over
// (cell, line) work items -- NT threads get several times more items than there are 1D lines, so
// the passes stay balanced and the dependency chains short (v5; v2-v4 used one thread per line).
// ---------------------------------------------------------------------------------------------
template <typename T, int K, int BX, int BY, int BZ, int OCC, int NT, int C, bool RESID, bool TMA>
__device__ __forceinline__ void component(T* sm, T* sU, const Geo& G, T h, const Geo* Gn, const Blocks<const T>& X,
                                          const Blocks<T>& Y, const Blocks<const T>& B, const Maps& M, uint64_t* barP,
                                          uint64_t* barU = nullptr, unsigned* phU = nullptr, int nextC = -1,
                                          const Geo* Gnext = nullptr, int qsel = 0) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  using R = Ref<K>;
  constexpr int H = K + 1, P = K + 2;
  constexpr int O1 = BR::O1(C), O2 = BR::O2(C);
  constexpr int NCc = BR::B(C), NO1 = BR::B(O1), NO2 = BR::B(O2);
  constexpr int Nc = BR::N(C), No1 = BR::N(O1), No2 = BR::N(O2);
  constexpr int LC = BR::LC(C), PC = BR::PC(C), LO1H = BR::LO1H(C);
  constexpr int UX = BR::UX(C), UY = BR::UY(C);
  const int tid = threadIdx.x;
  const int n = G.n, m = G.m;
  int64_t gd[3] = {n, n, n};
  gd[C] = n + 1;
  const int64_t st[3] = {1, gd[0], gd[0] * gd[1]};

  T* sA1 = sm + BR::OFF_A1;
  T* sB1 = sm + BR::OFF_B1;
  T* sQ = sm + (BR::QDB && qsel ? BR::OFF_Q2 : BR::OFF_Q);
  T* sP = sm + BR::OFF_P;
  T* sYP = sm + BR::OFF_YP;
  T* sS = (BR::DB && BR::ALIAS) ? sU : sm + BR::OFF_ST;
  T* sT = BR::DB ? sS + BR::ST : sB1;  // single-buffer layout: T overwrites B1 in place (same cell block)

  constexpr int SQ2 = seg_cells(NO2, K), SQ = seg_cells(NO1, K), S1 = seg_cells(NO2, K), S2 = seg_cells(NO1, K),
                S3 = seg_cells(NCc, K);
  // Q = M_o1 M_o2 p (c in [-H, N_c), o1 / o2 owned) is computed inside passes 1 and 2: Q2 = M_o2 p
  // with the B1 items, then Q = M_o1 Q2 in place (block-diagonal mass: same cell block) with the S/T
  // items -- no separate passes or barriers for the pressure.
  constexpr int E1P = BR::N(1) + H;
  constexpr int PSC = BR::stride(C, BR::PXT, E1P), PSO1 = BR::stride(O1, BR::PXT, E1P),
                PSO2 = BR::stride(O2, BR::PXT, E1P);
  if constexpr (!BR::DB) {
    // single-buffer mode: U of this component was issued during the previous component's passes 2-3
    if (TMA) {
      mbar_wait(barU, *phU);
      *phU ^= 1;
      if (fix_needed<T, K, BX, BY, BZ, OCC>(C == 0, C == 2, G)) {
        fix_columns<T, K, BX, BY, BZ, OCC, NT>(C == 0 ? sU : nullptr, C == 1 ? sU : nullptr, C == 2 ? sU : nullptr,
                                               nullptr, G);
        __syncthreads();
      }
    } else {
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
    }
  }
  // ---- pass 1 (along o2): A1 = M_o2 U (c full, o1 with halo, o2 owned); B1 = L_o2 U (o1 owned) ----
  {
    constexpr int US = C == 2 ? UX : (C == 0 ? UX * BR::UYS : UX * UY);  // staged-box stride along o2
    const int bsh = brick_shift<T>(G, H);
    // element (c = ci, o1 = oi, o2 = 0) of the staged box
    auto ub = [&](int ci, int oi) {
      return C == 0 ? u0_row<T, BR::SUB0, UX>(G, H, oi) + ci : (C == 1 ? ci * UX + oi : ci * UY * UX + oi) + bsh;
    };
    constexpr int NLA = LC * LO1H;
    // SA: cells per A item. QDB k = 2 fp64: whole 4-cell o2 lines (288 items, one per thread, more
    // independent loads per item) handed out from the top thread down, so that threads 96..383 take them
    // and the threads 288..383 without a pass-3 item of the previous component start on them at once.
    // Measured (ab_vmult_qdb_wide_a.jsonl): C2 fp64 -1.3 % on top of QDB; fp32 at 32^3 +5 % -> fp64 only
    constexpr bool AWIDE = kWideA && BR::QDB && TMA && K == 2 && sizeof(T) == 8 && NO2 == 4 && NLA * (NO2 / 4) <= NT;
    constexpr int SA = AWIDE ? 4 : S1;
    for (int it = AWIDE ? NT - 1 - tid : tid; it < NLA * (NO2 / SA); it += NT) {
      const int e2 = (it / NLA) * SA, r = it % NLA;
      // consecutive items walk the staged box's x axis: c for C=0, o1 for C=1,2
      const int ci = C == 0 ? r % LC : r / LO1H;
      const int oi = C == 0 ? r / LC : r % LO1H;
      const T* src = sU + ub(ci, oi) + (e2 + 1) * H * US;
      T cu[SA * H], out[SA * H];
#pragma unroll
      for (int j = 0; j < SA * H; ++j) cu[j] = src[j * US];
      seg_mass<T, K, SA>(cu, out);
#pragma unroll
      for (int a = 0; a < SA * H; ++a) sA1[((e2 * H + a) * LO1H + oi) * PC + ci] = out[a];
    }
    const int cell_o2 = G.c0[O2];
    const int psh = brick_shift<T>(G, H);
    auto passB = [&](auto bnd) {
      constexpr bool BND = decltype(bnd)::value;
      constexpr int NLB = LC * No1;
      for (int it = tid; it < NLB * (NO2 / S1); it += NT) {
        const int e2 = (it / NLB) * S1, r = it % NLB;
        const int ci = C == 0 ? r % LC : r / No1;
        const int o = C == 0 ? r / LC : r % No1;
        const T* src = sU + ub(ci, o + H) + e2 * H * US;
        T in[(S1 + 2) * H], out[S1 * H];
#pragma unroll
        for (int j = 0; j < (S1 + 2) * H; ++j) in[j] = src[j * US];
        // the pressure column of Q2 below is loaded up front (its latency overlaps the SIPG rows; the
        // compiler cannot move loads above the sB1 stores); predicated off for the one column that
        // skips Q2 (C = 1, 2: ci = Nc + H, past the P box)
        const bool useq = (C == 0 && K <= 5) || ci < Nc + H;
        const T* ps = sP + psh + ci * PSC + (o + H) * PSO1 + (e2 + 1) * H * PSO2;
        T pc[S1 * H];
#pragma unroll
        for (int j = 0; j < S1 * H; ++j) pc[j] = useq ? ps[j * PSO2] : T(0);
        const int eg = cell_o2 + e2;  // global cell of the segment's first cell
        seg_sipg<T, K, S1, BND>(in, out, eg == 0 ? 0 : -1, (m - 1 - eg < S1) ? m - 1 - eg : -1);
#pragma unroll
        for (int a = 0; a < S1 * H; ++a) sB1[((e2 * H + a) * No1 + o) * PC + ci] = out[a];
        // Q2 = M_o2 p at the same (c, o1, o2-segment); the P box has the same origin. C = 0 walks c
        // fastest, so the last c column (never read as Q) is computed from the P box's pad column rather
        // than branched around in every warp
        if (useq) {  // (k >= 6: the extra column costs more than the branch)
          T q2[S1 * H];
          seg_mass<T, K, S1>(pc, q2);
#pragma unroll
          for (int a = 0; a < S1 * H; ++a) sQ[((e2 * H + a) * No1 + o) * PC + ci] = q2[a];
        }
      }
    };
    if (cell_o2 == 0 || cell_o2 + NO2 >= m) passB(bool_c<true>());
    else passB(bool_c<false>());
  }
  if constexpr (!BR::DB) {
    fence_proxy_async();  // generic reads of U / P happen-before the async-proxy writes of the next staging
    __syncthreads();
    if (C == 2 && Gn != nullptr) issue_p<T, K, BX, BY, BZ, OCC, NT, TMA>(sP, barP, X, M, *Gn);
    if (nextC == 0) issue_u<T, K, BX, BY, BZ, OCC, NT, 0, TMA>(sU, barU, X, M, *Gnext);
    else if (nextC == 1) issue_u<T, K, BX, BY, BZ, OCC, NT, 1, TMA>(sU, barU, X, M, *Gnext);
    else if (nextC == 2) issue_u<T, K, BX, BY, BZ, OCC, NT, 2, TMA>(sU, barU, X, M, *Gnext);
    if (!TMA) cp_async_commit();
  } else {
    fence_proxy_async();
    __syncthreads();
    if (C == 2 && Gn != nullptr) issue_p<T, K, BX, BY, BZ, OCC, NT, TMA>(sP, barP, X, M, *Gn);
    if (!TMA && C == 2) cp_async_commit();
  }
  // ---- pass 2 (along o1): S = M_o1 A1, T = L_o1 A1 + M_o1 B1 (c full, o1/o2 owned) ----
  {
    const int cell_o1 = G.c0[O1];
    auto pass2 = [&](auto bnd) {
      constexpr bool BND = decltype(bnd)::value;
      constexpr int NL = LC * No2;
      for (int it = tid; it < NL * (NO1 / S2); it += NT) {
        const int e1 = (it / NL) * S2, r = it % NL;
        const int ci = r % LC, oj = r / LC;
        const T* a1 = sA1 + (oj * LO1H + e1 * H) * PC + ci;
        const T* b1 = sB1 + (oj * No1 + e1 * H) * PC + ci;
        T in[(S2 + 2) * H], bb[S2 * H];
#pragma unroll
        for (int j = 0; j < (S2 + 2) * H; ++j) in[j] = a1[j * PC];
#pragma unroll
        for (int j = 0; j < S2 * H; ++j) bb[j] = b1[j * PC];
        // Q2 of this item loaded up front (see pass 1; predicated off for the column that skips Q)
        const bool useq = K <= 5 || ci < Nc + H;
        T* q = sQ + (oj * No1 + e1 * H) * PC + ci;
        T q2[S2 * H];
#pragma unroll
        for (int j = 0; j < S2 * H; ++j) q2[j] = useq ? q[j * PC] : T(0);
        T cu[S2 * H];
#pragma unroll
        for (int j = 0; j < S2 * H; ++j) cu[j] = in[H + j];
        T sv[S2 * H], tv[S2 * H], mb[S2 * H];
        seg_mass<T, K, S2>(cu, sv);
        const int eg = cell_o1 + e1;
        seg_sipg<T, K, S2, BND>(in, tv, eg == 0 ? 0 : -1, (m - 1 - eg < S2) ? m - 1 - eg : -1);
        seg_mass<T, K, S2>(bb, mb);
#pragma unroll
        for (int a = 0; a < S2 * H; ++a) {
          sS[(oj * No1 + e1 * H + a) * PC + ci] = sv[a];
          sT[(oj * No1 + e1 * H + a) * PC + ci] = tv[a] + mb[a];
        }
        if (useq) {  // Q = M_o1 Q2 in place (last c column never read as Q, see pass 1)
          T qq[S2 * H];
          seg_mass<T, K, S2>(q2, qq);
#pragma unroll
          for (int j = 0; j < S2 * H; ++j) q[j * PC] = qq[j];
        }
      }
    };
    if (cell_o1 == 0 || cell_o1 + NO1 >= m) pass2(bool_c<true>());
    else pass2(bool_c<false>());
  }
  __syncthreads();
  // ---- pass 3 (along c): y_c = h (L_c S + M_c T) + h^2 D^T Q ;  y_p += h^2 D S ----
  // item (o1 line oi, o2 line oj, cells e0 .. e0+S3-1) reads the window [e0 H, (e0 + S3 + 1) H] of the
  // c pencils
  constexpr int NCP = odd(Nc);
  T* sYC = sA1;  // C = 0: outputs staged in smem (A1 is dead) for a coalesced x-row write-out
  {
    const T h2 = h * h;
    const T* __restrict__ bc = RESID ? B.c[C] : nullptr;
    T* __restrict__ yc = Y.c[C];
    constexpr int YSC = BR::stride(C, BR::YX, BR::N(1)), YSO1 = BR::stride(O1, BR::YX, BR::N(1)),
                  YSO2 = BR::stride(O2, BR::YX, BR::N(1));
    constexpr int NL = No1 * No2;
    constexpr int W = (S3 + 1) * H;  // window length of q; s and t have one more node
    // high degrees: few (cell, line) items and many rows per item -> the H rows of an item are split
    // into RG compile-time row groups (group slowest, so stores stay coalesced)
    constexpr int ITEMS = NL * (NCc / S3);
    constexpr int RG = pass3_groups(ITEMS, NT, H, K);
    constexpr int RPG = H / RG;
    // FULL (CTA-uniform): every row of the brick is held, none is a constrained boundary row, and the
    // brick is not the last along c -- the store predicates drop out of the interior bricks' code
    // fewer items than threads (k = 3: 128 items for 256 threads): the velocity rows and the pressure
    // rows of an item become separate items on disjoint threads (the pressure rows need only S)
    // velocity items on the first PT0 threads (whole warps), pressure items on the rest. Measured
    // (tools/ab_lib.py, C2-size levels): k = 3 fp64 -3.5 %; k = 2 neutral, k = 4 fp64 +17 % -> k = 3 only
    constexpr int PT0 = (ITEMS + 31) / 32 * 32;
    constexpr bool SPLIT = K == 3 && RG == 1 && PT0 < NT;
    auto pass3 = [&](auto fulltag) {
    constexpr bool FULL = decltype(fulltag)::value;
    // MODE 0: velocity and pressure rows of the item, 1: velocity rows only, 2: pressure rows only
    auto item = [&](const int it, auto modetag) {
      constexpr int MODE = decltype(modetag)::value;
      constexpr bool DOV = MODE != 2, DOP = MODE != 1;
      const int grp = it / ITEMS, it0 = it - grp * ITEMS;
      const int e0 = (it0 / NL) * S3, r = it0 % NL;
      const int oi = r % No1, oj = r / No1;
      const int base = (oj * No1 + oi) * PC + e0 * H;
      T s[W + 1], t[W + 1], q[W];
#pragma unroll
      for (int j = 0; j < W + 1; ++j) {
        s[j] = sS[base + j];
        t[j] = DOV ? sT[base + j] : T(0);
      }
#pragma unroll
      for (int j = 0; j < W; ++j) q[j] = DOV ? sQ[base + j] : T(0);
      int g[3];
      g[O1] = G.g0[O1] + oi;
      g[O2] = G.g0[O2] + oj;
      const bool inside = g[O1] < G.nlim[O1] && g[O2] < G.nlim[O2];
      T* yp = sYP + oi * YSO1 + oj * YSO2;
      constexpr bool DIRECT = !(C == 0 && kStageUx);
      // global index of the item's first row (node G.g0[C] + e0 H along c); rows step by st[C]
      const int gc0 = G.g0[C] + e0 * H;
      const int64_t gbase = g[O1] * st[O1] + g[O2] * st[O2] + gc0 * st[C];
      const int64_t pbase = C == 2 ? (static_cast<int64_t>(gc0) * n + g[1]) * n + g[0] : 0;  // pressure, C = 2
      const int64_t pplane = static_cast<int64_t>(n) * n;
      auto rows = [&](auto gtag) {
        constexpr int A0 = decltype(gtag)::value * RPG, A1 = A0 + RPG;  // rows [A0, A1) of each cell
        // residual: the b values of this group's rows are loaded up front so their HBM latency overlaps
        // the contractions (loads inside the store path were exposed: residual 1.8x the plain apply)
        T bvel[S3 * RPG], bpre[S3 * RPG];
        if constexpr (RESID) {
#pragma unroll
          for (int ee = 0; ee < S3; ++ee)
#pragma unroll
            for (int j = 0; j < RPG; ++j) {
              const int row = ee * H + A0 + j;
              bvel[ee * RPG + j] = T(0);
              bpre[ee * RPG + j] = T(0);
              const bool ok = FULL || (inside && gc0 + row < G.nlim[C]);
              if (DOV && DIRECT && ok) bvel[ee * RPG + j] = bc[gbase + row * st[C]];
              if (DOP && C == 2 && ok) bpre[ee * RPG + j] = B.c[3][pbase + row * pplane];
            }
        }
#pragma unroll
        for (int ee = 0; ee < S3; ++ee) {
          const int e = e0 + ee;
#pragma unroll
          for (int a = A0; a < (DOV ? A1 : A0); ++a) {
            T v = T(0), w = T(0);
#pragma unroll
            for (int bq = 0; bq < P; ++bq) {
              v += cref<T>(R::LP + a * P + bq) * s[ee * H + H + bq] + cref<T>(R::MP + a * P + bq) * t[ee * H + H + bq];
              if (a == 0)
                v += cref<T>(R::LP + (K + 1) * P + bq) * s[ee * H + bq] +
                     cref<T>(R::MP + (K + 1) * P + bq) * t[ee * H + bq];
            }
#pragma unroll
            for (int i = 0; i < H; ++i) {
              w += cref<T>(R::D + i * P + a) * q[ee * H + H + i];
              if (a == 0) w += cref<T>(R::D + i * P + H) * q[ee * H + i];
            }
            const T val = h * v + h2 * w;
            if (C == 0 && kStageUx) {
              sYC[(oj * No1 + oi) * NCP + e * H + a] = val;
            } else {
              const int gc = gc0 + ee * H + a;
              if (FULL || (inside && gc < G.nlim[C])) {
                T rr = val;
                if (!FULL && gc == 0) rr = T(0);  // constrained boundary-normal row
                else if (RESID) rr = bvel[ee * RPG + a - A0] - rr;
                yc[gbase + (ee * H + a) * st[C]] = rr;
              }
            }
          }
          // pressure rows of cell e: y_p += h^2 D S
#pragma unroll
          for (int i = A0; i < (DOP ? A1 : A0); ++i) {
            T z = T(0);
#pragma unroll
            for (int bq = 0; bq < P; ++bq) z += cref<T>(R::D + i * P + bq) * s[ee * H + H + bq];
            // y_p = h^2 (D_x S_x + D_y S_y + D_z S_z): component 0 stores, 1 accumulates, 2 writes HBM
            if (C == 0) {
              yp[(e * H + i) * YSC] = h2 * z;
            } else if (C == 1) {
              yp[(e * H + i) * YSC] += h2 * z;
            } else {
              if (FULL || (inside && gc0 + ee * H + i < G.nlim[2])) {
                const T vp = yp[(e * H + i) * YSC] + h2 * z;
                Y.c[3][pbase + (ee * H + i) * pplane] = RESID ? bpre[ee * RPG + i - A0] - vp : vp;
              }
            }
          }
        }
      };
      if constexpr (RG == 1) {
        rows(std::integral_constant<int, 0>());
      } else {
        switch (grp) {
          case 0: rows(std::integral_constant<int, 0>()); break;
          case 1: rows(std::integral_constant<int, (RG > 1 ? 1 : 0)>()); break;
          case 2: if constexpr (RG > 2) rows(std::integral_constant<int, (RG > 2 ? 2 : 0)>()); break;
          case 3: if constexpr (RG > 3) rows(std::integral_constant<int, (RG > 3 ? 3 : 0)>()); break;
          case 4: if constexpr (RG > 4) rows(std::integral_constant<int, (RG > 4 ? 4 : 0)>()); break;
          case 5: if constexpr (RG > 5) rows(std::integral_constant<int, (RG > 5 ? 5 : 0)>()); break;
          case 6: if constexpr (RG > 6) rows(std::integral_constant<int, (RG > 6 ? 6 : 0)>()); break;
          default: if constexpr (RG > 7) rows(std::integral_constant<int, (RG > 7 ? 7 : 0)>()); break;
        }
      }
      // the constrained plane g_c = n belongs to the brick holding the last cell along c
      if (DOV && !FULL && grp == 0 && (C != 0 || !kStageUx) && e0 + S3 == NCc && inside &&
          G.c0[C] + NCc >= G.mlim[C] && G.mlim[C] == m) {
        g[C] = n;
        yc[g[0] * st[0] + g[1] * st[1] + g[2] * st[2]] = T(0);
      }
    };
    if constexpr (SPLIT) {
      if (tid < ITEMS) item(tid, std::integral_constant<int, 1>());
      else if (tid >= PT0)
        for (int it = tid - PT0; it < ITEMS; it += NT - PT0) item(it, std::integral_constant<int, 2>());
    } else {
      for (int it = tid; it < ITEMS * RG; it += NT) item(it, std::integral_constant<int, 0>());
    }
    };
    // (not for fp64 k = 7: the second copy of its long, row-grouped pass-3 body measured slower)
    constexpr bool kFullSpec = K != 7 || sizeof(T) == 4;
    if (kFullSpec && G.g0[O1] + No1 <= G.nlim[O1] && G.g0[O2] + No2 <= G.nlim[O2] && G.g0[C] > 0 &&
        G.g0[C] + Nc <= G.nlim[C] && G.c0[C] + NCc < G.mlim[C])
      pass3(bool_c<true>());
    else
      pass3(bool_c<false>());
    if (C == 0 && kStageUx) {
      __syncthreads();
      // coalesced write-out of the u_x rows (x = c fastest), plus the constrained plane x = n
      const bool last = G.c0[0] + NCc >= m;
      constexpr int NW = (Nc + 1) * No1 * No2;
      for (int i = tid; i < NW; i += NT) {
        const int lx = i % (Nc + 1), r = i / (Nc + 1);
        const int ly = r % No1, lz = r / No1;
        const int gx = G.g0[0] + lx, gy = G.g0[1] + ly, gz = G.g0[2] + lz;
        if (gy >= G.nlim[1] || gz >= G.nlim[2] || gx > n) continue;
        if (lx == Nc && !(last && gx == n)) continue;
        const int64_t gi = (static_cast<int64_t>(gz) * n + gy) * (n + 1) + gx;
        T rr;
        if (gx == 0 || gx == n) rr = T(0);
        else {
          rr = sYC[(lz * No1 + ly) * NCP + lx];
          if (RESID) rr = bc[gi] - rr;
        }
        yc[gi] = rr;
      }
    }
  }
  if constexpr (!(BR::QDB && TMA)) {  // (QDB: last_warp_done in the caller)
    fence_proxy_async();  // generic reads of this U buffer happen-before the next TMA into it
    __syncthreads();
  }
}

// QDB release of a component's U buffer: every warp arrives once its pass-3 reads are done; true in
// lane 0 of the last warp to arrive, which then issues the next staging into the buffer. The other
// warps go straight on to the next component (its U box was issued one component earlier).
template <int NT>
__device__ __forceinline__ bool last_warp_done(unsigned* cnt) {
  __syncwarp();
  bool last = false;
  if ((threadIdx.x & 31) == 0) {
    // no fence.proxy.async: a write-after-read release, ordered like a CUTLASS consumer release (the
    // reads have completed before __syncwarp; the issuer acquires the count before the TMA). Measured:
    // C2 fp64 0.2653 -> 0.2621 ms without the proxy fence (profiles/r02/ab_vmult_release_no_proxy_fence.jsonl)
    __threadfence_block();
    last = atomicInc(cnt, NT / 32 - 1) == NT / 32 - 1;  // wraps to 0 for the next release
    if (last) __threadfence_block();
  }
  return last;
}

__device__ __forceinline__ void brick_geo(Geo& G, int brick, int lnbx, int lnby, int bx, int by, int bz, int H,
                                          int zc0) {
  // bricks per x / y row are powers of two (m and the brick sizes are): shifts, no integer division
  const int ix = brick & ((1 << lnbx) - 1), iy = (brick >> lnbx) & ((1 << lnby) - 1), iz = brick >> (lnbx + lnby);
  G.c0[0] = ix * bx;
  G.c0[1] = iy * by;
  G.c0[2] = zc0 + iz * bz;
  for (int a = 0; a < 3; ++a) G.g0[a] = G.c0[a] * H;
}

// Persistent kernel: each CTA walks bricks blockIdx.x, blockIdx.x + gridDim.x, ... The three
// component boxes of a brick alternate between two U buffers (each with its own mbarrier) so that
// the TMA staging of the next component -- and of the next brick's first component and pressure
// box -- overlaps compute.
template <typename T, int K, int BX, int BY, int BZ, int OCC, int NT, bool RESID, bool TMA>
__global__ void __launch_bounds__(NT, OCC) stokes_vmult_kernel(const Blocks<const T> X, const Blocks<T> Y,
                                                             const Blocks<const T> B, int m, int zc0, int zc1, int zlo,
                                                             int zhi,
                                                             T h,
                                                             const Maps* __restrict__ mapsp) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  constexpr int H = K + 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (BR::BYTES - 3 * 8));  // [buf0, buf1, P]
  // bricks cover the cells [0, m)^2 x [zc0, zc1) (the whole level, or the cells a z-slab owns)
  const int nbx = (m + BX - 1) / BX, nby = (m + BY - 1) / BY, nbz = (zc1 - zc0 + BZ - 1) / BZ;
  const int lnbx = 31 - __clz(nbx), lnby = 31 - __clz(nby);
  const int nbricks = nbx * nby * nbz;
  Geo G, Gn;
  G.m = Gn.m = m;
  G.n = Gn.n = m * H;
  G.nlim[0] = G.nlim[1] = G.n;
  G.nlim[2] = zc1 * H;
  G.mlim[0] = G.mlim[1] = m;
  G.mlim[2] = zc1;
  G.zoff = Gn.zoff = zlo * H;
  G.zend = Gn.zend = zhi * H;
  for (int a = 0; a < 3; ++a) {
    Gn.nlim[a] = G.nlim[a];
    Gn.mlim[a] = G.mlim[a];
  }
  T* sP = sm + BR::OFF_P;
  const Maps& maps = *mapsp;  // tensor maps live in global memory (64-B aligned slots)
  int brick = blockIdx.x;
  if (brick >= nbricks) return;
  constexpr bool QB = BR::QDB && TMA;  // barrier-free pass-3 release (TMA staging only)
  __shared__ unsigned rel_cnt;          // QB: warps done with the current component's pass 3
  if (TMA && threadIdx.x == 0) {
    rel_cnt = 0;
    mbar_init(&bars[0], QB ? 1 : NT / 32);  // U buffers: the issuer (QB) or one arrival per warp (issue_u)
    mbar_init(&bars[1], QB ? 1 : NT / 32);
    mbar_init(&bars[2], 1);        // P box: thread 0
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_proxy_async();
  __syncthreads();
  brick_geo(G, brick, lnbx, lnby, BX, BY, BZ, H, zc0);
  issue_p<T, K, BX, BY, BZ, OCC, NT, TMA>(sP, &bars[2], X, maps, G);
  if constexpr (QB) {
    if (threadIdx.x == 0) issue_u<T, K, BX, BY, BZ, OCC, NT, 0, TMA, true>(sm, &bars[0], X, maps, G);
  } else {
    issue_u<T, K, BX, BY, BZ, OCC, NT, 0, TMA>(sm, &bars[0], X, maps, G);
  }
  if (!TMA) cp_async_commit();
  int u0 = 0;
  unsigned ph[2] = {0, 0}, phP = 0;  // mbarrier phase of buffer 0 / 1 / P
  if constexpr (!BR::DB) {
    // single U buffer, released early (component(): next staging issued after pass 1)
    for (; brick < nbricks; brick += gridDim.x) {
      const int next = brick + gridDim.x;
      const bool has_next = next < nbricks;
      if (has_next) brick_geo(Gn, next, lnbx, lnby, BX, BY, BZ, H, zc0);
      if (TMA) {
        mbar_wait(&bars[2], phP);
        phP ^= 1;
        if (fix_needed<T, K, BX, BY, BZ, OCC>(false, false, G)) {
          __syncthreads();
          fix_columns<T, K, BX, BY, BZ, OCC, NT>(nullptr, nullptr, nullptr, sP, G);
          __syncthreads();
        }
      } else {
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
      }
      component<T, K, BX, BY, BZ, OCC, NT, 0, RESID, TMA>(sm, sm, G, h, nullptr, X, Y, B, maps, &bars[2], &bars[0],
                                                          &ph[0], 1, &G);
      component<T, K, BX, BY, BZ, OCC, NT, 1, RESID, TMA>(sm, sm, G, h, nullptr, X, Y, B, maps, &bars[2], &bars[0],
                                                          &ph[0], 2, &G);
      component<T, K, BX, BY, BZ, OCC, NT, 2, RESID, TMA>(sm, sm, G, h, has_next ? &Gn : nullptr, X, Y, B, maps,
                                                          &bars[2], &bars[0], &ph[0], has_next ? 0 : -1, &Gn);
      G = Gn;  // (component() ends with a CTA barrier)
    }
    if (!TMA) cp_async_wait<0>();
  } else if constexpr (QB) {
    // two U buffers, two Q buffers, no CTA barrier after pass 3: the last warp done with a component's
    // pass 3 issues the staging that reuses its U buffer (component c + 2 in brick order)
    if (threadIdx.x == 0) issue_u<T, K, BX, BY, BZ, OCC, NT, 1, TMA, true>(sm + BR::OFF_U1, &bars[1], X, maps, G);
    int q = 0;
    for (; brick < nbricks; brick += gridDim.x) {
      const int ia = u0, ib = u0 ^ 1;
      T* bufA = sm + (ia ? BR::OFF_U1 : 0);  // components 0 and 2 of this brick, then 1 of the next
      T* bufB = sm + (ib ? BR::OFF_U1 : 0);  // component 1, then component 0 of the next brick
      const int next = brick + gridDim.x;
      const bool has_next = next < nbricks;
      if (has_next) brick_geo(Gn, next, lnbx, lnby, BX, BY, BZ, H, zc0);
      mbar_wait(&bars[2], phP);
      phP ^= 1;
      mbar_wait(&bars[ia], ph[ia]);
      ph[ia] ^= 1;
      if (fix_needed<T, K, BX, BY, BZ, OCC>(true, false, G)) {
        fix_columns<T, K, BX, BY, BZ, OCC, NT>(bufA, nullptr, nullptr, sP, G);
        __syncthreads();
      }
      component<T, K, BX, BY, BZ, OCC, NT, 0, RESID, TMA>(sm, bufA, G, h, nullptr, X, Y, B, maps, &bars[2], nullptr,
                                                          nullptr, -1, nullptr, q);
      q ^= 1;
      if (last_warp_done<NT>(&rel_cnt)) issue_u<T, K, BX, BY, BZ, OCC, NT, 2, TMA, true>(bufA, &bars[ia], X, maps, G);
      mbar_wait(&bars[ib], ph[ib]);
      ph[ib] ^= 1;
      if (fix_needed<T, K, BX, BY, BZ, OCC>(false, false, G)) {
        fix_columns<T, K, BX, BY, BZ, OCC, NT>(nullptr, bufB, nullptr, nullptr, G);
        __syncthreads();
      }
      component<T, K, BX, BY, BZ, OCC, NT, 1, RESID, TMA>(sm, bufB, G, h, nullptr, X, Y, B, maps, &bars[2], nullptr,
                                                          nullptr, -1, nullptr, q);
      q ^= 1;
      if (last_warp_done<NT>(&rel_cnt) && has_next)
        issue_u<T, K, BX, BY, BZ, OCC, NT, 0, TMA, true>(bufB, &bars[ib], X, maps, Gn);
      mbar_wait(&bars[ia], ph[ia]);
      ph[ia] ^= 1;
      if (fix_needed<T, K, BX, BY, BZ, OCC>(false, true, G)) {
        fix_columns<T, K, BX, BY, BZ, OCC, NT>(nullptr, nullptr, bufA, nullptr, G);
        __syncthreads();
      }
      component<T, K, BX, BY, BZ, OCC, NT, 2, RESID, TMA>(sm, bufA, G, h, has_next ? &Gn : nullptr, X, Y, B, maps,
                                                          &bars[2], nullptr, nullptr, -1, nullptr, q);
      q ^= 1;
      if (last_warp_done<NT>(&rel_cnt) && has_next)
        issue_u<T, K, BX, BY, BZ, OCC, NT, 1, TMA, true>(bufA, &bars[ia], X, maps, Gn);
      G = Gn;
      u0 ^= 1;
    }
  } else {
  for (; brick < nbricks; brick += gridDim.x) {
    const int ia = u0, ib = u0 ^ 1;
    T* bufA = sm + (ia ? BR::OFF_U1 : 0);  // components 0 and 2 of this brick
    T* bufB = sm + (ib ? BR::OFF_U1 : 0);  // component 1, then component 0 of the next brick
    const int next = brick + gridDim.x;
    const bool has_next = next < nbricks;
    if (has_next) brick_geo(Gn, next, lnbx, lnby, BX, BY, BZ, H, zc0);
    issue_u<T, K, BX, BY, BZ, OCC, NT, 1, TMA>(bufB, &bars[ib], X, maps, G);
    if (TMA) {
      mbar_wait(&bars[2], phP);
      phP ^= 1;
      mbar_wait(&bars[ia], ph[ia]);
      ph[ia] ^= 1;
    } else {
      cp_async_commit();
      cp_async_wait<1>();  // P box and U_0 of this brick
    }
    if (!TMA) __syncthreads();
    if (TMA && fix_needed<T, K, BX, BY, BZ, OCC>(true, false, G)) {
      fix_columns<T, K, BX, BY, BZ, OCC, NT>(bufA, nullptr, nullptr, sP, G);
      __syncthreads();
    }
    component<T, K, BX, BY, BZ, OCC, NT, 0, RESID, TMA>(sm, bufA, G, h, nullptr, X, Y, B, maps, &bars[2]);
    issue_u<T, K, BX, BY, BZ, OCC, NT, 2, TMA>(bufA, &bars[ia], X, maps, G);
    if (TMA) {
      mbar_wait(&bars[ib], ph[ib]);
      ph[ib] ^= 1;
    } else {
      cp_async_commit();
      cp_async_wait<1>();  // U_1
    }
    if (!TMA) __syncthreads();
    if (TMA && fix_needed<T, K, BX, BY, BZ, OCC>(false, false, G)) {
      fix_columns<T, K, BX, BY, BZ, OCC, NT>(nullptr, bufB, nullptr, nullptr, G);
      __syncthreads();
    }
    component<T, K, BX, BY, BZ, OCC, NT, 1, RESID, TMA>(sm, bufB, G, h, nullptr, X, Y, B, maps, &bars[2]);
    if (has_next) issue_u<T, K, BX, BY, BZ, OCC, NT, 0, TMA>(bufB, &bars[ib], X, maps, Gn);
    if (TMA) {
      mbar_wait(&bars[ia], ph[ia]);
      ph[ia] ^= 1;
    } else {
      cp_async_commit();
      cp_async_wait<1>();  // U_2
    }
    if (!TMA) __syncthreads();
    if (TMA && fix_needed<T, K, BX, BY, BZ, OCC>(false, true, G)) {
      fix_columns<T, K, BX, BY, BZ, OCC, NT>(nullptr, nullptr, bufA, nullptr, G);
      __syncthreads();
    }
    component<T, K, BX, BY, BZ, OCC, NT, 2, RESID, TMA>(sm, bufA, G, h, has_next ? &Gn : nullptr, X, Y, B, maps,
                                                   &bars[2]);
    G = Gn;  // (component() ends with a CTA barrier)
    u0 ^= 1;
  }
  if (!TMA) cp_async_wait<0>();
  }
}

// ---------------------------------------------------------------------------------------------
// host: tensor maps
// ---------------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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
void encode(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
            const uint32_t* box) {
  const uint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 rank, const_cast<void*>(base), dims, strides_bytes, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

// TMA needs 16-B aligned row pitches / base offsets (n * sizeof(T) % 16 == 0); boxes are kept no
// larger than the tensor (small coarse levels take the cp.async path).
template <typename T, int K, int BX, int BY, int BZ, int OCC>
bool tma_ok(int n, int nz) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  constexpr int H = K + 1;
  if ((static_cast<int64_t>(n) * sizeof(T)) % 16 != 0) return false;
  // boxes no larger than the maps: x / y extents against n - 1 (u_y drops two rows), z against the
  // held planes nz
  const int xy[] = {BR::UX(1), BR::UY(1), BR::UX(2), BR::UY(2), BR::PXT, BR::N(1) + H, BR::UX(0)};
  for (int e : xy)
    if (e > n - 1) return false;
  if (BR::UYS > n / BR::VEC) return false;
  const int zz[] = {BR::UZ(0), BR::UZ(1), BR::UZ(2), BR::N(2) + H};
  for (int e : zz)
    if (e > nz) return false;
  return true;
}

template <typename T, int K, int BX, int BY, int BZ, int OCC>
Maps make_maps(const LevelLayout& lay, const T* x) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  constexpr int H = K + 1;
  Maps M;
  std::memset(&M, 0, sizeof(M));
  const uint64_t es = sizeof(T);
  const uint64_t nn = static_cast<uint64_t>(lay.n);
  const uint64_t nz = static_cast<uint64_t>(lay.zhi - lay.zlo) * H;  // held z node planes
  // maps over the held part of each block (slab-local z = global z - zlo H; the kernel shifts)
  {  // u_x: the pitch n+1 is not a legal TMA stride, but the rows y = q (mod VEC) are: map q has base
     // q n (16-B aligned, n % VEC == 0), x' = x + q in [0, n+1+q), rows j = (y - q) / VEC, pitch VEC (n+1)
    constexpr int VEC = BR::VEC;
    for (int q = 0; q < VEC; ++q) {
      const uint64_t d[3] = {nn + 1 + q, nn / VEC, nz};
      const uint64_t s[2] = {VEC * (nn + 1) * es, nn * (nn + 1) * es};
      const uint32_t box[3] = {static_cast<uint32_t>(BR::UX(0)), static_cast<uint32_t>(BR::UYS),
                               static_cast<uint32_t>(BR::UZ(0))};
      encode<T>(&M.u0[q], x + lay.off[0] + q * nn, 3, d, s, box);
    }
  }
  {  // u_y: dims (x n, y n+1, z); base one row in -> y' = y - 1 in [0, n-1): the constrained rows are OOB
    const uint64_t d[3] = {nn, nn - 1, nz};
    const uint64_t s[2] = {nn * es, nn * (nn + 1) * es};
    const uint32_t box[3] = {static_cast<uint32_t>(BR::UX(1)), static_cast<uint32_t>(BR::UY(1)),
                             static_cast<uint32_t>(BR::UZ(1))};
    encode<T>(&M.u1, x + lay.off[1] + nn, 3, d, s, box);
  }
  {  // u_z: dims (x n, y n, z planes incl. the top one); constrained planes zeroed after landing
    const uint64_t d[3] = {nn, nn, nz + 1};
    const uint64_t s[2] = {nn * es, nn * nn * es};
    const uint32_t box[3] = {static_cast<uint32_t>(BR::UX(2)), static_cast<uint32_t>(BR::UY(2)),
                             static_cast<uint32_t>(BR::UZ(2))};
    encode<T>(&M.u2, x + lay.off[2], 3, d, s, box);
  }
  {  // p
    const uint64_t d[3] = {nn, nn, nz};
    const uint64_t s[2] = {nn * es, nn * nn * es};
    const uint32_t box[3] = {static_cast<uint32_t>(BR::PXT), static_cast<uint32_t>(BR::N(1) + H),
                             static_cast<uint32_t>(BR::N(2) + H)};
    encode<T>(&M.p, x + lay.off[3], 3, d, s, box);
  }
  return M;
}

// virtual global-index bases of the four blocks of a (slab) level vector
template <typename T>
Blocks<T> block_bases(const LevelLayout& lay, T* v) {
  Blocks<T> B;
  const int H = lay.k + 1;
  for (int c = 0; c < 4; ++c) B.c[c] = v ? v + lay.off[c] - static_cast<int64_t>(lay.zlo) * H * lay.plane[c] : nullptr;
  return B;
}

template <typename T, int K, int BX, int BY, int BZ, int OCC, int NT>
void launch_t(Context& ctx, int level, const VmultArgs& a) {
  using BR = Brick<T, K, BX, BY, BZ, OCC>;
  const int m = ctx.dev[0][level].lay.m, n = ctx.dev[0][level].lay.n;
  const LevelLayout lay = a.slab ? LevelLayout(K, level, a.zlo, a.zhi) : ctx.dev[0][level].lay;
  if (a.slab) {
    // the vector must hold one cell beyond each end of the computed range (inside the domain); staging
    // never reads planes outside the held range (bounds in the kernel, OOB fill of the slab-local maps),
    // and rows of a partial last brick beyond z1 are masked
    if (a.z0 < 0 || a.z1 > m || a.z0 >= a.z1 || a.zlo > std::max(a.z0 - 1, 0) || a.zhi < std::min(a.z1 + 1, m) ||
        a.zlo < 0 || a.zhi > m)
      throw std::invalid_argument("slab: the held cells must cover the computed cells plus one neighbour cell layer");
  }
  const Blocks<const T> X = block_bases(lay, static_cast<const T*>(a.x));
  const Blocks<T> Y = block_bases(lay, static_cast<T*>(a.y));
  const Blocks<const T> B = block_bases(lay, static_cast<const T*>(a.b));
  const T h = static_cast<T>(1.0 / m);
  const int nbricks = ((m + BX - 1) / BX) * ((m + BY - 1) / BY) * ((a.z1 - a.z0 + BZ - 1) / BZ);
  const dim3 grid(std::min(nbricks, OCC * ctx.num_sms));
  const size_t smem = BR::BYTES;
  static const bool no_tma = std::getenv("SMG_NO_TMA") != nullptr;  // diagnostics: force the cp.async path
  bool aligned = true;
  for (int c = 0; c < 4; ++c)
    aligned = aligned && (reinterpret_cast<uintptr_t>(a.x) + lay.off[c] * sizeof(T)) % 16 == 0;
  const bool tma = !no_tma && tma_ok<T, K, BX, BY, BZ, OCC>(n, (lay.zhi - lay.zlo) * (K + 1)) && aligned;
  const Maps* dmaps = nullptr;
  if (tma) {
    // tensor maps are cached per (input vector, slab, level, precision) in 64-B aligned global
    // slots, written stream-ordered before the launch
    const TmapKey key{a.x, level, static_cast<int>(sizeof(T)), a.zlo, a.zhi};
    auto it = ctx.tmap_slots.find(key);
    if (it == ctx.tmap_slots.end()) {
      const int slot = tmap_alloc_slot(ctx);
      Maps mh = make_maps<T, K, BX, BY, BZ, OCC>(lay, static_cast<const T*>(a.x));
      char* dst = static_cast<char*>(ctx.tmap_dev) + static_cast<size_t>(slot) * kTmapSlotBytes;
      SMG_CUDA(cudaMemcpyAsync(dst, &mh, sizeof(Maps), cudaMemcpyHostToDevice, ctx.stream));
      SMG_CUDA(cudaStreamSynchronize(ctx.stream));  // mh is a stack temporary
      it = ctx.tmap_slots.emplace(key, slot).first;
    }
    dmaps = reinterpret_cast<const Maps*>(static_cast<char*>(ctx.tmap_dev) +
                                          static_cast<size_t>(it->second) * kTmapSlotBytes);
    if (ctx.tmap_recording) ctx.tmap_recorded.insert(it->second);  // referenced by a graph being captured
  }
  static_assert(sizeof(Maps) <= kTmapSlotBytes, "tensor-map slot too small");
  auto go = [&](auto kern) {
    ensure_smem_attr(reinterpret_cast<const void*>(kern), ctx.device, smem);
    kern<<<grid, NT, smem, ctx.stream>>>(X, Y, B, m, a.z0, a.z1, a.zlo, a.zhi, h, dmaps);
  };
  if (a.b) {
    if (tma) go(stokes_vmult_kernel<T, K, BX, BY, BZ, OCC, NT, true, true>);
    else go(stokes_vmult_kernel<T, K, BX, BY, BZ, OCC, NT, true, false>);
  } else {
    if (tma) go(stokes_vmult_kernel<T, K, BX, BY, BZ, OCC, NT, false, true>);
    else go(stokes_vmult_kernel<T, K, BX, BY, BZ, OCC, NT, false, false>);
  }
  SMG_CUDA(cudaGetLastError());
  ++ctx.launches;
}

}  // namespace

// Brick shape (cells) per degree: fp64 SMEM ~80-200 KB, one persistent CTA per SM.
template <typename T, int K> struct BrickShape;
// NT: threads per CTA; OCC: resident CTAs per SM (persistent grid of OCC x #SMs, __launch_bounds__(NT, OCC))
template <typename T> struct BrickShape<T, 1> { static constexpr int X = 8, Y = 4, Z = 4, NT = 256, OCC = 2; };
// k=2: 4x4x4 cells, 384 threads, one CTA per SM (round 2: after the u_x tensor-map staging this shape
// beat the round-1 4x4x2 / 256 / 2-CTA default, 0.274 vs 0.295 ms at C2 fp64, tools/tune_k2.sh)
template <typename T> struct BrickShape<T, 2> { static constexpr int X = 4, Y = 4, Z = 4, NT = 384, OCC = 1; };
template <typename T> struct BrickShape<T, 3> { static constexpr int X = 4, Y = 2, Z = 2, NT = 256, OCC = 1; };
template <typename T> struct BrickShape<T, 4> { static constexpr int X = 2, Y = 2, Z = 2, NT = 384, OCC = 1; };
template <> struct BrickShape<double, 5> { static constexpr int X = 2, Y = 1, Z = 1, NT = 256, OCC = 1; };
template <> struct BrickShape<float, 5> { static constexpr int X = 2, Y = 2, Z = 1, NT = 256, OCC = 1; };
template <> struct BrickShape<double, 6> { static constexpr int X = 1, Y = 1, Z = 1, NT = 256, OCC = 1; };
template <> struct BrickShape<float, 6> { static constexpr int X = 2, Y = 1, Z = 1, NT = 256, OCC = 1; };
template <> struct BrickShape<double, 7> { static constexpr int X = 1, Y = 1, Z = 1, NT = 256, OCC = 1; };
template <> struct BrickShape<float, 7> { static constexpr int X = 2, Y = 1, Z = 1, NT = 256, OCC = 1; };

template <typename T, int K, class S>
void launch_shape(Context& ctx, int level, const VmultArgs& a) {
  static_assert(Brick<T, K, S::X, S::Y, S::Z, S::OCC>::BYTES <= (S::OCC == 1 ? 232448 : 233472 / S::OCC - 1024),
                "brick exceeds the shared memory of its occupancy");
  launch_t<T, K, S::X, S::Y, S::Z, S::OCC, S::NT>(ctx, level, a);
}

#ifdef SMG_TUNE
// tuning build only: alternative brick shapes selected by SMG_VMULT_VARIANT=1..N
template <int X_, int Y_, int Z_, int NT_, int OCC_>
struct Shape { static constexpr int X = X_, Y = Y_, Z = Z_, NT = NT_, OCC = OCC_; };
template <int K>
struct Variants {  // degrees without alternative shapes
  template <typename T>
  static bool run(int, Context&, int, const VmultArgs&) { return false; }
};
template <>
struct Variants<1> {
  template <typename T>
  static bool run(int v, Context& ctx, int level, const VmultArgs& a) {
    switch (v) {
      case 1: launch_shape<T, 1, Shape<8, 4, 2, 256, 2>>(ctx, level, a); return true;
      case 2: launch_shape<T, 1, Shape<4, 4, 4, 256, 2>>(ctx, level, a); return true;
      case 3: launch_shape<T, 1, Shape<8, 4, 4, 256, 2>>(ctx, level, a); return true;
      case 4: launch_shape<T, 1, Shape<8, 8, 2, 256, 2>>(ctx, level, a); return true;
      case 5: launch_shape<T, 1, Shape<8, 8, 4, 384, 1>>(ctx, level, a); return true;
      case 6: launch_shape<T, 1, Shape<8, 4, 4, 384, 1>>(ctx, level, a); return true;
      case 7: launch_shape<T, 1, Shape<8, 8, 4, 512, 1>>(ctx, level, a); return true;
      case 8: launch_shape<T, 1, Shape<8, 4, 8, 384, 1>>(ctx, level, a); return true;
      default: return false;
    }
  }
};
template <>
struct Variants<2> {
  template <typename T>
  static bool run(int v, Context& ctx, int level, const VmultArgs& a) {
    switch (v) {
      case 1: launch_shape<T, 2, Shape<4, 2, 2, 192, 3>>(ctx, level, a); return true;
      case 2: launch_shape<T, 2, Shape<4, 2, 2, 256, 3>>(ctx, level, a); return true;
      case 3: launch_shape<T, 2, Shape<4, 4, 1, 192, 3>>(ctx, level, a); return true;
      case 4: launch_shape<T, 2, Shape<4, 4, 4, 512, 1>>(ctx, level, a); return true;
      case 5: launch_shape<T, 2, Shape<8, 2, 1, 192, 3>>(ctx, level, a); return true;
      case 6: launch_shape<T, 2, Shape<4, 4, 2, 192, 2>>(ctx, level, a); return true;
      case 7: launch_shape<T, 2, Shape<8, 4, 2, 384, 1>>(ctx, level, a); return true;
      case 8: launch_shape<T, 2, Shape<4, 4, 4, 384, 1>>(ctx, level, a); return true;
      case 9: launch_shape<T, 2, Shape<4, 4, 2, 320, 2>>(ctx, level, a); return true;
      case 10: launch_shape<T, 2, Shape<4, 4, 4, 320, 1>>(ctx, level, a); return true;
      case 11: launch_shape<T, 2, Shape<4, 4, 4, 448, 1>>(ctx, level, a); return true;
      case 12: launch_shape<T, 2, Shape<4, 4, 4, 256, 1>>(ctx, level, a); return true;
      case 13: launch_shape<T, 2, Shape<4, 4, 4, 576, 1>>(ctx, level, a); return true;
      case 14: launch_shape<T, 2, Shape<4, 4, 2, 256, 2>>(ctx, level, a); return true;  // round-1 default
      default: return false;
    }
  }
};
template <>
struct Variants<3> {
  template <typename T>
  static bool run(int v, Context& ctx, int level, const VmultArgs& a) {
    switch (v) {
      case 1: launch_shape<T, 3, Shape<2, 2, 2, 256, 2>>(ctx, level, a); return true;
      case 2: launch_shape<T, 3, Shape<4, 2, 2, 256, 1>>(ctx, level, a); return true;
      case 3: launch_shape<T, 3, Shape<4, 2, 2, 384, 1>>(ctx, level, a); return true;
      case 4: launch_shape<T, 3, Shape<4, 2, 1, 256, 2>>(ctx, level, a); return true;
      case 5: launch_shape<T, 3, Shape<4, 4, 1, 384, 1>>(ctx, level, a); return true;
      case 6: launch_shape<T, 3, Shape<4, 4, 1, 256, 1>>(ctx, level, a); return true;
      case 7: launch_shape<T, 3, Shape<2, 2, 4, 384, 1>>(ctx, level, a); return true;
      case 8: launch_shape<T, 3, Shape<2, 4, 2, 384, 1>>(ctx, level, a); return true;
      default: return false;
    }
  }
};
template <>
struct Variants<4> {
  template <typename T>
  static bool run(int v, Context& ctx, int level, const VmultArgs& a) {
    switch (v) {
      case 1: launch_shape<T, 4, Shape<2, 2, 2, 256, 1>>(ctx, level, a); return true;
      case 2: launch_shape<T, 4, Shape<2, 2, 1, 256, 2>>(ctx, level, a); return true;
      case 3: launch_shape<T, 4, Shape<4, 2, 1, 256, 1>>(ctx, level, a); return true;
      case 4: launch_shape<T, 4, Shape<2, 2, 2, 512, 1>>(ctx, level, a); return true;
      case 5: launch_shape<T, 4, Shape<4, 2, 1, 384, 1>>(ctx, level, a); return true;
      case 6: launch_shape<T, 4, Shape<2, 2, 2, 320, 1>>(ctx, level, a); return true;
      default: return false;
    }
  }
};
#endif

template <int K>
void vmult_launch_k(Context& ctx, int level, int prec, const VmultArgs& a) {
#ifdef SMG_TUNE
  static const int variant = std::getenv("SMG_VMULT_VARIANT") ? std::atoi(std::getenv("SMG_VMULT_VARIANT")) : 0;
  if (variant > 0) {
    if (prec == SMG_F64 ? Variants<K>::template run<double>(variant, ctx, level, a)
                        : Variants<K>::template run<float>(variant, ctx, level, a))
      return;
  }
#endif
  if (prec == SMG_F64) launch_shape<double, K, BrickShape<double, K>>(ctx, level, a);
  else launch_shape<float, K, BrickShape<float, K>>(ctx, level, a);
}

template <int K>
void vmult_upload_k(const double* t, const float* f) {
  SMG_CUDA(cudaMemcpyToSymbol(c_ref_d, t, sizeof(double) * kRefTotal));
  SMG_CUDA(cudaMemcpyToSymbol(c_ref_f, f, sizeof(float) * kRefTotal));
}

#define SMG_INSTANTIATE_VMULT(K)                                                                  \
  template void vmult_launch_k<K>(Context&, int, int, const VmultArgs&);           \
  template void vmult_upload_k<K>(const double*, const float*);

}  // namespace smg
