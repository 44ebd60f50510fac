#pragma once
// K3: vertex-patch multiplicative Schwarz smoother, one colour per launch (smooth SPEC.md:400-408,
// Alg. 2), local solver = Schur complement + fast diagonalisation
// (schur_solve SPEC.md:356-364, Eq. 9):
//   S P = B A^-1 F - G,   S = B A^-1 B^T,   U = A^-1 (F - B^T P),
// with projected, pressure-mass-preconditioned CG on the patch pressure.
//
// B200 design: ONE WARP PER PATCH. All patch vectors live in the warp's slice of shared memory;
// every step is a warp-synchronous pencil contraction with compile-time shapes (no CTA barriers).
// Per component c and axis a, the fast-diagonalisation eigenvectors S_a are pre-multiplied with
// the divergence factor of that axis at setup (G_a = D S_par along c, G_a = M' S_orth otherwise),
// so B_c A_c^-1 B_c^T = (G (x) G (x) G) Lambda_c^-1 (G (x) G (x) G)^T costs 6 contractions instead of
// 12, and the final velocity is U_c = (S (x) S (x) S) Lambda_c^-1 [S^T F_c - G^T P] re-using the
// eigen-coefficients of F computed once. Same-colour patches write disjoint DoFs, so
// the scatter is race-free and order-independent. The residual r = b - A x is refreshed per colour by
// the vmult kernel in residual mode.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "smg_internal.cuh"
#include "smoother.cuh"

namespace smg {
namespace {

// Packed patch tables (pack_patch_tables; sizes in elements of T). Every matrix is stored twice, as
// rows of M and rows of M^T, each row padded to a multiple of 4 elements (R4), so that a contraction
// reads the coefficients of one output as 16-byte vectors (LDS.128) -- the coefficient broadcasts
// were the largest instruction class after FFMA (profiles/r01 ncu_smoother_v6).
constexpr int R4(int v) { return (v + 3) / 4 * 4; }
template <int K>
struct PD {
  static constexpr int NP = 2 * K + 1;  // parallel (C0 interior nodes of the 2-cell patch)
  static constexpr int NO = 2 * K + 2;  // orthogonal (DG) / pressure
  static constexpr int NV = NP * NO * NO;
  static constexpr int NPR = NO * NO * NO;
  static constexpr int BIG = NV > NPR ? NV : NPR;
  static constexpr int SQP = NP * R4(NP), SQO = NO * R4(NO);
  static constexpr int PAR_S = 0;                        // S_par rows          NP x R4(NP)
  static constexpr int PAR_ST = PAR_S + SQP;             // S_par^T rows        NP x R4(NP)
  static constexpr int PAR_L = PAR_ST + SQP;             // eigenvalues         R4(NP)
  static constexpr int ORTH_S = PAR_L + R4(NP);          // 4 x S_orth rows     NO x R4(NO)
  static constexpr int ORTH_ST = ORTH_S + 4 * SQO;       // 4 x S_orth^T rows
  static constexpr int ORTH_L = ORTH_ST + 4 * SQO;       // 4 x R4(NO)
  static constexpr int G_PAR = ORTH_L + 4 * R4(NO);      // (D S_par) rows      NO x R4(NP)
  static constexpr int G_PART = G_PAR + NO * R4(NP);     // (D S_par)^T rows    NP x R4(NO)
  static constexpr int G_ORTH = G_PART + NP * R4(NO);    // 4 x (M' S_orth) rows
  static constexpr int G_ORTHT = G_ORTH + 4 * SQO;       // 4 x transposed
  static constexpr int MPI = G_ORTHT + 4 * SQO;          // M'^-1 rows          NO x R4(NO)
  // fused halo residual (global-operator rows over the patch window, see PatchTables::win_*)
  static constexpr int NF = NP + 2, N4 = 2 * NO;         // C0 window nodes, DG window (4 cells)
  static constexpr int WLO = MPI + SQO;                  // 4 x SIPG window    NO x R4(N4)
  static constexpr int WMO4 = WLO + 4 * NO * R4(N4);     // DG mass window     NO x R4(N4)
  static constexpr int WMOO = WMO4 + NO * R4(N4);        // DG mass (own)      NO x R4(NO)
  static constexpr int WLP = WMOO + SQO;                 // 4 x C0 stiffness   NP x R4(NF)
  static constexpr int WMP = WLP + 4 * NP * R4(NF);      // 4 x C0 mass        NP x R4(NF)
  static constexpr int WD = WMP + 4 * NP * R4(NF);       // 4 x divergence     NO x R4(NF)
  static constexpr int WDT = WD + 4 * NO * R4(NF);       // D^T                NP x R4(NO)
  static constexpr int TAB = WDT + NP * R4(NO);
  // the unfused kernel stages only the tables up to the fused-residual windows
  static constexpr int TAB0 = WLO, TABP0 = (TAB0 + 3) / 4 * 4;
  static constexpr int tabp(bool fused) { return fused ? TABP : TABP0; }
  static constexpr int TABP = (TAB + 3) / 4 * 4;
  // CTA-shared reciprocal eigenvalue sums of interior patches; none for k >= 6 (the table would not fit
  // next to the one-patch workspace, those patches divide like the boundary ones)
  static constexpr int LINV = K >= 6 ? 0 : (3 * NV + 3) / 4 * 4;
  // per-patch workspace: Fh (3 NV) | r z d q x (5 NPR) | T1 T2 (2 BIG)
  static constexpr int WS = 3 * NV + 5 * NPR + 2 * BIG;
  // fused halo residual: the window gathers and contractions run in the CG region (free before the
  // solve), grown where needed, plus the pressure rows B u and the patch pressure (2 NPR)
  static constexpr int SX = NF * N4 * NO, SST = NF * NO * NO;
  static constexpr int RS = (5 * NPR + 2 * BIG) > (2 * SX + 2 * SST) ? (5 * NPR + 2 * BIG) : (2 * SX + 2 * SST);
  static constexpr int WSF = 3 * NV + RS + 2 * NPR;
  static_assert(SX + NV <= 5 * NPR && 2 * NPR <= SX, "fused residual scratch layout");
  static constexpr int dv(int c, int a) { return a == c ? NP : NO; }
};

template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int N = 4;
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int N = 2;
};

// out = (M applied along axis AX) in;  in dims (D0,D1,D2), out extent along AX = R.
// M(i,j) = A[i * R4(C) + j] (rows padded to 16 B). One pencil per lane; the coefficients of output i
// are read as 16-byte vectors (broadcast LDS.128).
template <typename T, int D0, int D1, int D2, int AX, int R, int GS, bool ACC = false>
__device__ __forceinline__ void warp_axis_fma(const T* __restrict__ in, const T* __restrict__ A, T* __restrict__ out,
                                              int lane, const T* __restrict__ scale = nullptr) {
  constexpr int DI[3] = {D0, D1, D2};
  constexpr int C = DI[AX];
  constexpr int DO0 = AX == 0 ? R : D0, DO1 = AX == 1 ? R : D1;
  constexpr int SI = AX == 0 ? 1 : (AX == 1 ? D0 : D0 * D1);
  constexpr int SO = AX == 0 ? 1 : (AX == 1 ? DO0 : DO0 * DO1);
  constexpr int QA = AX == 0 ? D1 : D0;  // the two other axes, in order
  constexpr int NPEN = D0 * D1 * D2 / C;
  using V = typename Vec16<T>::type;
  constexpr int NV = Vec16<T>::N, LD = R4(C), NVR = (C + NV - 1) / NV;
  auto bases = [&](int p, int& bi, int& bo) {
    const int u = p % QA, v = p / QA;
    if (AX == 0) {
      bi = (v * D1 + u) * D0;
      bo = (v * DO1 + u) * DO0;
    } else if (AX == 1) {
      bi = v * D0 * D1 + u;
      bo = v * DO0 * DO1 + u;
    } else {
      bi = v * D0 + u;
      bo = v * DO0 + u;
    }
  };
  auto load = [&](int bi, T (&x)[NVR * NV]) {
#pragma unroll
    for (int j = 0; j < NVR * NV; ++j) x[j] = j < C ? in[bi + j * SI] : T(0);
    if (scale) {  // elementwise input scaling folded into the load (the interior patches' Lambda^-1)
#pragma unroll
      for (int j = 0; j < C; ++j) x[j] *= scale[bi + j * SI];
    }
  };
  auto row = [&](int i, const T (&x)[NVR * NV]) {
    const V* Ai = reinterpret_cast<const V*>(A + i * LD);
    T s = T(0);
#pragma unroll
    for (int q = 0; q < NVR; ++q) {
      const V a = Ai[q];
      if constexpr (Vec16<T>::N == 4) {
        s += a.x * x[4 * q];
        if (4 * q + 1 < C) s += a.y * x[4 * q + 1];
        if (4 * q + 2 < C) s += a.z * x[4 * q + 2];
        if (4 * q + 3 < C) s += a.w * x[4 * q + 3];
      } else {
        s += a.x * x[2 * q];
        if (2 * q + 1 < C) s += a.y * x[2 * q + 1];
      }
    }
    return s;
  };
  // whole rounds: one pencil per lane, all R outputs
  constexpr int NFULL = NPEN / GS * GS, TAIL = NPEN - NFULL;
  constexpr int LPP = TAIL > 0 ? GS / TAIL : 0;          // lanes per tail pencil
  constexpr int OPL = LPP > 0 ? (R + LPP - 1) / LPP : 0;  // outputs per lane
  constexpr bool SPREAD = LPP >= 2;
  for (int p = lane; p < (SPREAD ? NFULL : NPEN); p += GS) {
    int bi, bo;
    bases(p, bi, bo);
    T x[NVR * NV];
    load(bi, x);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const T s = row(i, x);
      if (ACC) out[bo + i * SO] += s;
      else out[bo + i * SO] = s;
    }
  }
  // a partial last round (e.g. 36 pencils on 32 lanes: 4 pencils) is spread over (output, pencil) lanes
  // instead of leaving all but TAIL lanes idle for a whole pencil's work (same sums in the same order).
  // Output-major: the lanes of a quarter warp read at most two coefficient rows (LDS.128 broadcasts);
  // pencil-major lanes (6 rows per quarter warp) measured slower (C2 smoothing step 19.2 vs 18.4 ms)
  if constexpr (SPREAD) {
    const int i0 = lane / TAIL, pt = lane - i0 * TAIL;
    if (i0 < LPP && i0 < R) {
      int bi, bo;
      bases(NFULL + pt, bi, bo);
      T x[NVR * NV];
      load(bi, x);
#pragma unroll
      for (int m = 0; m < OPL; ++m) {
        const int i = i0 + m * LPP;
        if (m == 0 || i < R) {
          const T s = row(i, x);
          if (ACC) out[bo + i * SO] += s;
          else out[bo + i * SO] = s;
        }
      }
    }
  }
}

// ---- tensor-core contraction (fp32 data, warp per patch): 3xTF32 mma.sync m16n8k8 ----
// The same contraction as warp_axis_fma as a GEMM Out(pencils x R) = In(pencils x C) A^T: m16 tiles of
// pencils, n8 tiles of outputs, k8 steps of inputs. Each fp32 operand is split into tf32 hi + lo and
// the product taken as hi*hi + hi*lo + lo*hi (fp32 accumulate), which keeps fp32-level accuracy
// (the smoother parity bar is 1e-5 against the fp64 oracle). Replaces the coefficient broadcasts
// (39 % of the FFMA kernel's shared-memory wavefronts) by two coefficient loads per lane and k step.
// Measured (round 2): parity holds (fp32 smoother tests pass at 1e-5) but the C2 fp32 smoothing step
// takes 26.2 ms against 18.6 ms with warp_axis_fma -- the 6x6 blocks fill 56 % of an m16n8k8 tile,
// the split / fragment / predicate work costs more instructions than the FFMAs it replaces, and the
// three chained MMAs per tile add latency. Off by default; build with -DSMG_SMOOTHER_MMA=1 to A/B.
#ifndef SMG_SMOOTHER_MMA
#define SMG_SMOOTHER_MMA 0
#endif
__device__ __forceinline__ unsigned to_tf32(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void split_tf32(float x, unsigned& hi, unsigned& lo) {
  hi = to_tf32(x);
  lo = to_tf32(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <int D0, int D1, int D2, int AX, int R, bool ACC>
__device__ __forceinline__ void warp_axis_mma(const float* __restrict__ in, const float* __restrict__ A,
                                              float* __restrict__ out, int lane) {
  constexpr int DI[3] = {D0, D1, D2};
  constexpr int C = DI[AX];
  constexpr int DO0 = AX == 0 ? R : D0, DO1 = AX == 1 ? R : D1;
  constexpr int SI = AX == 0 ? 1 : (AX == 1 ? D0 : D0 * D1);
  constexpr int SO = AX == 0 ? 1 : (AX == 1 ? DO0 : DO0 * DO1);
  constexpr int QA = AX == 0 ? D1 : D0;
  constexpr int NPEN = D0 * D1 * D2 / C;
  constexpr int LD = R4(C);
  constexpr int MT = (NPEN + 15) / 16, NTL = (R + 7) / 8, KS = (C + 7) / 8;
  const int g = lane >> 2, t = lane & 3;
  // coefficient fragments: B[k][n] = A(n, k)
  unsigned bh[NTL][KS][2], bl[NTL][KS][2];
#pragma unroll
  for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = nt * 8 + g, k = ks * 8 + t + 4 * h;
        const float v = (n < R && k < C) ? A[n * LD + k] : 0.0f;
        split_tf32(v, bh[nt][ks][h], bl[nt][ks][h]);
      }
  auto pen = [&](int p, int& bi, int& bo) {
    const int uu = p % QA, vv = p / QA;
    if (AX == 0) {
      bi = (vv * D1 + uu) * D0;
      bo = (vv * DO1 + uu) * DO0;
    } else if (AX == 1) {
      bi = vv * D0 * D1 + uu;
      bo = vv * DO0 * DO1 + uu;
    } else {
      bi = vv * D0 + uu;
      bo = vv * DO0 + uu;
    }
  };
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int p0 = mt * 16 + g, p1 = p0 + 8;
    const bool a0 = p0 < NPEN, a1 = p1 < NPEN;
    int bi0 = 0, bo0 = 0, bi1 = 0, bo1 = 0;
    if (a0) pen(p0, bi0, bo0);
    if (a1) pen(p1, bi1, bo1);
    float acc[NTL][4];
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.0f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k0 = ks * 8 + t, k1 = k0 + 4;
      const float x[4] = {(a0 && k0 < C) ? in[bi0 + k0 * SI] : 0.0f, (a1 && k0 < C) ? in[bi1 + k0 * SI] : 0.0f,
                          (a0 && k1 < C) ? in[bi0 + k1 * SI] : 0.0f, (a1 && k1 < C) ? in[bi1 + k1 * SI] : 0.0f};
      unsigned ah[4], al[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) split_tf32(x[e], ah[e], al[e]);
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt) {
        mma_tf32(acc[nt], al, bh[nt][ks][0], bh[nt][ks][1]);
        mma_tf32(acc[nt], ah, bl[nt][ks][0], bl[nt][ks][1]);
        mma_tf32(acc[nt], ah, bh[nt][ks][0], bh[nt][ks][1]);
      }
    }
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int n = nt * 8 + 2 * t + (e & 1);
        const bool row1 = e >= 2;
        if (n < R && (row1 ? a1 : a0)) {
          float* o = out + (row1 ? bo1 : bo0) + n * SO;
          if (ACC) *o += acc[nt][e];
          else *o = acc[nt][e];
        }
      }
  }
}

template <typename T, int D0, int D1, int D2, int AX, int R, int GS, bool ACC = false>
__device__ __forceinline__ void warp_axis(const T* __restrict__ in, const T* __restrict__ A, T* __restrict__ out,
                                          int lane, const T* __restrict__ scale = nullptr) {
  constexpr int DI[3] = {D0, D1, D2};
  if constexpr (SMG_SMOOTHER_MMA && GS == 32 && std::is_same<T, float>::value && DI[AX] <= 16 && R <= 16) {
    (void)scale;  // (the MMA path is only built without the scaled callers)
    warp_axis_mma<D0, D1, D2, AX, R, ACC>(in, A, out, lane);
  } else {
    warp_axis_fma<T, D0, D1, D2, AX, R, GS, ACC>(in, A, out, lane, scale);
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// a patch is solved by a group of GS threads: one warp (GS = 32, many patches per CTA, warp-synchronous)
// or a whole CTA (GS > 32, coarse levels where there are too few patches to fill the GPU and the
// per-patch latency dominates)
template <int GS>
__device__ __forceinline__ void gsync() {
  if constexpr (GS == 32) __syncwarp();
  else __syncthreads();
}
template <int GS, typename T>
__device__ __forceinline__ T group_sum(T v) {
  v = warp_sum(v);
  if constexpr (GS == 32) {
    return v;
  } else {
    __shared__ T red[GS / 32];
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    T s = T(0);
#pragma unroll
    for (int w = 0; w < GS / 32; ++w) s += red[w];
    return s;
  }
}

template <typename T, int K, int GS>
struct Patch {
  using P = PD<K>;
  const T* tab;
  const T* linv;  // 3 x NV reciprocal eigenvalue sums of the interior variant (CTA-shared)
  bool interior;
  int var[3];
  int lane;

  // rows of S (TR = false) or of S^T (TR = true) along axis a of component c
  __device__ const T* S(int c, int a, bool tr) const {
    return a == c ? tab + (tr ? P::PAR_ST : P::PAR_S) : tab + (tr ? P::ORTH_ST : P::ORTH_S) + var[a] * P::SQO;
  }
  __device__ const T* L(int c, int a) const { return a == c ? tab + P::PAR_L : tab + P::ORTH_L + var[a] * R4(P::NO); }
  __device__ const T* G(int c, int a, bool tr) const {
    return a == c ? tab + (tr ? P::G_PART : P::G_PAR) : tab + (tr ? P::G_ORTHT : P::G_ORTH) + var[a] * P::SQO;
  }

  // eigen-space transforms of a velocity-shaped array of component C (S square per axis):
  // out = (S0 (x) S1 (x) S2)^T in (TR = true) or (S0 (x) S1 (x) S2) in; uses tmp; out != in.
  template <int C, bool TR>
  __device__ void s3(const T* in, T* out, T* tmp) const {
    constexpr int A0 = P::dv(C, 0), A1 = P::dv(C, 1), A2 = P::dv(C, 2);
    warp_axis<T, A0, A1, A2, 0, A0, GS>(in, S(C, 0, TR), out, lane);
    gsync<GS>();
    warp_axis<T, A0, A1, A2, 1, A1, GS>(out, S(C, 1, TR), tmp, lane);
    gsync<GS>();
    warp_axis<T, A0, A1, A2, 2, A2, GS>(tmp, S(C, 2, TR), out, lane);
    gsync<GS>();
  }
  // pressure (NO^3) -> eigen space of component C: out = (G0 (x) G1 (x) G2)^T in
  template <int C>
  __device__ void gt3(const T* in, T* out, T* tmp) const {
    constexpr int NO = P::NO;
    constexpr int A0 = P::dv(C, 0), A1 = P::dv(C, 1), A2 = P::dv(C, 2);
    warp_axis<T, NO, NO, NO, 0, A0, GS>(in, G(C, 0, true), out, lane);
    gsync<GS>();
    warp_axis<T, A0, NO, NO, 1, A1, GS>(out, G(C, 1, true), tmp, lane);
    gsync<GS>();
    warp_axis<T, A0, A1, NO, 2, A2, GS>(tmp, G(C, 2, true), out, lane);
    gsync<GS>();
  }
  // the first contraction of gt3 (axis 0), shared by components 1 and 2 (both orthogonal to x: same
  // matrix G_orth(var0)^T): out = (G0^T (x) I (x) I) in
  __device__ void gt3_axis0_orth(const T* in, T* out) const {
    constexpr int NO = P::NO;
    warp_axis<T, NO, NO, NO, 0, NO, GS>(in, G(1, 0, true), out, lane);
    gsync<GS>();
  }
  // the last two contractions of gt3 from the axis-0 result x0: out = (I (x) G1^T (x) G2^T) x0
  template <int C>
  __device__ void gt3_from_axis0(const T* x0, T* out, T* tmp) const {
    constexpr int NO = P::NO;
    constexpr int A0 = P::dv(C, 0), A1 = P::dv(C, 1), A2 = P::dv(C, 2);
    warp_axis<T, A0, NO, NO, 1, A1, GS>(x0, G(C, 1, true), tmp, lane);
    gsync<GS>();
    warp_axis<T, A0, A1, NO, 2, A2, GS>(tmp, G(C, 2, true), out, lane);
    gsync<GS>();
  }
  // eigen space of component C -> pressure: out = (G0 (x) G1 (x) G2) in
  // acc (=|+=) (G0 (x) G1 (x) G2) in; s1, s2 scratch
  // scale (optional): in is multiplied elementwise on load (Lambda_C^-1 of interior patches)
  template <int C, bool ACC>
  __device__ void g3acc(const T* in, T* acc, T* s1, T* s2, const T* scale = nullptr) const {
    constexpr int NO = P::NO;
    constexpr int A0 = P::dv(C, 0), A1 = P::dv(C, 1), A2 = P::dv(C, 2);
    warp_axis<T, A0, A1, A2, 0, NO, GS>(in, G(C, 0, false), s1, lane, scale);
    gsync<GS>();
    warp_axis<T, NO, A1, A2, 1, NO, GS>(s1, G(C, 1, false), s2, lane);
    gsync<GS>();
    warp_axis<T, NO, NO, A2, 2, NO, GS, ACC>(s2, G(C, 2, false), acc, lane);
    gsync<GS>();
  }
  template <int C>
  __device__ void g3(const T* in, T* out, T* tmp) const {
    constexpr int NO = P::NO;
    constexpr int A0 = P::dv(C, 0), A1 = P::dv(C, 1), A2 = P::dv(C, 2);
    warp_axis<T, A0, A1, A2, 0, NO, GS>(in, G(C, 0, false), out, lane);
    gsync<GS>();
    warp_axis<T, NO, A1, A2, 1, NO, GS>(out, G(C, 1, false), tmp, lane);
    gsync<GS>();
    warp_axis<T, NO, NO, A2, 2, NO, GS>(tmp, G(C, 2, false), out, lane);
    gsync<GS>();
  }
  // t *= Lambda_C^-1 (eigen space of component C). Interior patches (all end variants 0, the vast
  // majority) multiply by the reciprocal eigenvalue sums tabulated once per CTA (linv); patches at the
  // domain boundary divide (the division inside the CG loop was 11 % of the smoother's instructions)
  template <int C>
  __device__ void lam_inv(T* t) const {
    if (interior) {
      const T* li = linv + C * P::NV;
      for (int o = lane; o < P::NV; o += GS) t[o] *= li[o];
    } else {
      constexpr int A0 = P::dv(C, 0), A1 = P::dv(C, 1);
      const T* l0 = L(C, 0);
      const T* l1 = L(C, 1);
      const T* l2 = L(C, 2);
      for (int o = lane; o < P::NV; o += GS) {
        const int x = o % A0, y = (o / A0) % A1, z = o / (A0 * A1);
        t[o] = t[o] / (l0[x] + l1[y] + l2[z]);
      }
    }
    gsync<GS>();
  }
  __device__ void project(T* p) const {
    T s = T(0);
    for (int o = lane; o < P::NPR; o += GS) s += p[o];
    s = group_sum<GS>(s) / T(P::NPR);
    gsync<GS>();
    for (int o = lane; o < P::NPR; o += GS) p[o] -= s;
    gsync<GS>();
  }
  __device__ T dot(const T* a, const T* b) const {
    T s = T(0);
    for (int o = lane; o < P::NPR; o += GS) s += a[o] * b[o];
    return group_sum<GS>(s);
  }
};

// per-block base pointers of a level vector in the global index space (a z-slab vector passes bases
// shifted back by its first plane)
template <typename T>
struct SBlocks {
  T* c[4];
};

template <typename T, int K, int W, int MINB, int GS, bool FUSED>
__global__ void __launch_bounds__(GS * W, MINB) patch_smooth_kernel(const SBlocks<T> x, const SBlocks<const T> r,
                                                              const SBlocks<const T> xin,
                                                              const T* __restrict__ ptab, int m, int colour,
                                                              int vz_first, int cnt_z, int cg_max_iter, T cg_tol,
                                                              int cg_fixed, int cg_precond,
                                                              unsigned long long* __restrict__ stats) {
  using P = PD<K>;
  constexpr int H = K + 1, NO = P::NO;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tab = reinterpret_cast<T*>(smem_raw);
  constexpr int TABPF = P::tabp(FUSED);
  for (int i = threadIdx.x; i < (FUSED ? P::TAB : P::TAB0); i += blockDim.x) tab[i] = ptab[i];
  __syncthreads();
  if constexpr (P::LINV > 0) {  // reciprocal eigenvalue sums of interior patches (end variant 0 on every axis)
    T* li = tab + TABPF;
    for (int i = threadIdx.x; i < 3 * P::NV; i += blockDim.x) {
      const int c = i / P::NV, o = i % P::NV;
      const int A0 = P::dv(c, 0), A1 = P::dv(c, 1);
      const int xyz[3] = {o % A0, (o / A0) % A1, o / (A0 * A1)};
      T sum = T(0);
      for (int a = 0; a < 3; ++a) sum += a == c ? tab[P::PAR_L + xyz[a]] : tab[P::ORTH_L + xyz[a]];
      li[i] = T(1) / sum;
    }
    __syncthreads();
  }
  const int warp = threadIdx.x / GS, lane = threadIdx.x % GS;  // patch slot in the CTA, thread in its group
  // vertices of the colour: x / y over the whole level, z from vz_first (cnt_z planes, step 2)
  const int cnt[3] = {(colour & 1) ? m / 2 : m / 2 - 1, ((colour >> 1) & 1) ? m / 2 : m / 2 - 1, cnt_z};
  const int npatch = cnt[0] * cnt[1] * cnt[2];
  const int pid = blockIdx.x * W + warp;
  if (pid >= npatch) return;
  const int v[3] = {((colour & 1) ? 1 : 2) + 2 * (pid % cnt[0]), (((colour >> 1) & 1) ? 1 : 2) + 2 * ((pid / cnt[0]) % cnt[1]),
                    vz_first + 2 * (pid / (cnt[0] * cnt[1]))};
  T* ws = tab + TABPF + P::LINV + warp * (FUSED ? P::WSF : P::WS);
  T* Fh = ws;                // 3 x NV eigen coefficients of F_c
  T* Pr = Fh + 3 * P::NV;    // CG residual
  T* Pz = Pr + P::NPR;       // preconditioned residual
  T* Pd = Pz + P::NPR;       // search direction
  T* Pq = Pd + P::NPR;       // S d
  T* Px = Pq + P::NPR;       // pressure iterate
  T* T1 = Px + P::NPR;       // scratch (BIG)
  T* T2 = T1 + P::BIG;       // scratch (BIG)

  Patch<T, K, GS> ps;
  ps.tab = tab;
  ps.lane = lane;
  for (int a = 0; a < 3; ++a) ps.var[a] = 2 * (v[a] == 1) + (v[a] == m - 1);
  ps.linv = tab + TABPF;  // CTA-shared table filled above
  ps.interior = P::LINV > 0 && ps.var[0] == 0 && ps.var[1] == 0 && ps.var[2] == 0;
  const int n = m * H;

  // ---- gather R_j r: velocity blocks -> T1 -> eigen coefficients Fh_c; pressure -> Pq (= G) ----
  auto vel_index = [&](int c, int o) {
    const int d0 = P::dv(c, 0), d1 = P::dv(c, 1);
    const int xx = o % d0, yy = (o / d0) % d1, zz = o / (d0 * d1);
    int64_t gd0 = n, gd1 = n;
    if (c == 0) gd0 = n + 1;
    if (c == 1) gd1 = n + 1;
    const int b0 = (v[0] - 1) * H + (c == 0), b1 = (v[1] - 1) * H + (c == 1), b2 = (v[2] - 1) * H + (c == 2);
    return (static_cast<int64_t>(b2 + zz) * gd1 + b1 + yy) * gd0 + b0 + xx;
  };
  auto pres_index = [&](int o) {
    const int xx = o % NO, yy = (o / NO) % NO, zz = o / (NO * NO);
    return (static_cast<int64_t>((v[2] - 1) * H + zz) * n + (v[1] - 1) * H + yy) * n + (v[0] - 1) * H + xx;
  };
#define SMG_FOR_C(...) \
  { constexpr int C = 0; __VA_ARGS__ } { constexpr int C = 1; __VA_ARGS__ } { constexpr int C = 2; __VA_ARGS__ }
  if constexpr (FUSED) {
    // ---- fused halo residual: r = b - A x_in on the patch rows, from the patch window of
    // the snapshot x_in (cells v-2 .. v+1 across, the 2 patch cells along each component's own axis)
    // with the global operator's rows (PatchTables::win_*); x (the output buffer) holds a copy of x_in
    T* R = Pr;                     // contraction scratch (the CG region, free before the solve)
    T* PB = Fh + 3 * P::NV + P::RS;  // pressure rows B x_in
    T* PP = PB + P::NPR;           // patch pressure of x_in
    constexpr int NF = P::NF, N4 = P::N4, NP = P::NP;
    for (int o = lane; o < P::NPR; o += GS) PP[o] = xin.c[3][pres_index(o)];
    SMG_FOR_C({
      constexpr int O1 = C == 0 ? 1 : 0, O2 = C == 2 ? 1 : 2;
      // extents per axis: along C xc, along O1 x1, along O2 x2
      constexpr auto dm = [](int a, int xc, int x1, int x2) { return a == C ? xc : (a == O1 ? x1 : x2); };
      int64_t gd[3] = {n, n, n};
      gd[C] = n + 1;
      // gather a window: along C the C0 nodes (v_C - 1) H + i, i < NF (constrained nodes 0, n read as 0);
      // along O1 / O2 `wide` ? 4 cells from v - 2 : the 2 patch cells
      auto gather = [&](T* dst, bool wide1, bool wide2) {
        const int e0 = NF, e1 = wide1 ? N4 : NO, e2 = wide2 ? N4 : NO;
        const int ext[3] = {dm(0, e0, e1, e2), dm(1, e0, e1, e2), dm(2, e0, e1, e2)};
        int org[3];
        for (int a = 0; a < 3; ++a)
          org[a] = (v[a] - ((a == O1 && wide1) || (a == O2 && wide2) ? 2 : 1)) * H;
        for (int o = lane; o < ext[0] * ext[1] * ext[2]; o += GS) {
          const int g0 = org[0] + o % ext[0], g1 = org[1] + (o / ext[0]) % ext[1], g2 = org[2] + o / (ext[0] * ext[1]);
          const int gc = C == 0 ? g0 : (C == 1 ? g1 : g2);
          const bool ok = g0 >= 0 && g1 >= 0 && g2 >= 0 && g0 < gd[0] && g1 < gd[1] && g2 < gd[2] && gc != 0 && gc != n;
          dst[o] = ok ? xin.c[C][(static_cast<int64_t>(g2) * gd[1] + g1) * gd[0] + g0] : T(0);
        }
        gsync<GS>();
      };
      constexpr int SX = P::SX, SST = P::SST;
      T* X1 = R;
      T* A = R + SX;
      T* S = R + 2 * SX;
      T* Tt = S + SST;
      const T* wlo1 = tab + P::WLO + ps.var[O1] * NO * R4(N4);
      const T* wlo2 = tab + P::WLO + ps.var[O2] * NO * R4(N4);
      const T* wmo4 = tab + P::WMO4;
      const T* wmoo = tab + P::WMOO;
      // M_o2 (own) then M_o1 / L_o1 across: S = M_o1 M_o2 x, T = L_o1 M_o2 x
      gather(X1, true, false);
      warp_axis<T, dm(0, NF, N4, NO), dm(1, NF, N4, NO), dm(2, NF, N4, NO), O2, NO, GS>(X1, wmoo, A, lane);
      gsync<GS>();
      warp_axis<T, dm(0, NF, N4, NO), dm(1, NF, N4, NO), dm(2, NF, N4, NO), O1, NO, GS>(A, wmo4, S, lane);
      warp_axis<T, dm(0, NF, N4, NO), dm(1, NF, N4, NO), dm(2, NF, N4, NO), O1, NO, GS>(A, wlo1, Tt, lane);
      gsync<GS>();
      // T += M_o1 L_o2 x (L across o2 on the own o1 rows)
      T* X2 = R;
      T* Bo = R + SX;
      gather(X2, false, true);
      warp_axis<T, dm(0, NF, NO, N4), dm(1, NF, NO, N4), dm(2, NF, NO, N4), O2, NO, GS>(X2, wlo2, Bo, lane);
      gsync<GS>();
      warp_axis<T, dm(0, NF, NO, NO), dm(1, NF, NO, NO), dm(2, NF, NO, NO), O1, NO, GS, true>(Bo, wmoo, Tt, lane);
      gsync<GS>();
      // velocity rows y = L_c S + M_c T + D_c^T M M p (interior C0 nodes along c), pressure rows += D_c S
      T* Y = R + SX;
      const T* wlp = tab + P::WLP + ps.var[C] * NP * R4(NF);
      const T* wmp = tab + P::WMP + ps.var[C] * NP * R4(NF);
      const T* wd = tab + P::WD + ps.var[C] * NO * R4(NF);
      warp_axis<T, dm(0, NF, NO, NO), dm(1, NF, NO, NO), dm(2, NF, NO, NO), C, NP, GS>(S, wlp, Y, lane);
      gsync<GS>();
      warp_axis<T, dm(0, NF, NO, NO), dm(1, NF, NO, NO), dm(2, NF, NO, NO), C, NP, GS, true>(Tt, wmp, Y, lane);
      warp_axis<T, dm(0, NF, NO, NO), dm(1, NF, NO, NO), dm(2, NF, NO, NO), C, NO, GS, (C > 0)>(S, wd, PB, lane);
      gsync<GS>();
      T* Q1 = R;
      T* Q = R + P::NPR;
      warp_axis<T, NO, NO, NO, O1, NO, GS>(PP, wmoo, Q1, lane);
      gsync<GS>();
      warp_axis<T, NO, NO, NO, O2, NO, GS>(Q1, wmoo, Q, lane);
      gsync<GS>();
      warp_axis<T, NO, NO, NO, C, NP, GS, true>(Q, tab + P::WDT, Y, lane);
      gsync<GS>();
      for (int o = lane; o < P::NV; o += GS) T1[o] = r.c[C][vel_index(C, o)] - Y[o];
      gsync<GS>();
      ps.template s3<C, true>(T1, Fh + C * P::NV, T2);
    })
    for (int o = lane; o < P::NPR; o += GS) Pq[o] = r.c[3][pres_index(o)] - PB[o];
  } else {
    SMG_FOR_C({
      for (int o = lane; o < P::NV; o += GS) T1[o] = r.c[C][vel_index(C, o)];
      gsync<GS>();
      ps.template s3<C, true>(T1, Fh + C * P::NV, T2);
    })
    for (int o = lane; o < P::NPR; o += GS) Pq[o] = r.c[3][pres_index(o)];
  }
  // ---- rhs = sum_c G_c Lambda_c^-1 Fh_c - G  (projected) -> Pr ----
  for (int o = lane; o < P::NPR; o += GS) Pr[o] = -Pq[o];
  gsync<GS>();
  SMG_FOR_C({
    for (int o = lane; o < P::NV; o += GS) T1[o] = Fh[C * P::NV + o];
    gsync<GS>();
    ps.template lam_inv<C>(T1);
    ps.template g3<C>(T1, T2, Pq);  // result in T2 (Pq used as scratch)
    for (int o = lane; o < P::NPR; o += GS) Pr[o] += T2[o];
    gsync<GS>();
  })
  ps.project(Pr);
  auto precond = [&](const T* rr, T* zz) {
    if (cg_precond) {
      const T* Mi = tab + P::MPI;
      warp_axis<T, NO, NO, NO, 0, NO, GS>(rr, Mi, zz, lane);
      gsync<GS>();
      warp_axis<T, NO, NO, NO, 1, NO, GS>(zz, Mi, T1, lane);
      gsync<GS>();
      warp_axis<T, NO, NO, NO, 2, NO, GS>(T1, Mi, zz, lane);
      gsync<GS>();
    } else {
      for (int o = lane; o < P::NPR; o += GS) zz[o] = rr[o];
      gsync<GS>();
    }
    ps.project(zz);
  };
  precond(Pr, Pz);
  for (int o = lane; o < P::NPR; o += GS) {
    Pd[o] = Pz[o];
    Px[o] = T(0);
  }
  gsync<GS>();
  T rz = ps.dot(Pr, Pz);
  const T r0 = sqrt(ps.dot(Pr, Pr));
  int it = 0;
  for (; it < cg_max_iter; ++it) {
    if (!cg_fixed) {
      if (sqrt(ps.dot(Pr, Pr)) <= cg_tol * r0) break;
    }
    // Pq = S Pd = sum_c G_c Lambda_c^-1 G_c^T Pd

    // component 0, then 1 and 2 sharing their first contraction (x0 kept in Pz, which is free here:
    // it is recomputed by the preconditioner below)
    ps.template gt3<0>(Pd, T1, T2);
    // Lambda_C^-1: folded into the first contraction of g3acc for interior patches (its table is
    // CTA-shared), a separate pass (division) for boundary patches
    if (!ps.interior) ps.template lam_inv<0>(T1);
    ps.template g3acc<0, false>(T1, Pq, T2, T1, ps.interior ? ps.linv : nullptr);
    ps.gt3_axis0_orth(Pd, Pz);
    ps.template gt3_from_axis0<1>(Pz, T1, T2);
    if (!ps.interior) ps.template lam_inv<1>(T1);
    ps.template g3acc<1, true>(T1, Pq, T2, T1, ps.interior ? ps.linv + P::NV : nullptr);
    ps.template gt3_from_axis0<2>(Pz, T1, T2);
    if (!ps.interior) ps.template lam_inv<2>(T1);
    ps.template g3acc<2, true>(T1, Pq, T2, T1, ps.interior ? ps.linv + 2 * P::NV : nullptr);
    const T dq = ps.dot(Pd, Pq);
    if (!(dq > T(0)) || rz == T(0)) break;
    const T alpha = rz / dq;
    for (int o = lane; o < P::NPR; o += GS) {
      Px[o] += alpha * Pd[o];
      Pr[o] -= alpha * Pq[o];
    }
    gsync<GS>();
    ps.project(Pr);
    precond(Pr, Pz);
    const T rzn = ps.dot(Pr, Pz);
    const T beta = rzn / rz;
    rz = rzn;
    for (int o = lane; o < P::NPR; o += GS) Pd[o] = Pz[o] + beta * Pd[o];
    gsync<GS>();
  }
  ps.project(Px);
  if (lane == 0) {  // patches solved and inner CG iterations (smg_smoother_stats)
    atomicAdd(&stats[0], 1ull);
    atomicAdd(&stats[1], static_cast<unsigned long long>(it));
  }
  // ---- U_c = (S (x) S (x) S) Lambda_c^-1 [Fh_c - G_c^T P];  x += R^T (U, P) ----
  SMG_FOR_C({
    ps.template gt3<C>(Px, T1, T2);
    for (int o = lane; o < P::NV; o += GS) T1[o] = Fh[C * P::NV + o] - T1[o];
    gsync<GS>();
    ps.template lam_inv<C>(T1);
    ps.template s3<C, false>(T1, T2, Pz);
    for (int o = lane; o < P::NV; o += GS) x.c[C][vel_index(C, o)] += T2[o];
  })
#undef SMG_FOR_C
  for (int o = lane; o < P::NPR; o += GS) x.c[3][pres_index(o)] += Px[o];
}

// CTAs per SM that shared memory allows for W warp-patches per CTA (1 KB reserved per CTA)
template <typename T, int K, bool FUSED>
constexpr int ctas_per_sm(int w) {
  const int bytes =
      static_cast<int>(sizeof(T)) * (PD<K>::tabp(FUSED) + PD<K>::LINV + w * (FUSED ? PD<K>::WSF : PD<K>::WS)) + 1024;
  const int c = 233472 / bytes;
  return c > 3 ? 3 : c;
}
// warp-patches per CTA maximising the patches resident per SM (ties: fewer per CTA)
template <typename T, int K, bool FUSED>
constexpr int warps_per_cta() {
  int best = 1, best_p = 0;
  // at most 24 resident warp-patches (~85 registers per thread). 26 (13 per CTA, 2 CTAs, 78 registers)
  // measured: level-4 step of C2 2.80 vs 3.05 ms (one wave for 3600-3840 patches), level 5 18.35 vs
  // 18.11 ms, V-cycle unchanged -- not adopted
  for (int w = 1; w <= 8; ++w) {
    const int c = ctas_per_sm<T, K, FUSED>(w);
    const int p = w * c > 24 ? 0 : w * c;
    if (p > best_p) {
      best = w;
      best_p = p;
    }
  }
  return best;
}

template <typename T>
SBlocks<T> sblocks(const LevelLayout& lay, T* v) {
  SBlocks<T> B;
  const int H = lay.k + 1;
  for (int c = 0; c < 4; ++c) B.c[c] = v + lay.off[c] - static_cast<int64_t>(lay.zlo) * H * lay.plane[c];
  return B;
}

template <typename T, int K, int W, int GS, bool FUSED = false>
void launch_group(Context& ctx, const DevLevel& dl, const LevelLayout& lay, int npatch, int colour, int vz_first,
                  int cnt_z, void* x, const void* r, const void* xin = nullptr) {
  using P = PD<K>;
  constexpr int WSP = FUSED ? P::WSF : P::WS;
  const size_t smem = sizeof(T) * (P::tabp(FUSED) + P::LINV + W * WSP);
  // as many resident CTAs as shared memory allows (up to 3): registers are capped accordingly
  constexpr size_t smem_c = sizeof(T) * (P::tabp(FUSED) + P::LINV + W * WSP) + 1024;
  constexpr int MINB = smem_c * 3 <= 233472 ? 3 : (smem_c * 2 <= 233472 ? 2 : 1);
  static_assert(smem_c <= 233472, "patch workspace exceeds shared memory");
  auto kern = patch_smooth_kernel<T, K, W, MINB, GS, FUSED>;
  ensure_smem_attr(reinterpret_cast<const void*>(kern), ctx.device, smem);
  kern<<<(npatch + W - 1) / W, GS * W, smem, ctx.stream>>>(
      sblocks(lay, static_cast<T*>(x)), sblocks(lay, static_cast<const T*>(r)),
      sblocks(lay, static_cast<const T*>(xin ? xin : r)), static_cast<const T*>(dl.patch),
      dl.lay.m, colour, vz_first, cnt_z, ctx.cfg.cg_max_iter, static_cast<T>(ctx.cfg.cg_tol), ctx.cfg.cg_fixed,
      ctx.cfg.cg_precond, static_cast<unsigned long long*>(ctx.smoother_stats));
  SMG_CUDA(cudaGetLastError());
  ++ctx.launches;
}

// patches of one colour with vertex z planes in [vz0, vz1] (clipped to 1..m-1), on vectors holding the
// cells [zlo, zhi) of the level
template <typename T, int K>
void launch_k(Context& ctx, int level, int colour, void* x, const void* r, int zlo, int zhi, int vz0, int vz1) {
  const DevLevel& dl = ctx.dev[sizeof(T) == 8 ? 0 : 1][level];
  const int m = dl.lay.m;
  const LevelLayout lay(K, level, zlo, zhi);
  auto cnt = [&](int bit) { return bit ? m / 2 : m / 2 - 1; };
  const int zbit = (colour >> 2) & 1;
  int vf = std::max(vz0, 1);
  if ((vf & 1) != zbit) ++vf;  // odd planes for bit 1, even for bit 0
  const int vl = std::min(vz1, m - 1);
  const int cnt_z = vl >= vf ? (vl - vf) / 2 + 1 : 0;
  if (cnt_z > 0 && (vf - 1 < zlo || vl + 1 > zhi))
    throw std::invalid_argument("smooth: patches need the cells on both sides of their vertex plane");
  const int npatch = cnt(colour & 1) * cnt((colour >> 1) & 1) * cnt_z;
  if (npatch <= 0) return;
  if constexpr (K >= 5) {
    // high degrees (k = 5..7): one 8-warp CTA per patch -- a patch's workspace
    // (fp32 k = 7: 161 KB) only fits one per SM; fp64 fits up to k = 5
    if constexpr (sizeof(T) == 8 && K >= 6)
      throw std::invalid_argument("the fp64 patch smoother supports k <= 5: run the V-cycle in fp32 "
                                  "(vcycle_precision = SMG_F32) for k = 6, 7");
    else
      launch_group<T, K, 1, 256>(ctx, dl, lay, npatch, colour, vf, cnt_z, x, r);
  } else {
    // few patches (coarse levels): a 4- or 8-warp CTA per patch cuts the per-patch latency; many
    // patches: one warp per patch, several per CTA
    if (npatch <= 148) launch_group<T, K, 1, 256>(ctx, dl, lay, npatch, colour, vf, cnt_z, x, r);
    else if (npatch < 148 * 8) launch_group<T, K, 1, 128>(ctx, dl, lay, npatch, colour, vf, cnt_z, x, r);
    else launch_group<T, K, warps_per_cta<T, K, false>(), 32>(ctx, dl, lay, npatch, colour, vf, cnt_z, x, r);
  }
}

// fused halo-residual variant (k <= 3, whole level): x_out (a copy of x_in) += the patch corrections
// computed from r = b - A x_in on the patch rows
template <typename T, int K>
void launch_fused_k(Context& ctx, int level, int colour, void* x_out, const void* x_in, const void* b) {
  if constexpr (K > 3) {
    throw std::invalid_argument("the fused halo-residual smoother supports k <= 3");
  } else {
    const DevLevel& dl = ctx.dev[sizeof(T) == 8 ? 0 : 1][level];
    const int m = dl.lay.m;
    const LevelLayout lay(K, level);
    auto cnt = [&](int bit) { return bit ? m / 2 : m / 2 - 1; };
    const int zbit = (colour >> 2) & 1;
    const int vf = zbit ? 1 : 2, cnt_z = cnt(zbit);
    const int npatch = cnt(colour & 1) * cnt((colour >> 1) & 1) * cnt_z;
    if (npatch <= 0) return;
    if (npatch <= 148) launch_group<T, K, 1, 256, true>(ctx, dl, lay, npatch, colour, vf, cnt_z, x_out, b, x_in);
    else if (npatch < 148 * 8) launch_group<T, K, 1, 128, true>(ctx, dl, lay, npatch, colour, vf, cnt_z, x_out, b, x_in);
    else
      launch_group<T, K, warps_per_cta<T, K, true>(), 32, true>(ctx, dl, lay, npatch, colour, vf, cnt_z, x_out, b,
                                                                x_in);
  }
}

}  // namespace

template <int K>
void smooth_launch_k(Context& ctx, int level, int prec, int colour, void* x, const void* r, int zlo, int zhi, int vz0,
                     int vz1) {
  if (prec == SMG_F64) launch_k<double, K>(ctx, level, colour, x, r, zlo, zhi, vz0, vz1);
  else launch_k<float, K>(ctx, level, colour, x, r, zlo, zhi, vz0, vz1);
}

template <int K>
void smooth_fused_launch_k(Context& ctx, int level, int prec, int colour, void* x_out, const void* x_in,
                           const void* b) {
  if (prec == SMG_F64) launch_fused_k<double, K>(ctx, level, colour, x_out, x_in, b);
  else launch_fused_k<float, K>(ctx, level, colour, x_out, x_in, b);
}

#define SMG_INSTANTIATE_SMOOTH(K)                                                                      \
  template void smooth_launch_k<K>(Context&, int, int, int, void*, const void*, int, int, int, int); \
  template void smooth_fused_launch_k<K>(Context&, int, int, int, void*, const void*, const void*);

}  // namespace smg
