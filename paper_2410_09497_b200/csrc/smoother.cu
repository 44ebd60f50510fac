// K3 dispatch (kernel in smoother_kernel.cuh, one TU per degree smoother_k<K>.cu) and the packed patch
// tables uploaded at context creation.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "smoother.cuh"

namespace smg {
namespace {

constexpr int R4(int v) { return (v + 3) / 4 * 4; }

void dispatch(Context& ctx, int level, int prec, int colour, void* x, const void* r, int zlo, int zhi, int vz0, int vz1) {
  switch (ctx.cfg.degree) {
    case 1: smooth_launch_k<1>(ctx, level, prec, colour, x, r, zlo, zhi, vz0, vz1); break;
    case 2: smooth_launch_k<2>(ctx, level, prec, colour, x, r, zlo, zhi, vz0, vz1); break;
    case 3: smooth_launch_k<3>(ctx, level, prec, colour, x, r, zlo, zhi, vz0, vz1); break;
    case 4: smooth_launch_k<4>(ctx, level, prec, colour, x, r, zlo, zhi, vz0, vz1); break;
    case 5: smooth_launch_k<5>(ctx, level, prec, colour, x, r, zlo, zhi, vz0, vz1); break;
    case 6: smooth_launch_k<6>(ctx, level, prec, colour, x, r, zlo, zhi, vz0, vz1); break;
    case 7: smooth_launch_k<7>(ctx, level, prec, colour, x, r, zlo, zhi, vz0, vz1); break;
    default: throw std::invalid_argument("degree not supported by the patch smoother kernel (1..7)");
  }
}

}  // namespace

void launch_smooth_colour(Context& ctx, int level, int prec, int colour, void* x, const void* r) {
  const int m = ctx.dev[0][level].lay.m;
  dispatch(ctx, level, prec, colour, x, r, 0, m, 1, m - 1);
}

void launch_smooth_colour_fused(Context& ctx, int level, int prec, int colour, void* x_out, const void* x_in,
                                const void* b) {
  switch (ctx.cfg.degree) {
    case 1: smooth_fused_launch_k<1>(ctx, level, prec, colour, x_out, x_in, b); break;
    case 2: smooth_fused_launch_k<2>(ctx, level, prec, colour, x_out, x_in, b); break;
    case 3: smooth_fused_launch_k<3>(ctx, level, prec, colour, x_out, x_in, b); break;
    default: throw std::invalid_argument("the fused halo-residual smoother supports k <= 3");
  }
}

void launch_smooth_colour_held(Context& ctx, int level, int prec, int colour, void* x, const void* r, int zlo,
                               int zhi, int vz0, int vz1) {
  dispatch(ctx, level, prec, colour, x, r, zlo, zhi, vz0, vz1);
}

// packed patch table (order of PD<K> offsets): every matrix as padded rows of M and of M^T
std::vector<double> pack_patch_tables(const PatchTables& P) {
  const int k = P.k, NP = 2 * k + 1, NO = 2 * k + 2;
  std::vector<double> t;
  auto rows = [&](int nr, int nc, auto f) {  // rows of an nr x nc matrix, padded to R4(nc)
    for (int i = 0; i < nr; ++i)
      for (int j = 0; j < R4(nc); ++j) t.push_back(j < nc ? f(i, j) : 0.0);
  };
  auto vec = [&](const std::vector<double>& v) {
    for (int j = 0; j < R4(static_cast<int>(v.size())); ++j) t.push_back(j < static_cast<int>(v.size()) ? v[j] : 0.0);
  };
  Dense Gp(NO, NP);  // D S_par
  for (int i = 0; i < NO; ++i)
    for (int j = 0; j < NP; ++j) {
      double s = 0.0;
      for (int l = 0; l < NP; ++l) s += P.D(i, l) * P.par_S(l, j);
      Gp(i, j) = s;
    }
  Dense Go[4];  // M' S_orth[v]
  for (int v = 0; v < 4; ++v) {
    Go[v] = Dense(NO, NO);
    for (int i = 0; i < NO; ++i)
      for (int j = 0; j < NO; ++j) {
        double s = 0.0;
        for (int l = 0; l < NO; ++l) s += P.Mp(i, l) * P.orth_S[v](l, j);
        Go[v](i, j) = s;
      }
  }
  rows(NP, NP, [&](int i, int j) { return P.par_S(i, j); });
  rows(NP, NP, [&](int i, int j) { return P.par_S(j, i); });
  vec(P.par_lam);
  for (int v = 0; v < 4; ++v) rows(NO, NO, [&](int i, int j) { return P.orth_S[v](i, j); });
  for (int v = 0; v < 4; ++v) rows(NO, NO, [&](int i, int j) { return P.orth_S[v](j, i); });
  for (int v = 0; v < 4; ++v) vec(P.orth_lam[v]);
  rows(NO, NP, [&](int i, int j) { return Gp(i, j); });
  rows(NP, NO, [&](int i, int j) { return Gp(j, i); });
  for (int v = 0; v < 4; ++v) rows(NO, NO, [&](int i, int j) { return Go[v](i, j); });
  for (int v = 0; v < 4; ++v) rows(NO, NO, [&](int i, int j) { return Go[v](j, i); });
  rows(NO, NO, [&](int i, int j) { return P.Mpinv(i, j); });
  // fused halo-residual windows (PD<K>::WLO ...): every matrix as padded rows
  const int NF = NP + 2, N4 = 2 * NO;
  for (int v = 0; v < 4; ++v) rows(NO, N4, [&](int i, int j) { return P.win_LO[v](i, j); });
  rows(NO, N4, [&](int i, int j) { return P.win_MO4(i, j); });
  rows(NO, NO, [&](int i, int j) { return P.Mp(i, j); });
  for (int v = 0; v < 4; ++v) rows(NP, NF, [&](int i, int j) { return P.win_LP[v](i, j); });
  for (int v = 0; v < 4; ++v) rows(NP, NF, [&](int i, int j) { return P.win_MP[v](i, j); });
  for (int v = 0; v < 4; ++v) rows(NO, NF, [&](int i, int j) { return P.win_D[v](i, j); });
  rows(NP, NO, [&](int i, int j) { return P.D(j, i); });  // D^T: C0 interior rows from DG pressure
  return t;
}

}  // namespace smg
