// Host setup of the 1D tables (see setup1d.hpp). fp64, microseconds per level.
#include "setup1d.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace smg {
namespace {

// Gauss-Legendre rule on [0,1] (quadrature.hpp:38-62 semantics), Newton on P_n from the
// cos(pi (i - 1/4)/(n + 1/2)) guesses.
void gauss_rule(int n, std::vector<double>& x, std::vector<double>& w) {
  x.resize(n);
  w.resize(n);
  for (int i = 1; i <= n; ++i) {
    double t = std::cos(M_PI * (i - 0.25) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = t;
      for (int j = 2; j <= n; ++j) {
        const double p2 = ((2 * j - 1) * t * p1 - (j - 1) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) p0 = 1.0;
      dp = n * (t * p1 - p0) / (t * t - 1.0);
      const double dt = p1 / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    x[n - i] = 0.5 * (1.0 + t);
    w[n - i] = 1.0 / ((1.0 - t * t) * dp * dp);
  }
}

// Gauss-Lobatto nodes of a degree-p nodal basis on [0,1] (basis.hpp:23-27, quadrature.hpp:65-86);
// degree 0 uses the midpoint. Interior nodes: roots of P'_p by Newton with P'' from Legendre's ODE.
std::vector<double> gl_nodes(int p) {
  if (p == 0) return {0.5};
  std::vector<double> z(p + 1);
  z[0] = 0.0;
  z[p] = 1.0;
  for (int i = 1; i < p; ++i) {
    double t = -std::cos(M_PI * i / p);
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = t;
      for (int j = 2; j <= p; ++j) {
        const double p2 = ((2 * j - 1) * t * p1 - (j - 1) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      const double d1 = p * (t * p1 - p0) / (t * t - 1.0);
      const double d2 = (2.0 * t * d1 - p * (p + 1.0) * p1) / (1.0 - t * t);
      const double dt = d1 / d2;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    z[i] = 0.5 * (1.0 + t);
  }
  return z;
}

// nodal Lagrange value / derivative via the barycentric-free product rule
double lag(const std::vector<double>& z, int i, double x) {
  double v = 1.0;
  for (size_t j = 0; j < z.size(); ++j)
    if (static_cast<int>(j) != i) v *= (x - z[j]) / (z[i] - z[j]);
  return v;
}
double dlag(const std::vector<double>& z, int i, double x) {
  double s = 0.0;
  for (size_t l = 0; l < z.size(); ++l) {
    if (static_cast<int>(l) == i) continue;
    double v = 1.0 / (z[i] - z[l]);
    for (size_t j = 0; j < z.size(); ++j)
      if (static_cast<int>(j) != i && j != l) v *= (x - z[j]) / (z[i] - z[j]);
    s += v;
  }
  return s;
}

struct CellMats {
  Dense Mo, Ko;  // DG degree k: mass (h), stiffness (1/h)
  Dense Mp, Kp;  // C0 degree k+1 cell matrices
  Dense Dc;      // (k+1) x (k+2): int psi_a phi_b'
  std::vector<double> v0, v1, d0, d1;  // DG degree-k traces and physical derivatives at 0, 1
};

CellMats cell_mats(int k, double h) {
  CellMats C;
  const auto zo = gl_nodes(k), zp = gl_nodes(k + 1);
  std::vector<double> qx, qw;
  gauss_rule(k + 3, qx, qw);  // exact for every product below (degree <= 2k+2)
  const int no = k + 1, np = k + 2;
  C.Mo = Dense(no, no); C.Ko = Dense(no, no); C.Mp = Dense(np, np); C.Kp = Dense(np, np); C.Dc = Dense(no, np);
  for (size_t q = 0; q < qx.size(); ++q) {
    const double x = qx[q], w = qw[q];
    for (int i = 0; i < no; ++i)
      for (int j = 0; j < no; ++j) {
        C.Mo(i, j) += w * h * lag(zo, i, x) * lag(zo, j, x);
        C.Ko(i, j) += w / h * dlag(zo, i, x) * dlag(zo, j, x);
      }
    for (int i = 0; i < np; ++i)
      for (int j = 0; j < np; ++j) {
        C.Mp(i, j) += w * h * lag(zp, i, x) * lag(zp, j, x);
        C.Kp(i, j) += w / h * dlag(zp, i, x) * dlag(zp, j, x);
      }
    for (int i = 0; i < no; ++i)
      for (int j = 0; j < np; ++j) C.Dc(i, j) += w * lag(zo, i, x) * dlag(zp, j, x);
  }
  C.v0.resize(no); C.v1.resize(no); C.d0.resize(no); C.d1.resize(no);
  for (int a = 0; a < no; ++a) {
    C.v0[a] = lag(zo, a, 0.0);
    C.v1[a] = lag(zo, a, 1.0);
    C.d0[a] = dlag(zo, a, 0.0) / h;
    C.d1[a] = dlag(zo, a, 1.0) / h;
  }
  return C;
}

// SIPG face blocks for the DG degree-k Laplacian (fem1d.hpp:130-174): face between L=e and R=e+1
// with jump = left - right, average derivative; Nitsche ends on the domain boundary.
struct FaceBlocks {
  Dense LL, LR, RL, RR, NitL, NitR;
};
FaceBlocks face_blocks(const CellMats& C, double g) {
  const int n = static_cast<int>(C.v0.size());
  FaceBlocks F;
  F.LL = Dense(n, n); F.LR = Dense(n, n); F.RL = Dense(n, n); F.RR = Dense(n, n);
  F.NitL = Dense(n, n); F.NitR = Dense(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      // test row i, trial column j
      F.LL(i, j) = g * C.v1[i] * C.v1[j] - 0.5 * (C.v1[i] * C.d1[j] + C.d1[i] * C.v1[j]);
      F.LR(i, j) = -g * C.v1[i] * C.v0[j] - 0.5 * C.v1[i] * C.d0[j] + 0.5 * C.d1[i] * C.v0[j];
      F.RL(i, j) = -g * C.v0[i] * C.v1[j] + 0.5 * C.v0[i] * C.d1[j] - 0.5 * C.d0[i] * C.v1[j];
      F.RR(i, j) = g * C.v0[i] * C.v0[j] + 0.5 * (C.v0[i] * C.d0[j] + C.d0[i] * C.v0[j]);
      F.NitL(i, j) = 2.0 * g * C.v0[i] * C.v0[j] + (C.v0[i] * C.d0[j] + C.d0[i] * C.v0[j]);
      F.NitR(i, j) = 2.0 * g * C.v1[i] * C.v1[j] - (C.v1[i] * C.d1[j] + C.d1[i] * C.v1[j]);
    }
  return F;
}

}  // namespace

LevelTables build_level_tables(int k, int level) {
  if (k < 1) throw std::invalid_argument("degree must be >= 1");
  if (level < 0) throw std::invalid_argument("level must be >= 0");
  LevelTables T;
  T.k = k;
  T.m = 2 << level;
  T.h = 1.0 / T.m;
  T.gamma = (k + 1) * (k + 2) / T.h;  // fem1d.hpp:267-269
  T.ops.assign(static_cast<size_t>(N_OPS) * T.op_stride(), 0.0);
  const CellMats C = cell_mats(k, T.h);
  const FaceBlocks F = face_blocks(C, T.gamma);
  const int no = k + 1, np = k + 2;
  for (int var = 0; var < 3; ++var) {
    const bool first = (var == 0), last = (var == 2);
    // DG mass: block diagonal
    for (int a = 0; a < no; ++a)
      for (int b = 0; b < no; ++b) T.w(OP_MO, var, 0, a, b) = C.Mo(a, b);
    // DG SIPG with Nitsche ends (sipg_laplace_1d weak_nitsche)
    for (int a = 0; a < no; ++a)
      for (int b = 0; b < no; ++b) {
        T.w(OP_LO, var, 0, a, b) = C.Ko(a, b) + (first ? F.NitL(a, b) : F.RR(a, b)) + (last ? F.NitR(a, b) : F.LL(a, b));
        if (!first) T.w(OP_LO, var, -1, a, b) = F.RL(a, b);
        if (!last) T.w(OP_LO, var, 1, a, b) = F.LR(a, b);
      }
    // C0 mass / stiffness: output node a of cell e is global node e(k+1)+a; the vertex row a=0
    // collects from cells e-1 (its local node k+1) and e. Global node 0 is constrained: zero row.
    for (int b = 0; b < np; ++b) {
      for (int a = 0; a < no; ++a) {
        if (a == 0 && first) continue;
        T.w(OP_MP, var, 0, a, b) = C.Mp(a, b);
        T.w(OP_LP, var, 0, a, b) = C.Kp(a, b);
      }
      if (!first) {
        T.w(OP_MP, var, -1, 0, b) = C.Mp(k + 1, b);
        T.w(OP_LP, var, -1, 0, b) = C.Kp(k + 1, b);
      }
    }
    // B_c factor: pressure rows of cell e from the C0 nodes of cell e
    for (int a = 0; a < no; ++a)
      for (int b = 0; b < np; ++b) T.w(OP_D, var, 0, a, b) = C.Dc(a, b);
    // B_c^T factor: C0 rows from the pressure nodes of the cells sharing the node
    for (int a = 0; a < no; ++a) {
      if (a == 0 && first) continue;
      for (int b = 0; b < no; ++b) T.w(OP_DT, var, 0, a, b) = C.Dc(b, a);
      if (a == 0)
        for (int b = 0; b < no; ++b) T.w(OP_DT, var, -1, 0, b) = C.Dc(b, k + 1);
    }
  }
  return T;
}

PatchTables build_patch_tables(const LevelTables& lt) {
  const int k = lt.k, no = k + 1, np = k + 2;
  PatchTables P;
  P.k = k;
  const CellMats C = cell_mats(k, lt.h);
  const FaceBlocks F = face_blocks(C, lt.gamma);
  // parallel axis: 2-cell C0 assembly restricted to the 2k+1 interior nodes (patch-boundary normal
  // DoFs excluded), i.e. the principal submatrix of the global C0 operator
  {
    const int nf = 2 * k + 3;
    Dense Lf(nf, nf), Mf(nf, nf);
    for (int e = 0; e < 2; ++e)
      for (int a = 0; a < np; ++a)
        for (int b = 0; b < np; ++b) {
          Lf(e * no + a, e * no + b) += C.Kp(a, b);
          Mf(e * no + a, e * no + b) += C.Mp(a, b);
        }
    P.par_L = Dense(nf - 2, nf - 2);
    P.par_M = Dense(nf - 2, nf - 2);
    for (int i = 0; i < nf - 2; ++i)
      for (int j = 0; j < nf - 2; ++j) {
        P.par_L(i, j) = Lf(i + 1, j + 1);
        P.par_M(i, j) = Mf(i + 1, j + 1);
      }
    gen_eig(P.par_L, P.par_M, P.par_S, P.par_lam);
    Dense Df(2 * no, nf);
    for (int e = 0; e < 2; ++e)
      for (int a = 0; a < no; ++a)
        for (int b = 0; b < np; ++b) Df(e * no + a, e * no + b) += C.Dc(a, b);
    P.D = Dense(2 * no, nf - 2);
    for (int i = 0; i < 2 * no; ++i)
      for (int j = 0; j < nf - 2; ++j) P.D(i, j) = Df(i, j + 1);
  }
  // orthogonal axes: principal 2-cell submatrix of the global SIPG operator. A patch end inside the
  // mesh keeps the neighbour face's own-side terms (interior_face), an end on the boundary keeps the
  // Nitsche terms (fem1d.hpp:17-30, 155-174).
  const int n2 = 2 * no;
  P.orth_M = Dense(n2, n2);
  for (int e = 0; e < 2; ++e)
    for (int a = 0; a < no; ++a)
      for (int b = 0; b < no; ++b) P.orth_M(e * no + a, e * no + b) = C.Mo(a, b);
  for (int v = 0; v < 4; ++v) {
    const bool lb = (v >> 1) & 1, rb = v & 1;
    Dense& L = P.orth_L[v];
    L = Dense(n2, n2);
    for (int a = 0; a < no; ++a)
      for (int b = 0; b < no; ++b) {
        L(a, b) = C.Ko(a, b) + (lb ? F.NitL(a, b) : F.RR(a, b)) + F.LL(a, b);
        L(no + a, no + b) = C.Ko(a, b) + F.RR(a, b) + (rb ? F.NitR(a, b) : F.LL(a, b));
        L(a, no + b) = F.LR(a, b);
        L(no + a, b) = F.RL(a, b);
      }
    gen_eig(L, P.orth_M, P.orth_S[v], P.orth_lam[v]);
  }
  P.Mp = P.orth_M;
  P.Mpinv = inverse(P.Mp);
  // global-operator rows at the patch DoFs over the patch window (fused halo residual)
  {
    const int nf = 2 * k + 3, n4 = 4 * no;
    P.win_MO4 = Dense(n2, n4);
    for (int e = 0; e < 2; ++e)
      for (int a = 0; a < no; ++a)
        for (int b = 0; b < no; ++b) P.win_MO4(e * no + a, (e + 1) * no + b) = C.Mo(a, b);
    Dense Lf(nf, nf), Mf(nf, nf), Df(n2, nf);
    for (int e = 0; e < 2; ++e) {
      for (int a = 0; a < np; ++a)
        for (int b = 0; b < np; ++b) {
          Lf(e * no + a, e * no + b) += C.Kp(a, b);
          Mf(e * no + a, e * no + b) += C.Mp(a, b);
        }
      for (int a = 0; a < no; ++a)
        for (int b = 0; b < np; ++b) Df(e * no + a, e * no + b) += C.Dc(a, b);
    }
    for (int v = 0; v < 4; ++v) {
      const bool lb = (v >> 1) & 1, rb = v & 1;
      Dense& W = P.win_LO[v];
      W = Dense(n2, n4);
      for (int a = 0; a < no; ++a)
        for (int b = 0; b < no; ++b) {
          // cell v-1 (window cell 1): left neighbour (window cell 0) exists unless lb
          if (!lb) W(a, b) = F.RL(a, b);
          W(a, no + b) = C.Ko(a, b) + (lb ? F.NitL(a, b) : F.RR(a, b)) + F.LL(a, b);
          W(a, 2 * no + b) = F.LR(a, b);
          // cell v (window cell 2): right neighbour (window cell 3) exists unless rb
          W(no + a, no + b) = F.RL(a, b);
          W(no + a, 2 * no + b) = C.Ko(a, b) + F.RR(a, b) + (rb ? F.NitR(a, b) : F.LL(a, b));
          if (!rb) W(no + a, 3 * no + b) = F.LR(a, b);
        }
      P.win_LP[v] = Dense(nf - 2, nf);
      P.win_MP[v] = Dense(nf - 2, nf);
      P.win_D[v] = Dense(n2, nf);
      for (int j = 0; j < nf; ++j) {
        const bool constrained = (j == 0 && lb) || (j == nf - 1 && rb);  // global node 0 / n
        if (constrained) continue;
        for (int i = 0; i < nf - 2; ++i) {
          P.win_LP[v](i, j) = Lf(i + 1, j);
          P.win_MP[v](i, j) = Mf(i + 1, j);
        }
        for (int i = 0; i < n2; ++i) P.win_D[v](i, j) = Df(i, j);
      }
    }
  }
  return P;
}

TransferTables build_transfer_tables(int k) {
  TransferTables T;
  T.k = k;
  const auto zc = gl_nodes(k + 1), zd = gl_nodes(k);
  T.Ec = Dense(2 * (k + 1) + 1, k + 2);
  for (int r = 0; r <= 2 * (k + 1); ++r) {
    const double x = r <= k + 1 ? 0.5 * zc[r] : 0.5 * (1.0 + zc[r - (k + 1)]);
    for (int j = 0; j < k + 2; ++j) T.Ec(r, j) = lag(zc, j, x);
  }
  T.Ed = Dense(2 * (k + 1), k + 1);
  for (int r = 0; r < 2 * (k + 1); ++r) {
    const double x = r <= k ? 0.5 * zd[r] : 0.5 * (1.0 + zd[r - (k + 1)]);
    for (int j = 0; j < k + 1; ++j) T.Ed(r, j) = lag(zd, j, x);
  }
  return T;
}

std::vector<double> reference_cell_tables() {
  std::vector<double> t(kRefTotal, 0.0);
  for (int k = 1; k <= kMaxK; ++k) {
    const int H = k + 1, P = k + 2;
    const CellMats C = cell_mats(k, 1.0);
    const FaceBlocks F = face_blocks(C, (k + 1) * (k + 2));
    double* o = t.data() + ref_base(k);
    auto put = [&](const Dense& A) {
      for (double v : A.a) *o++ = v;
    };
    Dense LO0(H, H), DLF(H, H), DLL(H, H);
    for (int a = 0; a < H; ++a)
      for (int b = 0; b < H; ++b) {
        LO0(a, b) = C.Ko(a, b) + F.RR(a, b) + F.LL(a, b);
        DLF(a, b) = F.NitL(a, b) - F.RR(a, b);
        DLL(a, b) = F.NitR(a, b) - F.LL(a, b);
      }
    put(C.Mo);
    put(LO0);
    put(F.RL);
    put(F.LR);
    put(DLF);
    put(DLL);
    put(C.Mp);
    put(C.Kp);
    put(C.Dc);
    (void)P;
  }
  return t;
}

std::vector<double> pressure_node_weights(int k) {
  const auto z = gl_nodes(k);
  std::vector<double> qx, qw, w(k + 1, 0.0);
  gauss_rule(k + 1, qx, qw);
  for (int a = 0; a <= k; ++a)
    for (size_t q = 0; q < qx.size(); ++q) w[a] += qw[q] * lag(z, a, qx[q]);
  return w;
}

void sym_eig(const Dense& A0, Dense& V, std::vector<double>& w) {
  const int n = A0.r;
  Dense A = A0;
  V = Dense(n, n);
  for (int i = 0; i < n; ++i) V(i, i) = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i == j ? diag : off) += A(i, j) * A(i, j);
    if (off <= 1e-32 * diag) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double tau = (A(q, q) - A(p, p)) / (2.0 * apq);
        const double t = std::copysign(1.0, tau) / (std::fabs(tau) + std::hypot(1.0, tau));
        const double c = 1.0 / std::hypot(1.0, t), s = t * c;
        for (int r = 0; r < n; ++r) {
          const double arp = A(r, p), arq = A(r, q);
          A(r, p) = c * arp - s * arq;
          A(r, q) = s * arp + c * arq;
        }
        for (int r = 0; r < n; ++r) {
          const double apr = A(p, r), aqr = A(q, r);
          A(p, r) = c * apr - s * aqr;
          A(q, r) = s * apr + c * aqr;
        }
        for (int r = 0; r < n; ++r) {
          const double vrp = V(r, p), vrq = V(r, q);
          V(r, p) = c * vrp - s * vrq;
          V(r, q) = s * vrp + c * vrq;
        }
      }
  }
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return A(a, a) < A(b, b); });
  Dense Vs(n, n);
  w.resize(n);
  for (int j = 0; j < n; ++j) {
    w[j] = A(idx[j], idx[j]);
    for (int i = 0; i < n; ++i) Vs(i, j) = V(i, idx[j]);
  }
  V = Vs;
}

void gen_eig(const Dense& L, const Dense& M, Dense& S, std::vector<double>& lam) {
  const int n = L.r;
  Dense Q;
  std::vector<double> mu;
  sym_eig(M, Q, mu);
  for (double v : mu)
    if (!(v > 0.0)) throw std::runtime_error("gen_eig: mass matrix not SPD");
  Dense Mih(n, n);  // M^{-1/2}
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int l = 0; l < n; ++l) s += Q(i, l) * Q(j, l) / std::sqrt(mu[l]);
      Mih(i, j) = s;
    }
  Dense T(n, n), C(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int l = 0; l < n; ++l) s += L(i, l) * Mih(l, j);
      T(i, j) = s;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int l = 0; l < n; ++l) s += Mih(i, l) * T(l, j);
      C(i, j) = s;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) C(i, j) = C(j, i) = 0.5 * (C(i, j) + C(j, i));
  Dense W;
  sym_eig(C, W, lam);
  S = Dense(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int l = 0; l < n; ++l) s += Mih(i, l) * W(l, j);
      S(i, j) = s;
    }
}

Dense inverse(const Dense& A) {
  const int n = A.r;
  Dense a = A, x(n, n);
  for (int i = 0; i < n; ++i) x(i, i) = 1.0;
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int i = c + 1; i < n; ++i)
      if (std::fabs(a(i, c)) > std::fabs(a(p, c))) p = i;
    if (a(p, c) == 0.0) throw std::runtime_error("inverse: singular matrix");
    for (int j = 0; j < n; ++j) {
      std::swap(a(c, j), a(p, j));
      std::swap(x(c, j), x(p, j));
    }
    const double d = 1.0 / a(c, c);
    for (int j = 0; j < n; ++j) {
      a(c, j) *= d;
      x(c, j) *= d;
    }
    for (int i = 0; i < n; ++i) {
      if (i == c || a(i, c) == 0.0) continue;
      const double f = a(i, c);
      for (int j = 0; j < n; ++j) {
        a(i, j) -= f * a(c, j);
        x(i, j) -= f * x(c, j);
      }
    }
  }
  return x;
}

}  // namespace smg
