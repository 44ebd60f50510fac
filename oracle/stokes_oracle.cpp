// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see stokes_oracle.h for the contract).
//
// Restatement of the reference algorithm. Every function cites the reference file:line it follows
// (paths relative to /root/reference). Style is deliberately plain: correctness and independence
// from the product's Kronecker/CUDA formulation matter here, not speed, except that the operator and
// the smoother are OpenMP-parallel so the oracle doubles as the timed CPU baseline.
#include "stokes_oracle.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <tuple>
#include <vector>

namespace {

// ================================================================================================
// dense helpers
// ================================================================================================
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rr, int cc) : r(rr), c(cc), a(static_cast<size_t>(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
};

Mat transpose(const Mat& m) {
  Mat t(m.c, m.r);
  for (int i = 0; i < m.r; ++i)
    for (int j = 0; j < m.c; ++j) t(j, i) = m(i, j);
  return t;
}

int emit(const Mat& m, double* out, int cap, int* r, int* c) {
  *r = m.r;
  *c = m.c;
  if (m.r * m.c > cap) return -1;
  std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
  return 0;
}

// ================================================================================================
// L0: quadrature and nodal bases (quadrature.hpp:38-86, basis.hpp:16-54)
// ================================================================================================
// Legendre P_n(t) and P_n'(t) by the three-term recurrence (quadrature.hpp:22-33).
void legendre_pd(int n, double t, double& p, double& dp) {
  if (n == 0) { p = 1.0; dp = 0.0; return; }
  double pm1 = 1.0, pc = t;
  for (int j = 2; j <= n; ++j) {
    double pn = ((2.0 * j - 1.0) * t * pc - (j - 1.0) * pm1) / j;
    pm1 = pc;
    pc = pn;
  }
  p = pc;
  dp = n * (t * pc - pm1) / (t * t - 1.0);
}

struct Rule { std::vector<double> x, w; };

// n-point Gauss-Legendre on [0,1], ascending (quadrature.hpp:38-62: Newton from a Chebyshev guess).
Rule gauss(int n) {
  if (n < 1) throw std::invalid_argument("gauss: n < 1");
  Rule q;
  q.x.assign(n, 0.0);
  q.w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5)), p, dp = 0;
    for (int it = 0; it < 100; ++it) {
      legendre_pd(n, t, p, dp);
      double step = p / dp;
      t -= step;
      if (std::fabs(step) < 1e-15) { legendre_pd(n, t, p, dp); break; }
    }
    q.x[n - 1 - i] = 0.5 * (1.0 + t);
    q.w[n - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);
  }
  return q;
}

// Gauss-Lobatto points on [0,1] incl. endpoints: interior points are roots of P'_{n-1}
// (quadrature.hpp:65-86).
std::vector<double> lobatto(int npts) {
  if (npts < 2) throw std::invalid_argument("lobatto: npts < 2");
  const int n = npts - 1;
  std::vector<double> x(npts);
  x[0] = 0.0;
  x[n] = 1.0;
  for (int i = 1; i < n; ++i) {
    double t = std::cos(M_PI * i / n), p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre_pd(n, t, p, dp);
      double d2 = (2.0 * t * dp - n * (n + 1.0) * p) / (1.0 - t * t);
      double step = dp / d2;
      t -= step;
      if (std::fabs(step) < 1e-15) break;
    }
    x[n - i] = 0.5 * (t + 1.0);
  }
  return x;
}

// Nodal Lagrange basis at GL points; degree 0 -> node {0.5} (basis.hpp:23-27).
struct Nodal {
  std::vector<double> z;
  explicit Nodal(int degree) {
    if (degree < 0) throw std::invalid_argument("Nodal: negative degree");
    z = degree == 0 ? std::vector<double>{0.5} : lobatto(degree + 1);
  }
  int size() const { return static_cast<int>(z.size()); }
  double phi(int i, double x) const {  // basis.hpp:33-38
    double v = 1.0;
    for (int j = 0; j < size(); ++j)
      if (j != i) v *= (x - z[j]) / (z[i] - z[j]);
    return v;
  }
  double dphi(int i, double x) const {  // basis.hpp:40-50 (sum over the dropped factor)
    double s = 0.0;
    for (int l = 0; l < size(); ++l) {
      if (l == i) continue;
      double v = 1.0 / (z[i] - z[l]);
      for (int j = 0; j < size(); ++j)
        if (j != i && j != l) v *= (x - z[j]) / (z[i] - z[j]);
      s += v;
    }
    return s;
  }
};

// ================================================================================================
// L1: univariate FEM matrices (fem1d.hpp:25-269)
// ================================================================================================
enum End { E_NONE = 0, E_STRONG = 1, E_NITSCHE = 2, E_INTERIOR = 3 };  // fem1d.hpp:25-30

// h * int test_i ansatz_j (fem1d.hpp:37-49): (deg_a + deg_t)/2 + 1 Gauss points.
Mat mass1d(const Nodal& ans, const Nodal& tst, double h) {
  Rule q = gauss((ans.size() - 1 + tst.size() - 1) / 2 + 1);
  Mat m(tst.size(), ans.size());
  for (size_t l = 0; l < q.x.size(); ++l)
    for (int i = 0; i < tst.size(); ++i)
      for (int j = 0; j < ans.size(); ++j) m(i, j) += h * q.w[l] * tst.phi(i, q.x[l]) * ans.phi(j, q.x[l]);
  return m;
}

// int psi_i phi_j' on the reference cell (fem1d.hpp:53-65), h-independent.
Mat deriv1d(const Nodal& pres, const Nodal& vel) {
  Rule q = gauss((pres.size() - 1 + vel.size() - 1 + 1) / 2 + 1);
  Mat d(pres.size(), vel.size());
  for (size_t l = 0; l < q.x.size(); ++l)
    for (int i = 0; i < pres.size(); ++i)
      for (int j = 0; j < vel.size(); ++j) d(i, j) += q.w[l] * pres.phi(i, q.x[l]) * vel.dphi(j, q.x[l]);
  return d;
}

// (1/h) int phi_i' phi_j' with max(deg,1) Gauss points (fem1d.hpp:70-81).
Mat stiff1d(const Nodal& b, double h) {
  Rule q = gauss(std::max(b.size() - 1, 1));
  Mat k(b.size(), b.size());
  for (size_t l = 0; l < q.x.size(); ++l)
    for (int i = 0; i < b.size(); ++i)
      for (int j = 0; j < b.size(); ++j) k(i, j) += q.w[l] / h * b.dphi(i, q.x[l]) * b.dphi(j, q.x[l]);
  return k;
}

// SIPG Laplacian on `cells` intervals (fem1d.hpp:93-176).
Mat sipg(int degree, int cells, double h, double gamma, int left, int right) {
  if (gamma <= 0.0) throw std::invalid_argument("sipg: gamma <= 0");
  if (cells < 1) throw std::invalid_argument("sipg: cells < 1");
  Nodal b(degree);
  const int nb = b.size();
  Mat kc = stiff1d(b, h);
  if (left == E_STRONG || right == E_STRONG) {
    if (left != right) throw std::invalid_argument("sipg: mixed strong_zero ends");
    // C0 glue, endpoints removed (fem1d.hpp:105-115)
    const int nfull = cells * degree + 1;
    Mat full(nfull, nfull);
    for (int e = 0; e < cells; ++e)
      for (int i = 0; i < nb; ++i)
        for (int j = 0; j < nb; ++j) full(e * degree + i, e * degree + j) += kc(i, j);
    Mat out(nfull - 2, nfull - 2);
    for (int i = 0; i < nfull - 2; ++i)
      for (int j = 0; j < nfull - 2; ++j) out(i, j) = full(i + 1, j + 1);
    return out;
  }
  const int n = cells * nb;
  Mat m(n, n);
  for (int e = 0; e < cells; ++e)
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j) m(e * nb + i, e * nb + j) += kc(i, j);
  std::vector<double> v0(nb), v1(nb), d0(nb), d1(nb);
  for (int a = 0; a < nb; ++a) {
    v0[a] = b.phi(a, 0.0);
    v1[a] = b.phi(a, 1.0);
    d0[a] = b.dphi(a, 0.0) / h;
    d1[a] = b.dphi(a, 1.0) / h;
  }
  // interior faces: gamma[[u]][[v]] - {{u'}}[[v]] - {{v'}}[[u]], jump = left - right (fem1d.hpp:130-152)
  for (int e = 0; e + 1 < cells; ++e) {
    const int L = e * nb, R = (e + 1) * nb;
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j) {
        // trial traces: left cell (v1,d1), right cell (v0,d0); test the same with jump sign
        const double jl_i = v1[i], jr_i = -v0[i];  // test jump contributions
        const double jl_j = v1[j], jr_j = -v0[j];  // trial jump contributions
        const double al_i = 0.5 * d1[i], ar_i = 0.5 * d0[i];
        const double al_j = 0.5 * d1[j], ar_j = 0.5 * d0[j];
        m(L + i, L + j) += gamma * jl_i * jl_j - al_j * jl_i - al_i * jl_j;
        m(L + i, R + j) += gamma * jl_i * jr_j - ar_j * jl_i - al_i * jr_j;
        m(R + i, L + j) += gamma * jr_i * jl_j - al_j * jr_i - ar_i * jl_j;
        m(R + i, R + j) += gamma * jr_i * jr_j - ar_j * jr_i - ar_i * jr_j;
      }
  }
  // end terms (fem1d.hpp:156-174): nitsche (2g, 1), interior_face (g, 1/2); outward normal -1 / +1
  auto end_terms = [&](int ec, int off, const std::vector<double>& tv, const std::vector<double>& td, double nrm) {
    double wp, wc;
    if (ec == E_NITSCHE) { wp = 2.0 * gamma; wc = 1.0; }
    else if (ec == E_INTERIOR) { wp = gamma; wc = 0.5; }
    else return;
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j)
        m(off + i, off + j) += wp * tv[i] * tv[j] - wc * nrm * (td[j] * tv[i] + td[i] * tv[j]);
  };
  end_terms(left, 0, v0, d0, -1.0);
  end_terms(right, (cells - 1) * nb, v1, d1, +1.0);
  return m;
}

Mat mass_dg(int degree, int cells, double h) {  // fem1d.hpp:194-201
  Nodal b(degree);
  Mat m = mass1d(b, b, h);
  Mat f(cells * m.r, cells * m.c);
  for (int e = 0; e < cells; ++e)
    for (int i = 0; i < m.r; ++i)
      for (int j = 0; j < m.c; ++j) f(e * m.r + i, e * m.c + j) = m(i, j);
  return f;
}

Mat mass_c0(int degree, int cells, double h, bool drop) {  // fem1d.hpp:205-216
  Nodal b(degree);
  Mat m = mass1d(b, b, h);
  const int nfull = cells * degree + 1;
  Mat f(nfull, nfull);
  for (int e = 0; e < cells; ++e)
    for (int i = 0; i < b.size(); ++i)
      for (int j = 0; j < b.size(); ++j) f(e * degree + i, e * degree + j) += m(i, j);
  if (!drop) return f;
  Mat o(nfull - 2, nfull - 2);
  for (int i = 0; i < nfull - 2; ++i)
    for (int j = 0; j < nfull - 2; ++j) o(i, j) = f(i + 1, j + 1);
  return o;
}

Mat deriv_c0(int pdeg, int cells, bool drop) {  // fem1d.hpp:221-236
  Nodal p(pdeg), v(pdeg + 1);
  Mat d = deriv1d(p, v);
  const int vdeg = pdeg + 1, rows = cells * p.size(), cfull = cells * vdeg + 1;
  Mat f(rows, cfull);
  for (int e = 0; e < cells; ++e)
    for (int i = 0; i < p.size(); ++i)
      for (int j = 0; j < v.size(); ++j) f(e * p.size() + i, e * vdeg + j) += d(i, j);
  if (!drop) return f;
  Mat o(rows, cfull - 2);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cfull - 2; ++j) o(i, j) = f(i, j + 1);
  return o;
}

Mat embed1d(int degree, bool continuous) {  // fem1d.hpp:243-264
  if (degree < 0) throw std::invalid_argument("embed1d: negative degree");
  Nodal b(degree);
  const int nb = b.size();
  if (continuous) {
    Mat e(2 * degree + 1, nb);
    for (int a = 0; a <= degree; ++a)
      for (int j = 0; j < nb; ++j) {
        e(a, j) = b.phi(j, 0.5 * b.z[a]);
        e(degree + a, j) = b.phi(j, 0.5 * (1.0 + b.z[a]));
      }
    return e;
  }
  Mat e(2 * nb, nb);
  for (int a = 0; a < nb; ++a)
    for (int j = 0; j < nb; ++j) {
      e(a, j) = b.phi(j, 0.5 * b.z[a]);
      e(nb + a, j) = b.phi(j, 0.5 * (1.0 + b.z[a]));
    }
  return e;
}

double penalty(int k, double h) { return (k + 1) * (k + 2) / h; }  // fem1d.hpp:267-269

// ---- generalized symmetric-definite eigensolver: Cholesky of M + cyclic Jacobi ----
void geneig(const Mat& L, const Mat& M, Mat& S, std::vector<double>& lam) {
  const int n = L.r;
  Mat C(n, n);  // M = C C^T
  for (int j = 0; j < n; ++j) {
    double s = M(j, j);
    for (int l = 0; l < j; ++l) s -= C(j, l) * C(j, l);
    if (s <= 0.0) throw std::runtime_error("geneig: mass matrix not SPD");
    C(j, j) = std::sqrt(s);
    for (int i = j + 1; i < n; ++i) {
      double t = M(i, j);
      for (int l = 0; l < j; ++l) t -= C(i, l) * C(j, l);
      C(i, j) = t / C(j, j);
    }
  }
  // A' = C^-1 L C^-T
  Mat X(n, n);  // X = C^-1 L
  for (int col = 0; col < n; ++col)
    for (int i = 0; i < n; ++i) {
      double t = L(i, col);
      for (int l = 0; l < i; ++l) t -= C(i, l) * X(l, col);
      X(i, col) = t / C(i, i);
    }
  Mat A(n, n);  // A = X C^-T  ->  A^T = C^-1 X^T
  for (int row = 0; row < n; ++row)
    for (int i = 0; i < n; ++i) {
      double t = X(row, i);
      for (int l = 0; l < i; ++l) t -= C(i, l) * A(row, l);
      A(row, i) = t / C(i, i);
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) A(i, j) = A(j, i) = 0.5 * (A(i, j) + A(j, i));
  Mat Q(n, n);
  for (int i = 0; i < n; ++i) Q(i, i) = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i == j ? tot : off) += A(i, j) * A(i, j);
    if (off <= 1e-30 * (tot + off)) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (std::fabs(A(p, q)) < 1e-300) continue;
        double theta = (A(q, q) - A(p, p)) / (2.0 * A(p, q));
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int l = 0; l < n; ++l) {
          double alp = A(l, p), aq = A(l, q);
          A(l, p) = c * alp - s * aq;
          A(l, q) = s * alp + c * aq;
        }
        for (int l = 0; l < n; ++l) {
          double alp = A(p, l), aq = A(q, l);
          A(p, l) = c * alp - s * aq;
          A(q, l) = s * alp + c * aq;
        }
        for (int l = 0; l < n; ++l) {
          double qp = Q(l, p), qq = Q(l, q);
          Q(l, p) = c * qp - s * qq;
          Q(l, q) = s * qp + c * qq;
        }
      }
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return A(a, a) < A(b, b); });
  lam.assign(n, 0.0);
  S = Mat(n, n);
  // S = C^-T Q (back substitution with C^T)
  for (int jj = 0; jj < n; ++jj) {
    const int j = ord[jj];
    lam[jj] = A(j, j);
    std::vector<double> y(n);
    for (int i = n - 1; i >= 0; --i) {
      double t = Q(i, j);
      for (int l = i + 1; l < n; ++l) t -= C(l, i) * y[l];
      y[i] = t / C(i, i);
    }
    for (int i = 0; i < n; ++i) S(i, jj) = y[i];
  }
}

// ================================================================================================
// L2/L3: level layout (mesh.hpp:16-36). Stored layout (documented in DESIGN.md):
// one contiguous vector [u_x | u_y | u_z | p]; component c is an n_z x n_y x n_x array, x fastest,
// with n+1 nodes along its own axis c (C0, both boundary planes constrained to 0) and n along the
// two others; pressure is n x n x n, global lexicographic. n = m (k+1), m = 2 << level.
// ================================================================================================
struct Level {
  int k, level, m, n;
  double h, gamma;
  int64_t dims[3][3];  // dims[c][axis]
  int64_t off[4];
  int64_t size[4];
  int64_t total;
  Level(int kk, int lvl) : k(kk), level(lvl) {
    if (kk < 1) throw std::invalid_argument("degree k must be >= 1");
    if (lvl < 0) throw std::invalid_argument("level must be >= 0");
    m = 2 << lvl;
    n = m * (k + 1);
    h = 1.0 / m;
    gamma = penalty(k, h);
    int64_t o = 0;
    for (int c = 0; c < 3; ++c) {
      for (int a = 0; a < 3; ++a) dims[c][a] = (a == c) ? n + 1 : n;
      off[c] = o;
      size[c] = dims[c][0] * dims[c][1] * dims[c][2];
      o += size[c];
    }
    off[3] = o;
    size[3] = static_cast<int64_t>(n) * n * n;
    total = o + size[3];
  }
  int64_t vidx(int c, int64_t gx, int64_t gy, int64_t gz) const {
    return off[c] + (gz * dims[c][1] + gy) * dims[c][0] + gx;
  }
  int64_t pidx(int64_t gx, int64_t gy, int64_t gz) const { return off[3] + (gz * n + gy) * n + gx; }
};

// apply a 1D matrix A (rows = new extent, cols = old extent) along `axis` of a 3D array (x fastest)
void apply_axis(const double* in, const int* din, int axis, const Mat& A, bool trans, double* out) {
  const int R = trans ? A.c : A.r, C = trans ? A.r : A.c;
  if (din[axis] != C) throw std::logic_error("apply_axis: extent mismatch");
  int dout[3] = {din[0], din[1], din[2]};
  dout[axis] = R;
  for (int z = 0; z < dout[2]; ++z)
    for (int y = 0; y < dout[1]; ++y)
      for (int x = 0; x < dout[0]; ++x) {
        int io[3] = {x, y, z};
        double s = 0.0;
        for (int j = 0; j < C; ++j) {
          int ii[3] = {x, y, z};
          ii[axis] = j;
          const double a = trans ? A(j, io[axis]) : A(io[axis], j);
          s += a * in[(ii[2] * din[1] + ii[1]) * din[0] + ii[0]];
        }
        out[(z * dout[1] + y) * dout[0] + x] = s;
      }
}

// tensor-product evaluation: apply T[0] along x, T[1] along y, T[2] along z
std::vector<double> tensor_apply(const std::vector<double>& in, const int* din, const Mat* T[3], bool trans,
                                 int* dout) {
  std::vector<double> cur = in, nxt;
  int d[3] = {din[0], din[1], din[2]};
  for (int a = 0; a < 3; ++a) {
    int nd[3] = {d[0], d[1], d[2]};
    nd[a] = trans ? T[a]->c : T[a]->r;
    nxt.assign(static_cast<size_t>(nd[0]) * nd[1] * nd[2], 0.0);
    apply_axis(cur.data(), d, a, *T[a], trans, nxt.data());
    cur.swap(nxt);
    d[0] = nd[0]; d[1] = nd[1]; d[2] = nd[2];
  }
  for (int a = 0; a < 3; ++a) dout[a] = d[a];
  return cur;
}

// ================================================================================================
// L4: matrix-free Stokes operator, Alg. 1: cell loop with
// sum-factorised quadrature, interior-face loop (each face once, owned by the lower cell), boundary
// faces with Nitsche terms, constrained rows zero. Quadrature: k+2 Gauss points.
// ================================================================================================
struct OpTables {
  int k, Q;
  Rule q;
  Mat Vp, Dp;  // velocity parallel basis (deg k+1) at quad points: Q x (k+2)
  Mat Vo, Do;  // orthogonal / pressure basis (deg k): Q x (k+1)
  Mat ep0, ep1, dp0, dp1;  // parallel basis value/derivative at x=0,1 as 1 x (k+2) rows (reference deriv)
  Mat eo0, eo1, do0, do1;  // orthogonal basis at x=0,1: 1 x (k+1)
  explicit OpTables(int kk) : k(kk), Q(kk + 2), q(gauss(kk + 2)) {
    Nodal bp(k + 1), bo(k);
    Vp = Mat(Q, k + 2); Dp = Mat(Q, k + 2); Vo = Mat(Q, k + 1); Do = Mat(Q, k + 1);
    for (int l = 0; l < Q; ++l) {
      for (int i = 0; i < k + 2; ++i) { Vp(l, i) = bp.phi(i, q.x[l]); Dp(l, i) = bp.dphi(i, q.x[l]); }
      for (int i = 0; i < k + 1; ++i) { Vo(l, i) = bo.phi(i, q.x[l]); Do(l, i) = bo.dphi(i, q.x[l]); }
    }
    ep0 = Mat(1, k + 2); ep1 = Mat(1, k + 2); dp0 = Mat(1, k + 2); dp1 = Mat(1, k + 2);
    eo0 = Mat(1, k + 1); eo1 = Mat(1, k + 1); do0 = Mat(1, k + 1); do1 = Mat(1, k + 1);
    for (int i = 0; i < k + 2; ++i) {
      ep0(0, i) = bp.phi(i, 0.0); ep1(0, i) = bp.phi(i, 1.0);
      dp0(0, i) = bp.dphi(i, 0.0); dp1(0, i) = bp.dphi(i, 1.0);
    }
    for (int i = 0; i < k + 1; ++i) {
      eo0(0, i) = bo.phi(i, 0.0); eo1(0, i) = bo.phi(i, 1.0);
      do0(0, i) = bo.dphi(i, 0.0); do1(0, i) = bo.dphi(i, 1.0);
    }
  }
};

// gather_cell / scatter_add_cell: local lexicographic per component, constrained
// (boundary-normal) DoFs read as 0 and dropped on scatter.
void gather_vel(const Level& L, int c, const int* e, const double* x, std::vector<double>& u, int* d) {
  for (int a = 0; a < 3; ++a) d[a] = (a == c) ? L.k + 2 : L.k + 1;
  u.assign(static_cast<size_t>(d[0]) * d[1] * d[2], 0.0);
  for (int i2 = 0; i2 < d[2]; ++i2)
    for (int i1 = 0; i1 < d[1]; ++i1)
      for (int i0 = 0; i0 < d[0]; ++i0) {
        int64_t g[3] = {e[0] * (L.k + 1) + i0, e[1] * (L.k + 1) + i1, e[2] * (L.k + 1) + i2};
        if (g[c] == 0 || g[c] == L.n) continue;
        u[(i2 * d[1] + i1) * d[0] + i0] = x[L.vidx(c, g[0], g[1], g[2])];
      }
}
void scatter_vel(const Level& L, int c, const int* e, const std::vector<double>& u, const int* d, double* y) {
  for (int i2 = 0; i2 < d[2]; ++i2)
    for (int i1 = 0; i1 < d[1]; ++i1)
      for (int i0 = 0; i0 < d[0]; ++i0) {
        int64_t g[3] = {e[0] * (L.k + 1) + i0, e[1] * (L.k + 1) + i1, e[2] * (L.k + 1) + i2};
        if (g[c] == 0 || g[c] == L.n) continue;
        y[L.vidx(c, g[0], g[1], g[2])] += u[(i2 * d[1] + i1) * d[0] + i0];
      }
}
void gather_p(const Level& L, const int* e, const double* x, std::vector<double>& p) {
  const int nb = L.k + 1;
  p.assign(static_cast<size_t>(nb) * nb * nb, 0.0);
  for (int i2 = 0; i2 < nb; ++i2)
    for (int i1 = 0; i1 < nb; ++i1)
      for (int i0 = 0; i0 < nb; ++i0)
        p[(i2 * nb + i1) * nb + i0] = x[L.pidx(e[0] * nb + i0, e[1] * nb + i1, e[2] * nb + i2)];
}
void scatter_p(const Level& L, const int* e, const std::vector<double>& p, double* y) {
  const int nb = L.k + 1;
  for (int i2 = 0; i2 < nb; ++i2)
    for (int i1 = 0; i1 < nb; ++i1)
      for (int i0 = 0; i0 < nb; ++i0)
        y[L.pidx(e[0] * nb + i0, e[1] * nb + i1, e[2] * nb + i2)] += p[(i2 * nb + i1) * nb + i0];
}

// Alg. 1 step i: cell integrals
void cell_integrals(const Level& L, const OpTables& T, const int* e, const double* x, double* y) {
  const int Q = T.Q;
  const double h = L.h;
  std::vector<double> u[3], p;
  int du[3][3];
  for (int c = 0; c < 3; ++c) gather_vel(L, c, e, x, u[c], du[c]);
  gather_p(L, e, x, p);
  const int dp[3] = {L.k + 1, L.k + 1, L.k + 1};
  const size_t nq = static_cast<size_t>(Q) * Q * Q;
  // pressure at quadrature points, weighted: (p, div v) = h^2 sum_q w p (ref-div v)
  const Mat* TV[3] = {&T.Vo, &T.Vo, &T.Vo};
  int dq[3];
  std::vector<double> pq = tensor_apply(p, dp, TV, false, dq);
  std::vector<double> divq(nq, 0.0);  // sum_c ref d_c u_c at quad points
  for (int c = 0; c < 3; ++c) {
    std::vector<double> yc(u[c].size(), 0.0);
    for (int d = 0; d < 3; ++d) {
      // gradient component d at quadrature points
      const Mat* Tf[3];
      for (int a = 0; a < 3; ++a) {
        const bool par = (a == c);
        Tf[a] = (a == d) ? (par ? &T.Dp : &T.Do) : (par ? &T.Vp : &T.Vo);
      }
      std::vector<double> g = tensor_apply(u[c], du[c], Tf, false, dq);
      if (d == c)
        for (size_t i = 0; i < nq; ++i) divq[i] += g[i];
      // weights: det J * (1/h)^2 = h; divergence test term weight h^2 for d == c
      for (int q2 = 0; q2 < Q; ++q2)
        for (int q1 = 0; q1 < Q; ++q1)
          for (int q0 = 0; q0 < Q; ++q0) {
            const size_t i = (q2 * Q + q1) * Q + q0;
            const double w = T.q.w[q0] * T.q.w[q1] * T.q.w[q2];
            g[i] = h * w * g[i] + (d == c ? h * h * w * pq[i] : 0.0);
          }
      int dd[3];
      std::vector<double> contrib = tensor_apply(g, dq, Tf, true, dd);
      for (size_t i = 0; i < yc.size(); ++i) yc[i] += contrib[i];
    }
    scatter_vel(L, c, e, yc, du[c], y);
  }
  // pressure test: (q, div u) = h^2 sum_q w psi (ref-div u)
  for (int q2 = 0; q2 < Q; ++q2)
    for (int q1 = 0; q1 < Q; ++q1)
      for (int q0 = 0; q0 < Q; ++q0) {
        const size_t i = (q2 * Q + q1) * Q + q0;
        divq[i] *= h * h * T.q.w[q0] * T.q.w[q1] * T.q.w[q2];
      }
  int dd[3];
  std::vector<double> zp = tensor_apply(divq, dq, TV, true, dd);
  scatter_p(L, e, zp, y);
}

// face traces of component c on a face with normal d: value and physical normal derivative at the
// face quadrature points (d-axis collapsed to extent 1).
void face_trace(const Level& L, const OpTables& T, int c, int d, bool upper_end, const std::vector<double>& u,
                const int* du, std::vector<double>& val, std::vector<double>& dn, int* dq) {
  const Mat* Tv[3];
  const Mat* Td[3];
  for (int a = 0; a < 3; ++a) {
    const bool par = (a == c);
    if (a == d) {
      // d != c always here: orthogonal basis along d
      Tv[a] = upper_end ? &T.eo1 : &T.eo0;
      Td[a] = upper_end ? &T.do1 : &T.do0;
    } else {
      Tv[a] = par ? &T.Vp : &T.Vo;
      Td[a] = Tv[a];
    }
  }
  val = tensor_apply(u, du, Tv, false, dq);
  dn = tensor_apply(u, du, Td, false, dq);
  for (auto& v : dn) v /= L.h;
}

void face_test(const Level& L, const OpTables& T, int c, int d, bool upper_end, const std::vector<double>& fv,
               const std::vector<double>& fd, const int* dq, std::vector<double>& yc) {
  const Mat* Tv[3];
  const Mat* Td[3];
  for (int a = 0; a < 3; ++a) {
    const bool par = (a == c);
    if (a == d) {
      Tv[a] = upper_end ? &T.eo1 : &T.eo0;
      Td[a] = upper_end ? &T.do1 : &T.do0;
    } else {
      Tv[a] = par ? &T.Vp : &T.Vo;
      Td[a] = Tv[a];
    }
  }
  int dd[3];
  std::vector<double> a1 = tensor_apply(fv, dq, Tv, true, dd);
  std::vector<double> a2 = tensor_apply(fd, dq, Td, true, dd);
  for (size_t i = 0; i < yc.size(); ++i) yc[i] += a1[i] + a2[i] / L.h;
}

// weight face quadrature values by h^2 w_a w_b (d-axis has extent 1)
void face_weights(const Level& L, const OpTables& T, const int* dq, std::vector<double>& f) {
  for (int z = 0; z < dq[2]; ++z)
    for (int y = 0; y < dq[1]; ++y)
      for (int x = 0; x < dq[0]; ++x) {
        double w = L.h * L.h;
        if (dq[0] > 1) w *= T.q.w[x];
        if (dq[1] > 1) w *= T.q.w[y];
        if (dq[2] > 1) w *= T.q.w[z];
        f[(z * dq[1] + y) * dq[0] + x] *= w;
      }
}

// Alg. 1 step ii: interior face between lower cell e and e + e_d
void interior_face(const Level& L, const OpTables& T, int d, const int* e, const double* x, double* y) {
  int ep[3] = {e[0], e[1], e[2]};
  ep[d] += 1;
  for (int c = 0; c < 3; ++c) {
    if (c == d) continue;  // normal component continuous: zero jump, no face terms
    std::vector<double> um, up;
    int du[3];
    gather_vel(L, c, e, x, um, du);
    gather_vel(L, c, ep, x, up, du);
    std::vector<double> vm, dm, vp, dpp;
    int dq[3];
    face_trace(L, T, c, d, true, um, du, vm, dm, dq);
    face_trace(L, T, c, d, false, up, du, vp, dpp, dq);
    const size_t nf = vm.size();
    std::vector<double> fvm(nf), fdm(nf), fvp(nf), fdp(nf);
    for (size_t i = 0; i < nf; ++i) {
      const double jump = vm[i] - vp[i], avg = 0.5 * (dm[i] + dpp[i]);
      const double flux = L.gamma * jump - avg;
      fvm[i] = flux;
      fvp[i] = -flux;
      fdm[i] = -0.5 * jump;
      fdp[i] = -0.5 * jump;
    }
    face_weights(L, T, dq, fvm);
    face_weights(L, T, dq, fvp);
    face_weights(L, T, dq, fdm);
    face_weights(L, T, dq, fdp);
    std::vector<double> ym(um.size(), 0.0), yp(up.size(), 0.0);
    face_test(L, T, c, d, true, fvm, fdm, dq, ym);
    face_test(L, T, c, d, false, fvp, fdp, dq, yp);
    scatter_vel(L, c, e, ym, du, y);
    scatter_vel(L, c, ep, yp, du, y);
  }
}

// Alg. 1 step iii: boundary face of cell e with normal d at the upper (x_d = 1) or lower end
// (SPEC.md:277-285): 2 gamma u v - (dn u) v - u (dn v) on the tangential components.
void boundary_face(const Level& L, const OpTables& T, int d, bool upper, const int* e, const double* x, double* y) {
  const double s = upper ? 1.0 : -1.0;
  for (int c = 0; c < 3; ++c) {
    if (c == d) continue;
    std::vector<double> u;
    int du[3];
    gather_vel(L, c, e, x, u, du);
    std::vector<double> v, dn;
    int dq[3];
    face_trace(L, T, c, d, upper, u, du, v, dn, dq);
    std::vector<double> fv(v.size()), fd(v.size());
    for (size_t i = 0; i < v.size(); ++i) {
      fv[i] = 2.0 * L.gamma * v[i] - s * dn[i];
      fd[i] = -s * v[i];
    }
    face_weights(L, T, dq, fv);
    face_weights(L, T, dq, fd);
    std::vector<double> yc(u.size(), 0.0);
    face_test(L, T, c, d, upper, fv, fd, dq, yc);
    scatter_vel(L, c, e, yc, du, y);
  }
}

const OpTables& tables(int k) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<OpTables>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto& p = cache[k];
  if (!p) p = std::make_unique<OpTables>(k);
  return *p;
}

// Cells with z in [z0, z1) only (default: all): the timed CPU-baseline legs use a z-slab of the
// benchmarked level as a bounded sample (same per-DoF work as the whole level); the rows near the
// ends of the sample are then incomplete, which only the timing legs accept.
void apply_stokes(const Level& L, const double* x, double* y, int z0 = 0, int z1 = -1) {
  const OpTables& T = tables(L.k);
  const int m = L.m;
  if (z1 < 0) z1 = m;
  if (z0 == 0 && z1 == m) {
    std::fill(y, y + L.total, 0.0);
  } else {
    const int64_t H = L.k + 1;
    for (int c = 0; c < 4; ++c) {
      const int64_t pl = c < 3 ? L.dims[c][0] * L.dims[c][1] : int64_t(L.n) * L.n;
      std::fill(y + L.off[c] + z0 * H * pl, y + L.off[c] + std::min<int64_t>(z1 * H + 1, c == 2 ? L.n + 1 : L.n) * pl,
                0.0);
    }
  }
  // first index >= lo with the parity p
  auto first = [](int p, int lo) { return lo + ((p - lo) & 1); };
  // cells in 8 parity colours: same-colour cells share no DoF, so the scatter is race-free and the
  // result is independent of the thread count.
  for (int col = 0; col < 8; ++col) {
    const int px = col & 1, py = (col >> 1) & 1, pz = (col >> 2) & 1;
#pragma omp parallel for collapse(2) schedule(static)
    for (int ez = first(pz, z0); ez < z1; ez += 2)
      for (int ey = py; ey < m; ey += 2)
        for (int ex = px; ex < m; ex += 2) {
          int e[3] = {ex, ey, ez};
          cell_integrals(L, T, e, x, y);
        }
  }
  // interior faces, owned by the lower cell. Cells adjacent in direction c share the C0 nodes of
  // velocity component c, so faces are swept in 8 parity colours of the lower cell as well.
  for (int d = 0; d < 3; ++d)
    for (int col = 0; col < 8; ++col) {
      const int px = col & 1, py = (col >> 1) & 1, pz = (col >> 2) & 1;
#pragma omp parallel for collapse(2) schedule(static)
      for (int ez = first(pz, z0); ez < z1; ez += 2)
        for (int ey = py; ey < m; ey += 2)
          for (int ex = px; ex < m; ex += 2) {
            int e[3] = {ex, ey, ez};
            if (e[d] + 1 >= m) continue;
            interior_face(L, T, d, e, x, y);
          }
    }
  // boundary faces, 4 parity colours of the tangential cell coordinates
  for (int d = 0; d < 3; ++d)
    for (int upper = 0; upper < 2; ++upper) {
      if (d == 2 && !(upper ? z1 == m : z0 == 0)) continue;
      for (int col = 0; col < 4; ++col) {
        const int a1 = (d + 1) % 3, a2 = (d + 2) % 3;
        // the loop coordinate along z (i for d = 1, j for d = 0) runs over [z0, z1)
        const int ilo = a1 == 2 ? z0 : 0, ihi = a1 == 2 ? z1 : m;
        const int jlo = a2 == 2 ? z0 : 0, jhi = a2 == 2 ? z1 : m;
#pragma omp parallel for collapse(2) schedule(static)
        for (int j = first(col >> 1, jlo); j < jhi; j += 2)
          for (int i = first(col & 1, ilo); i < ihi; i += 2) {
            int e[3];
            e[d] = upper ? m - 1 : 0;
            e[a1] = i;
            e[a2] = j;
            boundary_face(L, T, d, upper != 0, e, x, y);
          }
      }
    }
}

// ================================================================================================
// L4/L5: patch local solver and smoother
// ================================================================================================
// Patch 1D data for one axis position: parallel (C0, strong zero) or orthogonal with per-end
// conditions (interior_face inside the mesh, nitsche on the boundary).
struct Patch1D {
  Mat L, M, S;
  std::vector<double> lam;
};

struct PatchData {
  int k;
  Patch1D par;        // (2k+1)
  Patch1D orth[2][2];  // [left on boundary][right on boundary], (2k+2)
  Mat D;              // (2k+2) x (2k+1)
  Mat Mp, Mpinv;      // pressure mass (2k+2)^2 and its inverse
};

Mat inverse(const Mat& A) {  // Gauss-Jordan with partial pivoting
  const int n = A.r;
  Mat a = A, inv(n, n);
  for (int i = 0; i < n; ++i) inv(i, i) = 1.0;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int i = col + 1; i < n; ++i)
      if (std::fabs(a(i, col)) > std::fabs(a(piv, col))) piv = i;
    for (int j = 0; j < n; ++j) { std::swap(a(col, j), a(piv, j)); std::swap(inv(col, j), inv(piv, j)); }
    const double d = a(col, col);
    for (int j = 0; j < n; ++j) { a(col, j) /= d; inv(col, j) /= d; }
    for (int i = 0; i < n; ++i) {
      if (i == col) continue;
      const double f = a(i, col);
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) { a(i, j) -= f * a(col, j); inv(i, j) -= f * inv(col, j); }
    }
  }
  return inv;
}

const PatchData& patch_data(int k, double h) {
  static std::mutex mu;
  static std::map<std::pair<int, double>, std::unique_ptr<PatchData>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto& p = cache[{k, h}];
  if (p) return *p;
  p = std::make_unique<PatchData>();
  p->k = k;
  const double gm = penalty(k, h);
  p->par.L = sipg(k + 1, 2, h, gm, E_STRONG, E_STRONG);
  p->par.M = mass_c0(k + 1, 2, h, true);
  geneig(p->par.L, p->par.M, p->par.S, p->par.lam);
  for (int lb = 0; lb < 2; ++lb)
    for (int rb = 0; rb < 2; ++rb) {
      Patch1D& o = p->orth[lb][rb];
      o.L = sipg(k, 2, h, gm, lb ? E_NITSCHE : E_INTERIOR, rb ? E_NITSCHE : E_INTERIOR);
      o.M = mass_dg(k, 2, h);
      geneig(o.L, o.M, o.S, o.lam);
    }
  p->D = deriv_c0(k, 2, true);
  p->Mp = mass_dg(k, 2, h);
  p->Mpinv = inverse(p->Mp);
  return *p;
}

struct PatchCtx {
  const PatchData* pd;
  const Patch1D* ax[3][3];  // ax[c][axis]: 1D data of component c along axis
  int dv[3][3];             // velocity patch dims
  int np;                   // 2k+2
};

PatchCtx make_patch_ctx(const Level& L, const int* v) {
  PatchCtx P;
  P.pd = &patch_data(L.k, L.h);
  P.np = 2 * L.k + 2;
  for (int c = 0; c < 3; ++c)
    for (int a = 0; a < 3; ++a) {
      if (a == c) {
        P.ax[c][a] = &P.pd->par;
        P.dv[c][a] = 2 * L.k + 1;
      } else {
        P.ax[c][a] = &P.pd->orth[v[a] == 1][v[a] == L.m - 1];
        P.dv[c][a] = 2 * L.k + 2;
      }
    }
  return P;
}

// A_c^-1 r by fast diagonalisation (Eq. 9)
std::vector<double> apply_Ainv(const PatchCtx& P, int c, const std::vector<double>& r) {
  const Mat* S[3] = {&P.ax[c][0]->S, &P.ax[c][1]->S, &P.ax[c][2]->S};
  int d[3];
  std::vector<double> t = tensor_apply(r, P.dv[c], S, true, d);
  for (int z = 0; z < d[2]; ++z)
    for (int y = 0; y < d[1]; ++y)
      for (int x = 0; x < d[0]; ++x)
        t[(z * d[1] + y) * d[0] + x] /= P.ax[c][0]->lam[x] + P.ax[c][1]->lam[y] + P.ax[c][2]->lam[z];
  int d2[3];
  return tensor_apply(t, d, S, false, d2);
}

// B_c u_c: D along c, M' along the two other axes (Eq. 8)
std::vector<double> apply_B(const PatchCtx& P, int c, const std::vector<double>& u) {
  const Mat* T[3];
  for (int a = 0; a < 3; ++a) T[a] = (a == c) ? &P.pd->D : &P.pd->Mp;
  int d[3];
  return tensor_apply(u, P.dv[c], T, false, d);
}
std::vector<double> apply_Bt(const PatchCtx& P, int c, const std::vector<double>& p) {
  const Mat* T[3];
  for (int a = 0; a < 3; ++a) T[a] = (a == c) ? &P.pd->D : &P.pd->Mp;
  const int dp[3] = {P.np, P.np, P.np};
  int d[3];
  return tensor_apply(p, dp, T, true, d);
}

void project_mean(std::vector<double>& p) {  // Euclidean projection onto 1^perp (A9)
  double s = 0.0;
  for (double v : p) s += v;
  s /= static_cast<double>(p.size());
  for (double& v : p) v -= s;
}
double dotv(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// Schur-complement solve: S P = B A^-1 F - G, S = B A^-1 B^T; U = A^-1 (F - B^T P)
int schur_solve(const PatchCtx& P, const std::vector<double>* F, const std::vector<double>& G,
                std::vector<double>* U, std::vector<double>& Pout, const orc_cg_opts& o) {
  const size_t npr = G.size();
  std::vector<double> rhs(npr, 0.0);
  for (int c = 0; c < 3; ++c) {
    std::vector<double> t = apply_B(P, c, apply_Ainv(P, c, F[c]));
    for (size_t i = 0; i < npr; ++i) rhs[i] += t[i];
  }
  for (size_t i = 0; i < npr; ++i) rhs[i] -= G[i];
  project_mean(rhs);
  const int dp[3] = {P.np, P.np, P.np};
  const Mat* Mi[3] = {&P.pd->Mpinv, &P.pd->Mpinv, &P.pd->Mpinv};
  auto precond = [&](const std::vector<double>& r) {
    std::vector<double> z;
    if (o.cg_precond) {
      int d[3];
      z = tensor_apply(r, dp, Mi, false, d);
    } else {
      z = r;
    }
    project_mean(z);
    return z;
  };
  auto applyS = [&](const std::vector<double>& v) {
    std::vector<double> s(npr, 0.0);
    for (int c = 0; c < 3; ++c) {
      std::vector<double> t = apply_B(P, c, apply_Ainv(P, c, apply_Bt(P, c, v)));
      for (size_t i = 0; i < npr; ++i) s[i] += t[i];
    }
    return s;
  };
  std::vector<double> x(npr, 0.0), r = rhs, z = precond(r), dvec = z;
  double rz = dotv(r, z);
  const double r0 = std::sqrt(dotv(rhs, rhs));
  int it = 0;
  for (; it < o.cg_max_iter; ++it) {
    if (!o.cg_fixed && std::sqrt(dotv(r, r)) <= o.cg_tol * r0) break;
    std::vector<double> q = applyS(dvec);
    const double dq = dotv(dvec, q);
    if (!(dq > 0.0) || rz == 0.0) break;
    const double alpha = rz / dq;
    for (size_t i = 0; i < npr; ++i) {
      x[i] += alpha * dvec[i];
      r[i] -= alpha * q[i];
    }
    project_mean(r);
    z = precond(r);
    const double rzn = dotv(r, z);
    const double beta = rzn / rz;
    rz = rzn;
    for (size_t i = 0; i < npr; ++i) dvec[i] = z[i] + beta * dvec[i];
  }
  project_mean(x);
  Pout = x;
  for (int c = 0; c < 3; ++c) {
    std::vector<double> bt = apply_Bt(P, c, x);
    std::vector<double> f = F[c];
    for (size_t i = 0; i < f.size(); ++i) f[i] -= bt[i];
    U[c] = apply_Ainv(P, c, f);
  }
  return it;
}

// R_j: patch DoFs of vertex v (mesh.hpp:39-94): velocity comp c along its own axis: global nodes
// (v_c-1)(k+1)+1 .. (v_c+1)(k+1)-1 (patch-boundary normals excluded); along the others: cells v-1, v
// -> nodes (v-1)(k+1) .. (v+1)(k+1)-1. Pressure: all 8 cells' nodes.
void patch_gather(const Level& L, const PatchCtx& P, const int* v, const double* r, std::vector<double>* F,
                  std::vector<double>& G) {
  const int nb = L.k + 1;
  for (int c = 0; c < 3; ++c) {
    const int* d = P.dv[c];
    F[c].assign(static_cast<size_t>(d[0]) * d[1] * d[2], 0.0);
    int64_t base[3];
    for (int a = 0; a < 3; ++a) base[a] = (v[a] - 1) * nb + (a == c ? 1 : 0);
    for (int z = 0; z < d[2]; ++z)
      for (int y = 0; y < d[1]; ++y)
        for (int x = 0; x < d[0]; ++x)
          F[c][(z * d[1] + y) * d[0] + x] = r[L.vidx(c, base[0] + x, base[1] + y, base[2] + z)];
  }
  const int np = P.np;
  G.assign(static_cast<size_t>(np) * np * np, 0.0);
  for (int z = 0; z < np; ++z)
    for (int y = 0; y < np; ++y)
      for (int x = 0; x < np; ++x)
        G[(z * np + y) * np + x] = r[L.pidx((v[0] - 1) * nb + x, (v[1] - 1) * nb + y, (v[2] - 1) * nb + z)];
}
void patch_scatter_add(const Level& L, const PatchCtx& P, const int* v, const std::vector<double>* U,
                       const std::vector<double>& Pp, double* x) {
  const int nb = L.k + 1;
  for (int c = 0; c < 3; ++c) {
    const int* d = P.dv[c];
    int64_t base[3];
    for (int a = 0; a < 3; ++a) base[a] = (v[a] - 1) * nb + (a == c ? 1 : 0);
    for (int z = 0; z < d[2]; ++z)
      for (int y = 0; y < d[1]; ++y)
        for (int xx = 0; xx < d[0]; ++xx)
          x[L.vidx(c, base[0] + xx, base[1] + y, base[2] + z)] += U[c][(z * d[1] + y) * d[0] + xx];
  }
  const int np = P.np;
  for (int z = 0; z < np; ++z)
    for (int y = 0; y < np; ++y)
      for (int xx = 0; xx < np; ++xx)
        x[L.pidx((v[0] - 1) * nb + xx, (v[1] - 1) * nb + y, (v[2] - 1) * nb + z)] += Pp[(z * np + y) * np + xx];
}

// one smoothing step (Alg. 2): colours 0..7 in fixed order (mesh.hpp:83-85,
// SPEC.md:425); per colour a fresh global residual, then all patches of the colour
// independently (their writes are disjoint).
// vz_lo / vz_hi: only the patches with vertex z plane in [vz_lo, vz_hi] and the residual on the cells
// around them (timing samples of the CPU-baseline legs; default: the whole level)
int smooth(const Level& L, double* x, const double* b, const orc_cg_opts& o, int vz_lo = 1, int vz_hi = -1) {
  const int nv = L.m - 1;
  if (nv <= 0) return 0;
  if (vz_hi < 0) vz_hi = nv;
  const bool full = vz_lo <= 1 && vz_hi >= nv;
  std::vector<double> r(L.total);
  int total_iters = 0;
  for (int col = 0; col < 8; ++col) {
    if (full) apply_stokes(L, x, r.data());
    else apply_stokes(L, x, r.data(), std::max(vz_lo - 1, 0), std::min(vz_hi + 1, L.m));
    for (int64_t i = 0; i < L.total; ++i) r[i] = b[i] - r[i];
    const int px = col & 1, py = (col >> 1) & 1, pz = (col >> 2) & 1;
    // vertex coordinate v_i has parity bit (v_i % 2) == colour bit i
    const int sx = px ? 1 : 2, sy = py ? 1 : 2, sz = pz ? 1 : 2;
    int iters = 0;
    const int vz0 = std::max(sz, vz_lo + ((sz - vz_lo) & 1));
#pragma omp parallel for collapse(2) schedule(dynamic) reduction(+ : iters)
    for (int vz = vz0; vz <= std::min(nv, vz_hi); vz += 2)
      for (int vy = sy; vy <= nv; vy += 2)
        for (int vx = sx; vx <= nv; vx += 2) {
          int v[3] = {vx, vy, vz};
          PatchCtx P = make_patch_ctx(L, v);
          std::vector<double> F[3], G, U[3], Pp;
          patch_gather(L, P, v, r.data(), F, G);
          iters += schur_solve(P, F, G, U, Pp, o);
          patch_scatter_add(L, P, v, U, Pp, x);
        }
    total_iters += iters;
  }
  return total_iters;
}

// ================================================================================================
// L6: transfer (fem1d.hpp:243-264). Global 1D prolongations: each fine node gets
// its row from exactly one coarse cell (shared C0 vertices carry identical values from both sides).
// ================================================================================================
struct Sparse1D {
  int rows, cols;
  std::vector<std::vector<std::pair<int, double>>> row;
};

Sparse1D prolong1d(int k, int mc, bool continuous) {
  Sparse1D P;
  if (continuous) {
    const int deg = k + 1;
    Mat E = embed1d(deg, true);  // (2deg+1) x (deg+1)
    P.rows = 2 * mc * deg + 1;
    P.cols = mc * deg + 1;
    P.row.resize(P.rows);
    std::vector<bool> done(P.rows, false);
    for (int ec = 0; ec < mc; ++ec)
      for (int r = 0; r < E.r; ++r) {
        const int gf = 2 * ec * deg + r;
        if (done[gf]) continue;
        done[gf] = true;
        for (int j = 0; j < E.c; ++j)
          if (E(r, j) != 0.0) P.row[gf].push_back({ec * deg + j, E(r, j)});
      }
  } else {
    const int nb = k + 1;
    Mat E = embed1d(k, false);  // 2nb x nb
    P.rows = 2 * mc * nb;
    P.cols = mc * nb;
    P.row.resize(P.rows);
    for (int ec = 0; ec < mc; ++ec)
      for (int r = 0; r < E.r; ++r)
        for (int j = 0; j < E.c; ++j)
          if (E(r, j) != 0.0) P.row[2 * ec * nb + r].push_back({ec * nb + j, E(r, j)});
  }
  return P;
}

// y (dims dout) += / = (P_z x P_y x P_x) x (dims din); transpose applies P^T
void kron3_apply(const Sparse1D* P[3], bool trans, const double* x, const int64_t* din, double* y,
                 const int64_t* dout) {
  // separable, axis by axis via temporaries
  std::vector<double> cur(x, x + din[0] * din[1] * din[2]);
  int64_t d[3] = {din[0], din[1], din[2]};
  for (int a = 0; a < 3; ++a) {
    int64_t nd[3] = {d[0], d[1], d[2]};
    nd[a] = dout[a];
    std::vector<double> nxt(nd[0] * nd[1] * nd[2], 0.0);
    const int64_t s_in = (a == 0) ? 1 : (a == 1 ? d[0] : d[0] * d[1]);
    const int64_t s_out = (a == 0) ? 1 : (a == 1 ? nd[0] : nd[0] * nd[1]);
    const int64_t other = d[0] * d[1] * d[2] / d[a];
#pragma omp parallel for schedule(static)
    for (int64_t o = 0; o < other; ++o) {
      // decompose o into the two non-`a` coordinates
      int64_t c3[3];
      int64_t rem = o;
      for (int b = 0; b < 3; ++b) {
        if (b == a) { c3[b] = 0; continue; }
        c3[b] = rem % d[b];
        rem /= d[b];
      }
      const int64_t bin = c3[0] + d[0] * (c3[1] + d[1] * c3[2]) - c3[a] * s_in;
      int64_t co[3] = {c3[0], c3[1], c3[2]};
      co[a] = 0;
      const int64_t bo = co[0] + nd[0] * (co[1] + nd[1] * co[2]);
      if (!trans) {
        for (int i = 0; i < P[a]->rows; ++i) {
          double s = 0.0;
          for (auto& [j, v] : P[a]->row[i]) s += v * cur[bin + j * s_in];
          nxt[bo + i * s_out] = s;
        }
      } else {
        for (int i = 0; i < P[a]->rows; ++i)
          for (auto& [j, v] : P[a]->row[i]) nxt[bo + j * s_out] += v * cur[bin + i * s_in];
      }
    }
    cur.swap(nxt);
    for (int b = 0; b < 3; ++b) d[b] = nd[b];
  }
  for (int64_t i = 0; i < d[0] * d[1] * d[2]; ++i) y[i] = cur[i];
}

void zero_constrained(const Level& L, double* x) {
  for (int c = 0; c < 3; ++c)
    for (int64_t z = 0; z < L.dims[c][2]; ++z)
      for (int64_t y = 0; y < L.dims[c][1]; ++y)
        for (int64_t xx = 0; xx < L.dims[c][0]; ++xx) {
          const int64_t g[3] = {xx, y, z};
          if (g[c] == 0 || g[c] == L.n) x[L.vidx(c, xx, y, z)] = 0.0;
        }
}

void transfer(const Level& Lc, const Level& Lf, const double* in, double* out, bool restrict_) {
  Sparse1D Pc = prolong1d(Lc.k, Lc.m, true), Pd = prolong1d(Lc.k, Lc.m, false);
  for (int c = 0; c < 4; ++c) {
    const Sparse1D* P[3];
    int64_t dc[3], df[3];
    for (int a = 0; a < 3; ++a) {
      const bool par = (c < 3 && a == c);
      P[a] = par ? &Pc : &Pd;
      dc[a] = c < 3 ? Lc.dims[c][a] : Lc.n;
      df[a] = c < 3 ? Lf.dims[c][a] : Lf.n;
    }
    if (!restrict_) {
      std::vector<double> t(df[0] * df[1] * df[2]);
      kron3_apply(P, false, in + Lc.off[c], dc, t.data(), df);
      for (int64_t i = 0; i < Lf.size[c]; ++i) out[Lf.off[c] + i] += t[i];
    } else {
      kron3_apply(P, true, in + Lf.off[c], df, out + Lc.off[c], dc);
    }
  }
}

// ================================================================================================
// L6: coarse solve: pseudo-inverse of the level-0 operator on the free DoFs,
// computed as the leading block of the inverse of the bordered system [[A, e],[e^T, 0]] where e is
// the constant-pressure kernel vector (equals A^+ for symmetric A with ker A = span e).
// ================================================================================================
struct Coarse {
  std::vector<int64_t> free;
  Mat pinv;
};
const Coarse& coarse_data(int k) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Coarse>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto& p = cache[k];
  if (p) return *p;
  p = std::make_unique<Coarse>();
  Level L(k, 0);
  std::vector<double> one(L.total, 0.0), col(L.total);
  for (int64_t i = 0; i < L.total; ++i) one[i] = 1.0;
  zero_constrained(L, one.data());
  for (int64_t i = 0; i < L.total; ++i)
    if (one[i] != 0.0) p->free.push_back(i);
  const int nf = static_cast<int>(p->free.size());
  Mat K(nf + 1, nf + 1);
  std::vector<double> e(L.total, 0.0);
  for (int j = 0; j < nf; ++j) {
    std::fill(e.begin(), e.end(), 0.0);
    e[p->free[j]] = 1.0;
    apply_stokes(L, e.data(), col.data());
    for (int i = 0; i < nf; ++i) K(i, j) = col[p->free[i]];
  }
  for (int i = 0; i < nf; ++i)
    if (p->free[i] >= L.off[3]) K(i, nf) = K(nf, i) = 1.0;
  Mat Ki = inverse(K);
  p->pinv = Mat(nf, nf);
  for (int i = 0; i < nf; ++i)
    for (int j = 0; j < nf; ++j) p->pinv(i, j) = 0.5 * (Ki(i, j) + Ki(j, i));
  return *p;
}

void coarse_solve(int k, const double* b, double* x) {
  const Coarse& C = coarse_data(k);
  Level L(k, 0);
  std::fill(x, x + L.total, 0.0);
  const int nf = static_cast<int>(C.free.size());
  for (int i = 0; i < nf; ++i) {
    double s = 0.0;
    for (int j = 0; j < nf; ++j) s += C.pinv(i, j) * b[C.free[j]];
    x[C.free[i]] = s;
  }
}

// V-cycle: x = S(0,b); x += I^up P^-1 I^down (b - A x); x = S(x,b)
void vcycle(int k, int level, const double* b, double* x, const orc_cg_opts& o) {
  if (level == 0) { coarse_solve(k, b, x); return; }
  Level L(k, level), Lc(k, level - 1);
  std::fill(x, x + L.total, 0.0);
  smooth(L, x, b, o);
  std::vector<double> r(L.total), rc(Lc.total), xc(Lc.total);
  apply_stokes(L, x, r.data());
  for (int64_t i = 0; i < L.total; ++i) r[i] = b[i] - r[i];
  transfer(Lc, L, r.data(), rc.data(), true);
  zero_constrained(Lc, rc.data());
  vcycle(k, level - 1, rc.data(), xc.data(), o);
  transfer(Lc, L, xc.data(), x, false);
  smooth(L, x, b, o);
}

// mass-weighted zero-mean projection of the pressure block
void project_pressure_mass(const Level& L, double* x) {
  Nodal b(L.k);
  Rule q = gauss(L.k + 1);
  std::vector<double> w1(L.k + 1, 0.0);  // int psi_a over the reference cell
  for (int a = 0; a <= L.k; ++a)
    for (size_t l = 0; l < q.x.size(); ++l) w1[a] += q.w[l] * b.phi(a, q.x[l]);
  const int nb = L.k + 1;
  double s = 0.0, ws = 0.0;
  for (int64_t z = 0; z < L.n; ++z)
    for (int64_t y = 0; y < L.n; ++y)
      for (int64_t xx = 0; xx < L.n; ++xx) {
        const double w = w1[xx % nb] * w1[y % nb] * w1[z % nb];
        s += w * x[L.pidx(xx, y, z)];
        ws += w;
      }
  const double mean = s / ws;
  for (int64_t i = 0; i < L.size[3]; ++i) x[L.off[3] + i] -= mean;
}

double dotn(const double* a, const double* b, int64_t n) {
  double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// FGMRES: right preconditioned, no restart, MGS with one
// re-orthogonalisation pass when orthogonality is lost, x0 = 0.
int fgmres(int k, int level, const double* b, double* x, double tol, int max_iter, const orc_cg_opts& o,
           double* hist) {
  Level L(k, level);
  const int64_t N = L.total;
  std::vector<std::vector<double>> V, Z;
  std::vector<std::vector<double>> H(max_iter + 1, std::vector<double>(max_iter, 0.0));
  std::vector<double> cs(max_iter), sn(max_iter), g(max_iter + 1, 0.0);
  const double beta = std::sqrt(dotn(b, b, N));
  std::fill(x, x + N, 0.0);
  if (hist) hist[0] = beta;
  if (beta == 0.0) return 0;
  V.emplace_back(b, b + N);
  for (auto& v : V[0]) v /= beta;
  g[0] = beta;
  int it = 0;
  for (; it < max_iter;) {
    const int j = it;
    Z.emplace_back(N);
    vcycle(k, level, V[j].data(), Z[j].data(), o);
    std::vector<double> w(N);
    apply_stokes(L, Z[j].data(), w.data());
    const double wn0 = std::sqrt(dotn(w.data(), w.data(), N));
    for (int i = 0; i <= j; ++i) {
      const double hij = dotn(w.data(), V[i].data(), N);
      H[i][j] = hij;
      for (int64_t l = 0; l < N; ++l) w[l] -= hij * V[i][l];
    }
    double wn = std::sqrt(dotn(w.data(), w.data(), N));
    (void)wn0;
    // second MGS pass ("twice is enough"): always run, which meets SPEC.md:550's 1e-10 criterion
    for (int i = 0; i <= j; ++i) {
      const double c = dotn(w.data(), V[i].data(), N);
      H[i][j] += c;
      for (int64_t l = 0; l < N; ++l) w[l] -= c * V[i][l];
    }
    wn = std::sqrt(dotn(w.data(), w.data(), N));
    H[j + 1][j] = wn;
    for (int i = 0; i < j; ++i) {  // apply previous Givens rotations
      const double t = cs[i] * H[i][j] + sn[i] * H[i + 1][j];
      H[i + 1][j] = -sn[i] * H[i][j] + cs[i] * H[i + 1][j];
      H[i][j] = t;
    }
    const double den = std::hypot(H[j][j], H[j + 1][j]);
    cs[j] = H[j][j] / den;
    sn[j] = H[j + 1][j] / den;
    H[j][j] = den;
    H[j + 1][j] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    ++it;
    if (hist) hist[it] = std::fabs(g[j + 1]);
    if (std::fabs(g[j + 1]) <= tol * beta || wn == 0.0) break;
    V.emplace_back(w);
    for (auto& v : V.back()) v /= wn;
  }
  std::vector<double> y(it);
  for (int i = it - 1; i >= 0; --i) {
    double s = g[i];
    for (int l = i + 1; l < it; ++l) s -= H[i][l] * y[l];
    y[i] = s / H[i][i];
  }
  for (int i = 0; i < it; ++i)
    for (int64_t l = 0; l < N; ++l) x[l] += y[i] * Z[i][l];
  project_pressure_mass(L, x);
  return it;
}

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument&) {
    return -22;  // EINVAL
  } catch (const std::exception&) {
    return -1;
  }
}

}  // namespace

// ================================================================================================
// C ABI
// ================================================================================================
extern "C" {

int orc_gauss_quadrature(int n, double* pts, double* wts) {
  return guard([&] {
    Rule q = gauss(n);
    for (int i = 0; i < n; ++i) { pts[i] = q.x[i]; wts[i] = q.w[i]; }
    return 0;
  });
}
int orc_gauss_lobatto_points(int n, double* pts) {
  return guard([&] {
    auto p = lobatto(n);
    for (int i = 0; i < n; ++i) pts[i] = p[i];
    return 0;
  });
}
int orc_mass_matrix_1d(int da, int dt, double h, double* out, int cap, int* r, int* c) {
  return guard([&] { return emit(mass1d(Nodal(da), Nodal(dt), h), out, cap, r, c); });
}
int orc_derivative_matrix_1d(int dp, int dv, double* out, int cap, int* r, int* c) {
  return guard([&] { return emit(deriv1d(Nodal(dp), Nodal(dv)), out, cap, r, c); });
}
int orc_sipg_laplace_1d(int degree, int cells, double h, double gamma, int left, int right, double* out, int cap,
                        int* r, int* c) {
  return guard([&] { return emit(sipg(degree, cells, h, gamma, left, right), out, cap, r, c); });
}
int orc_mass_matrix_dg(int degree, int cells, double h, double* out, int cap, int* r, int* c) {
  return guard([&] { return emit(mass_dg(degree, cells, h), out, cap, r, c); });
}
int orc_mass_matrix_c0(int degree, int cells, double h, int drop, double* out, int cap, int* r, int* c) {
  return guard([&] { return emit(mass_c0(degree, cells, h, drop != 0), out, cap, r, c); });
}
int orc_derivative_matrix_c0(int pdeg, int cells, int drop, double* out, int cap, int* r, int* c) {
  return guard([&] { return emit(deriv_c0(pdeg, cells, drop != 0), out, cap, r, c); });
}
int orc_embedding_1d(int degree, int continuous, double* out, int cap, int* r, int* c) {
  return guard([&] { return emit(embed1d(degree, continuous != 0), out, cap, r, c); });
}
double orc_default_penalty(int k, double h) { return penalty(k, h); }

int orc_generalized_eig(int n, const double* Lp, const double* Mp, double* S, double* lambda) {
  return guard([&] {
    Mat L(n, n), M(n, n), Sm;
    std::memcpy(L.a.data(), Lp, sizeof(double) * n * n);
    std::memcpy(M.a.data(), Mp, sizeof(double) * n * n);
    std::vector<double> lam;
    geneig(L, M, Sm, lam);
    std::memcpy(S, Sm.a.data(), sizeof(double) * n * n);
    std::memcpy(lambda, lam.data(), sizeof(double) * n);
    return 0;
  });
}

void orc_sizes(int k, int level, int64_t* sizes) {
  Level L(k, level);
  for (int i = 0; i < 4; ++i) sizes[i] = L.size[i];
  sizes[4] = L.total;
}

int orc_apply_stokes(int k, int level, const double* x, double* y) {
  return guard([&] {
    Level L(k, level);
    apply_stokes(L, x, y);
    return 0;
  });
}

int orc_residual(int k, int level, const double* b, const double* x, double* r) {
  return guard([&] {
    Level L(k, level);
    apply_stokes(L, x, r);
    for (int64_t i = 0; i < L.total; ++i) r[i] = b[i] - r[i];
    return 0;
  });
}

int orc_smooth(int k, int level, double* x, const double* b, const orc_cg_opts* opts, int* iters) {
  return guard([&] {
    Level L(k, level);
    int it = smooth(L, x, b, *opts);
    if (iters) *iters = it;
    return 0;
  });
}

void orc_patch_sizes(int k, int* sizes) {
  sizes[0] = sizes[1] = sizes[2] = (2 * k + 1) * (2 * k + 2) * (2 * k + 2);
  sizes[3] = (2 * k + 2) * (2 * k + 2) * (2 * k + 2);
}

int orc_patch_solve(int k, int level, const int* vertex, const double* F, const double* G, double* U, double* P,
                    const orc_cg_opts* opts, int* iters) {
  return guard([&] {
    Level L(k, level);
    PatchCtx C = make_patch_ctx(L, vertex);
    int sz[4];
    orc_patch_sizes(k, sz);
    std::vector<double> Fv[3], Gv(G, G + sz[3]), Uv[3], Pv;
    for (int c = 0; c < 3; ++c) Fv[c].assign(F + c * sz[0], F + (c + 1) * sz[0]);
    int it = schur_solve(C, Fv, Gv, Uv, Pv, *opts);
    for (int c = 0; c < 3; ++c) std::memcpy(U + c * sz[0], Uv[c].data(), sizeof(double) * sz[0]);
    std::memcpy(P, Pv.data(), sizeof(double) * sz[3]);
    if (iters) *iters = it;
    return 0;
  });
}

int orc_prolongate_add(int k, int coarse_level, const double* xc, double* xf) {
  return guard([&] {
    Level Lc(k, coarse_level), Lf(k, coarse_level + 1);
    transfer(Lc, Lf, xc, xf, false);
    return 0;
  });
}
int orc_restrict(int k, int coarse_level, const double* rf, double* rc) {
  return guard([&] {
    Level Lc(k, coarse_level), Lf(k, coarse_level + 1);
    transfer(Lc, Lf, rf, rc, true);
    zero_constrained(Lc, rc);
    return 0;
  });
}
int orc_coarse_solve(int k, const double* b, double* x) {
  return guard([&] {
    coarse_solve(k, b, x);
    return 0;
  });
}
int orc_vcycle(int k, int level, const double* b, double* x, const orc_cg_opts* opts) {
  return guard([&] {
    vcycle(k, level, b, x, *opts);
    return 0;
  });
}
int orc_fgmres(int k, int level, const double* b, double* x, double rel_tol, int max_iter, const orc_cg_opts* opts,
               double* history) {
  return guard([&] { return fgmres(k, level, b, x, rel_tol, max_iter, *opts, history); });
}
// mass-weighted pressure mean removal on a full level vector (project_zero_mean SPEC.md:212-220)
int orc_project_zero_mean(int k, int level, double* x) {
  return guard([&] {
    project_pressure_mass(Level(k, level), x);
    return 0;
  });
}
// timing samples for the CPU-baseline legs (bench.py): the operator on the cells z in [z0, z1) of the
// level, and one smoothing step restricted to the patches with vertex z plane in [vz0, vz1]
int orc_apply_stokes_sample(int k, int level, const double* x, double* y, int z0, int z1) {
  return guard([&] {
    apply_stokes(Level(k, level), x, y, z0, z1);
    return 0;
  });
}
int orc_smooth_sample(int k, int level, double* x, const double* b, const orc_cg_opts* opts, int vz0, int vz1,
                      int* iters) {
  return guard([&] {
    *iters = smooth(Level(k, level), x, b, *opts, vz0, vz1);
    return 0;
  });
}
void orc_set_threads(int n) { omp_set_num_threads(n); }
}
