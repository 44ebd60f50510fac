// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A CPU restatement of the reference's algorithm for the hot path of arXiv 2410.09497 (matrix-free
// H(div)-DG Stokes operator, vertex-patch Schur/fast-diagonalisation smoother, intergrid transfer,
// V-cycle, mixed-precision FGMRES). It follows /root/reference/SPEC.md and the exact semantics of the
// reference headers /root/reference/proj/include/stokesmg/*.hpp (cited per function in the .cpp).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
// this library, and only as the checker or the timed CPU baseline. The product path
// (paper_2410_09497_b200/) never links or calls it.
//
// Parity pinning: the 1D FEM layer is pinned against golden vectors produced by the unmodified
// reference headers (tests/golden/make_golden.py -> tests/golden/fem1d_golden.json). The operator is
// pinned against an independent dense brute-force assembly (tests/oracle_dense.py).
// The eigensolver has no reference pin (Eigen is absent): it is cross-checked
// against numpy/LAPACK.
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

// ---- 1D layer (restated from fem1d.hpp / quadrature.hpp / basis.hpp) ---------------------------
int orc_gauss_quadrature(int n, double* pts, double* wts);
int orc_gauss_lobatto_points(int n, double* pts);
int orc_mass_matrix_1d(int deg_ansatz, int deg_test, double h, double* out, int cap, int* r, int* c);
int orc_derivative_matrix_1d(int deg_p, int deg_v, double* out, int cap, int* r, int* c);
int orc_sipg_laplace_1d(int degree, int cells, double h, double gamma, int left, int right, double* out, int cap,
                        int* r, int* c);
int orc_mass_matrix_dg(int degree, int cells, double h, double* out, int cap, int* r, int* c);
int orc_mass_matrix_c0(int degree, int cells, double h, int drop, double* out, int cap, int* r, int* c);
int orc_derivative_matrix_c0(int pdeg, int cells, int drop, double* out, int cap, int* r, int* c);
int orc_embedding_1d(int degree, int continuous, double* out, int cap, int* r, int* c);
double orc_default_penalty(int k, double h);
// generalized symmetric-definite eigenproblem L S = M S Lambda, S^T M S = I, ascending
int orc_generalized_eig(int n, const double* L, const double* M, double* S, double* lambda);

// ---- level layout ---------------------------------------------------------------------------------
// sizes[0..2] = stored velocity component sizes, sizes[3] = pressure, sizes[4] = total.
void orc_sizes(int k, int level, int64_t* sizes);

// ---- operators (fp64) -----------------------------------------------------------------------------
// y = A x (Alg. 1 of PAPER.md:115-151), symmetric sign [[A,B^T],[B,0]].
int orc_apply_stokes(int k, int level, const double* x, double* y);
// r = b - A x
int orc_residual(int k, int level, const double* b, const double* x, double* r);

// Local-solver / smoother options.
typedef struct {
  int cg_max_iter;   // inner Schur-CG iteration cap
  double cg_tol;     // relative tolerance on the projected Schur residual
  int cg_fixed;      // 1: run exactly cg_max_iter iterations (parity mode)
  int cg_precond;    // 0: none (SPEC-literal), 1: pressure-mass (M'^-1 x M'^-1 x M'^-1)
} orc_cg_opts;

// one multiplicative colour-by-colour smoothing step on x
int orc_smooth(int k, int level, double* x, const double* b, const orc_cg_opts* opts, int* cg_iters_total);
// local Schur solve on one patch (vertex v = (vx,vy,vz)), F/G in patch-local x-fastest ordering
int orc_patch_solve(int k, int level, const int* vertex, const double* F, const double* G, double* U, double* P,
                    const orc_cg_opts* opts, int* iters);
// patch-local sizes: [vel comp 0, 1, 2, pressure]
void orc_patch_sizes(int k, int* sizes);

// ---- transfer -------------------------------------------------------------------
int orc_prolongate_add(int k, int coarse_level, const double* xc, double* xf);  // xf += P xc
int orc_restrict(int k, int coarse_level, const double* rf, double* rc);       // rc = P^T rf

// ---- multigrid / Krylov ---------------------------------------------------------
int orc_coarse_solve(int k, const double* b, double* x);  // level-0 pseudo-inverse apply
int orc_vcycle(int k, int level, const double* b, double* x, const orc_cg_opts* opts);
// FGMRES, right-preconditioned by the V-cycle; returns iterations, history[0..it] = residual norms.
int orc_fgmres(int k, int level, const double* b, double* x, double rel_tol, int max_iter, const orc_cg_opts* opts,
               double* history);

// mass-weighted zero-mean projection of the pressure block of a level vector
int orc_project_zero_mean(int k, int level, double* x);

// timing samples (bench.py CPU legs): operator on the cells z in [z0, z1); one smoothing step on the
// patches with vertex z plane in [vz0, vz1] (rows at the sample ends are incomplete: timing only)
int orc_apply_stokes_sample(int k, int level, const double* x, double* y, int z0, int z1);
int orc_smooth_sample(int k, int level, double* x, const double* b, const orc_cg_opts* opts, int vz0, int vz1,
                      int* iters);

void orc_set_threads(int n);

#ifdef __cplusplus
}
#endif
