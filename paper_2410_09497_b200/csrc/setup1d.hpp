// Host-side setup of the constant 1D tables the sm_100a kernels consume.
//
// The operator is a Kronecker sum of banded 1D matrices on the uniform Cartesian mesh:
// per velocity component c, A_c = L_c (x) M_o1 (x) M_o2 + M_c (x) L_o1 (x) M_o2 + M_c (x) M_o1 (x) L_o2,
// B_c = D_c (x) M'_o1 (x) M'_o2, with the reference's univariate matrices
// (proj/include/stokesmg/fem1d.hpp:93-236): along c the C0 degree-(k+1) mass/stiffness
// (mass_matrix_c0, sipg_laplace_1d(strong_zero)); along the other axes the DG degree-k mass and SIPG
// Laplacian with Nitsche ends (mass_matrix_dg, sipg_laplace_1d(weak_nitsche)); D = derivative_matrix_c0.
//
// This file re-derives those matrices in the kernels' "cell-row block" form: for an output cell e
// (variant 0 = first cell, 1 = interior, 2 = last cell) and a neighbour offset delta in {-1,0,+1},
// W[variant][delta+1][a][b] couples output row a of cell e to input local node b of cell e+delta.
// Patch (2-cell) matrices of the smoother are principal submatrices of these global operators, which
// realises the per-position end conditions of fem1d.hpp:17-30.
#pragma once
#include <vector>

namespace smg {

enum Op1D { OP_MO = 0, OP_LO = 1, OP_MP = 2, OP_LP = 3, OP_D = 4, OP_DT = 5, N_OPS = 6 };

// Row-major dense matrix (host, fp64).
struct Dense {
  int r = 0, c = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(int rr, int cc) : r(rr), c(cc), a(static_cast<size_t>(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
};

struct LevelTables {
  int k = 0, m = 0;
  double h = 0, gamma = 0;
  // ops[op] holds 3 variants x 3 deltas x (k+1) rows x (k+2) cols (cols padded to k+2)
  std::vector<double> ops;
  int op_stride() const { return 9 * (k + 1) * (k + 2); }
  double& w(int op, int var, int delta, int a, int b) {
    return ops[static_cast<size_t>(op) * op_stride() + ((var * 3 + delta + 1) * (k + 1) + a) * (k + 2) + b];
  }
};

// Fast-diagonalisation data of the vertex-patch local solver (Eq. 9-10).
struct PatchTables {
  int k = 0;
  // parallel axis (C0, strong zero ends): (2k+1)x(2k+1) eigenvectors S (column j = eigvec j)
  Dense par_S;
  std::vector<double> par_lam;
  // orthogonal axis, variant v = 2*left_on_boundary + right_on_boundary: (2k+2)x(2k+2)
  Dense orth_S[4];
  std::vector<double> orth_lam[4];
  Dense D;      // (2k+2) x (2k+1) patch divergence factor
  Dense Mp;     // (2k+2)^2 pressure mass factor (= M' of Eq. 8)
  Dense Mpinv;  // its inverse (pressure-mass preconditioner of the inner CG)
  // patch matrices kept for tests / diagnostics
  Dense par_L, par_M, orth_L[4], orth_M;
  // rows of the GLOBAL operator at the patch DoFs, restricted to the columns of the patch window
  // (fused halo-residual smoother): per axis-position variant v = 2*left_on_boundary + right_on_boundary
  //   win_LO[v]  (2k+2) x (4k+4)  SIPG rows of the 2 patch cells from cells v-2 .. v+1
  //   win_MO4    (2k+2) x (4k+4)  DG mass of the 2 patch cells in the same 4-cell columns
  //   win_LP[v], win_MP[v]  (2k+1) x (2k+3)  C0 rows of the interior nodes from the 2 cells' C0 nodes
  //   win_D[v]   (2k+2) x (2k+3)  divergence rows; constrained (boundary-normal) columns are zero
  Dense win_LO[4], win_MO4, win_LP[4], win_MP[4], win_D[4];
};

// Transfer: canonical embedding (fem1d.hpp:243-264)
struct TransferTables {
  int k = 0;
  Dense Ec;  // continuous, (2k+3) x (k+2)
  Dense Ed;  // discontinuous, (2k+2) x (k+1)
};

LevelTables build_level_tables(int k, int level);
PatchTables build_patch_tables(const LevelTables& lt);
TransferTables build_transfer_tables(int k);

// Reference-cell (h = 1) operator blocks for the register-pencil kernels, for every k in 1..kMaxK,
// concatenated in the order of ref_layout(): per k
//   MO (H x H) DG mass | LO0 (H x H) interior SIPG diagonal block | LOM (H x H) delta=-1 block |
//   LOP (H x H) delta=+1 block | DLF (H x H) first-cell correction (Nitsche - interior face) |
//   DLL (H x H) last-cell correction | MP (P x P) C0 cell mass | LP (P x P) C0 cell stiffness |
//   D (H x P) divergence factor,     H = k+1, P = k+2.
// On level l (h = 2^-(l+1)) every mass block scales with h and every SIPG / stiffness block with 1/h
// (the penalty (k+1)(k+2)/h and the trace derivatives carry the same 1/h); D is h-independent.
constexpr int kMaxK = 7;
constexpr int ref_size(int k) { return 6 * (k + 1) * (k + 1) + 2 * (k + 2) * (k + 2) + (k + 1) * (k + 2); }
constexpr int ref_base(int k) {
  int s = 0;
  for (int j = 1; j < k; ++j) s += ref_size(j);
  return s;
}
constexpr int kRefTotal = ref_base(kMaxK + 1);
std::vector<double> reference_cell_tables();

// Weights of the mass-weighted pressure mean: int psi_a over the reference cell.
std::vector<double> pressure_node_weights(int k);

// Symmetric eigen-decomposition by cyclic Jacobi (A = V diag(w) V^T), ascending.
void sym_eig(const Dense& A, Dense& V, std::vector<double>& w);
// Generalised problem L S = M S Lambda with S^T M S = I, via M^{-1/2}.
void gen_eig(const Dense& L, const Dense& M, Dense& S, std::vector<double>& lam);
Dense inverse(const Dense& A);

}  // namespace smg
