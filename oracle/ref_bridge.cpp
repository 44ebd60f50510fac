// C-ABI bridge over the UNMODIFIED reference headers (/root/reference/proj/include/stokesmg/*.hpp),
// compiled in place by oracle/Makefile into oracle/_ref/libstokesmg_ref.so.
// TEST INFRASTRUCTURE ONLY: used by tests/golden/make_golden.py to produce golden vectors that pin
// the CPU oracle (oracle/stokes_oracle.cpp). Never linked into the product library.
#include <cstdint>
#include <cstring>

#include "stokesmg/block_vector.hpp"
#include "stokesmg/fem1d.hpp"
#include "stokesmg/mesh.hpp"

using namespace stokesmg;

namespace {
int copy_out(const Matrix& m, double* out, int cap, int* rows, int* cols) {
  *rows = m.rows();
  *cols = m.cols();
  if (m.rows() * m.cols() > cap) return -1;
  for (int i = 0; i < m.rows(); ++i)
    for (int j = 0; j < m.cols(); ++j) out[i * m.cols() + j] = m(i, j);
  return 0;
}
EndCondition ec(int e) { return static_cast<EndCondition>(e); }
}  // namespace

extern "C" {

int ref_gauss_quadrature(int n, double* pts, double* wts) {  // quadrature.hpp:38-62
  auto q = gauss_quadrature(n);
  for (int i = 0; i < n; ++i) { pts[i] = q.points[i]; wts[i] = q.weights[i]; }
  return 0;
}
int ref_gauss_lobatto_points(int n, double* pts) {  // quadrature.hpp:65-86
  auto p = gauss_lobatto_points(n);
  for (int i = 0; i < n; ++i) pts[i] = p[i];
  return 0;
}
// fem1d.hpp:37-49 with Basis1D::gauss_lobatto of the two degrees
int ref_mass_matrix_1d(int deg_ansatz, int deg_test, double h, double* out, int cap, int* r, int* c) {
  return copy_out(mass_matrix_1d(Basis1D::gauss_lobatto(deg_ansatz), Basis1D::gauss_lobatto(deg_test), h), out, cap, r, c);
}
int ref_derivative_matrix_1d(int deg_p, int deg_v, double* out, int cap, int* r, int* c) {  // fem1d.hpp:53-65
  return copy_out(derivative_matrix_1d(Basis1D::gauss_lobatto(deg_p), Basis1D::gauss_lobatto(deg_v)), out, cap, r, c);
}
int ref_sipg_laplace_1d(int degree, int cells, double h, double gamma, int left, int right, double* out, int cap,
                        int* r, int* c) {  // fem1d.hpp:93-176
  return copy_out(sipg_laplace_1d(degree, cells, h, gamma, ec(left), ec(right)), out, cap, r, c);
}
int ref_mass_matrix_dg(int degree, int cells, double h, double* out, int cap, int* r, int* c) {  // fem1d.hpp:194-201
  auto b = Basis1D::gauss_lobatto(degree);
  return copy_out(mass_matrix_dg(b, b, cells, h), out, cap, r, c);
}
int ref_mass_matrix_c0(int degree, int cells, double h, int drop, double* out, int cap, int* r, int* c) {  // 205-216
  return copy_out(mass_matrix_c0(degree, cells, h, drop != 0), out, cap, r, c);
}
int ref_derivative_matrix_c0(int pdeg, int cells, int drop, double* out, int cap, int* r, int* c) {  // 221-236
  return copy_out(derivative_matrix_c0(pdeg, cells, drop != 0), out, cap, r, c);
}
int ref_embedding_1d(int degree, int continuous, double* out, int cap, int* r, int* c) {  // 243-264
  return copy_out(embedding_1d(degree, continuous ? Continuity::continuous : Continuity::discontinuous), out, cap, r, c);
}
double ref_default_penalty(int k, double h) { return default_penalty(k, h); }  // 267-269

// mesh.hpp:60-103: patches of one level, flattened (vertex xyz, 8 cells, colour) per patch.
int64_t ref_enumerate_patches(int dim, int max_level, int level, int* vertex, int64_t* cells, int* color, int64_t cap) {
  auto mesh = build_hierarchy(dim, max_level);
  auto ps = enumerate_patches(mesh, level);
  if (static_cast<int64_t>(ps.size()) > cap) return -static_cast<int64_t>(ps.size());
  for (size_t i = 0; i < ps.size(); ++i) {
    for (int d = 0; d < 3; ++d) vertex[3 * i + d] = ps[i].vertex[d];
    for (int j = 0; j < 8; ++j) cells[8 * i + j] = ps[i].cells[j];
    color[i] = ps[i].color;
  }
  return static_cast<int64_t>(ps.size());
}

// block_vector.hpp:52-61: double-accumulated dot of float block vectors (dim 3).
double ref_dot_f32(const float* a, const float* b, int64_t n_each_v0, int64_t n_each_v1, int64_t n_each_v2,
                   int64_t np) {
  BlockVector<3, float> x, y;
  x.resize({n_each_v0, n_each_v1, n_each_v2}, np);
  y.resize({n_each_v0, n_each_v1, n_each_v2}, np);
  int64_t off = 0;
  int64_t ns[3] = {n_each_v0, n_each_v1, n_each_v2};
  for (int c = 0; c < 3; ++c) {
    std::memcpy(x.velocity[c].data(), a + off, ns[c] * 4);
    std::memcpy(y.velocity[c].data(), b + off, ns[c] * 4);
    off += ns[c];
  }
  std::memcpy(x.pressure.data(), a + off, np * 4);
  std::memcpy(y.pressure.data(), b + off, np * 4);
  return dot(x, y);
}
}
