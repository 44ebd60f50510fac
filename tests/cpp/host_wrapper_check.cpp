// Drives the C++ host wrapper (paper_2410_09497_b200/host/stokesmg_b200.hpp) the way a reference-side
// caller would: BlockVector in / out, device vectors, smoother / transfer / V-cycle / mixed solve.
// Built by tests/test_host_cpp.py (CPU: compile + link) and run there under -m gpu.
#include <array>
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "../../paper_2410_09497_b200/host/stokesmg_b200.hpp"

// The reference's own BlockVector (proj/include/stokesmg/block_vector.hpp:15-93, Eigen-free) when its
// header is on the include path (__graft_entry__.build() places it under baseline/_ref/include, git-
// ignored, from /root/reference); otherwise a caller-side struct with the same member layout.
#if __has_include(<stokesmg/block_vector.hpp>)
#include <stokesmg/block_vector.hpp>
template <int dim, class T>
using BlockVector = stokesmg::BlockVector<dim, T>;
static const char* kBlockVector = "reference stokesmg::BlockVector";
#else
template <int dim, class T>
struct BlockVector {
  std::array<std::vector<T>, dim> velocity;
  std::vector<T> pressure;
};
static const char* kBlockVector = "look-alike BlockVector";
#endif

using namespace stokesmg::b200;

#define REQUIRE(cond)                                                   \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::fprintf(stderr, "FAILED %s (line %d)\n", #cond, __LINE__);   \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int main() {
  const int k = 2, L = 3;
  Context ctx(k, L, 0, CgOptions{30, 1e-8, false, true});
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  BlockVector<3, double> x, y_host, y_dev;
  DeviceVector<double>::resize_blocks(ctx, L, x);
  for (auto& b : x.velocity)
    for (auto& v : b) v = U(rng);
  for (auto& v : x.pressure) v = U(rng);

  StokesOperator<double> A(ctx, L);
  A.vmult(y_host, x);  // host BlockVector path
  DeviceVector<double> dx(ctx, L), dy(ctx, L), dz(ctx, L), dAz(ctx, L);
  dx.upload(x);
  A.vmult(dy, dx);  // device path
  dy.download(y_dev);
  for (int c = 0; c < 3; ++c) REQUIRE(y_host.velocity[c] == y_dev.velocity[c]);
  REQUIRE(y_host.pressure == y_dev.pressure);

  // symmetry <A x, z> = <x, A z> on vectors with zero constrained entries (A applied once zeroes them)
  BlockVector<3, double> z;
  DeviceVector<double>::resize_blocks(ctx, L, z);
  for (auto& b : z.velocity)
    for (auto& v : b) v = U(rng);
  for (auto& v : z.pressure) v = U(rng);
  dz.upload(z);
  A.vmult(dAz, dz);  // dAz, dy have zero constrained rows
  DeviceVector<double> dAy(ctx, L), dAAz(ctx, L);
  A.vmult(dAy, dy);
  A.vmult(dAAz, dAz);
  const double s1 = dAy.dot(dAz), s2 = dy.dot(dAAz);
  REQUIRE(std::fabs(s1 - s2) <= 1e-9 * std::fabs(s1));

  // fp32 hierarchy pieces: smoother, transfer, V-cycle
  DeviceVector<float> b32(ctx, L), x32(ctx, L), xc(ctx, L - 1), rc(ctx, L - 1);
  b32.copy_from(dy);
  VertexPatchSmoother<float>(ctx, L).smooth(x32, b32, true);
  Transfer<float> T(ctx);
  T.restrict_down(L - 1, rc, b32);
  T.prolongate_add(L - 1, x32, xc);
  MGPreconditioner<float>(ctx, L).vmult(x32, b32);

  // mixed-precision MG-FGMRES
  DeviceVector<double> sol(ctx, L), r(ctx, L);
  const SolveResult res = solve_mixed(ctx, L, sol, dy, 1e-8, 40, true);
  A.residual(r, dy, sol);
  const double rn = std::sqrt(r.dot(r)), bn = std::sqrt(dy.dot(dy));
  REQUIRE(res.iterations >= 1 && res.iterations <= 15);
  REQUIRE(rn <= 1e-7 * bn);

  // errors surface as the reference's exception type
  bool threw = false;
  try {
    StokesOperator<double>(ctx, L + 1).vmult(dz, dx);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw);
  // the reference's BLAS-1 on the downloaded vectors agrees with the device dot (block_vector.hpp:53-61)
#if __has_include(<stokesmg/block_vector.hpp>)
  BlockVector<3, double> yd;
  dy.download(yd);
  REQUIRE(std::fabs(stokesmg::dot(yd, yd) - dy.dot(dy)) <= 1e-12 * dy.dot(dy));
#endif
  std::printf("host wrapper ok (%s): iterations %d, rel residual %.3e, launches %lld\n", kBlockVector,
              res.iterations, rn / bn, static_cast<long long>(ctx.launches()));
  return 0;
}
