// K1/K2 dispatch: y = A x / r = b - A x, one kernel instantiation set per degree (vmult_k<K>.cu,
// kernel design in vmult_kernel.cuh).
#include <algorithm>
#include <vector>

#include "vmult.cuh"

namespace smg {

void upload_reference_tables() {
  const std::vector<double> t = reference_cell_tables();
  const std::vector<float> f(t.begin(), t.end());
  vmult_upload_k<1>(t.data(), f.data());
  vmult_upload_k<2>(t.data(), f.data());
  vmult_upload_k<3>(t.data(), f.data());
  vmult_upload_k<4>(t.data(), f.data());
  vmult_upload_k<5>(t.data(), f.data());
  vmult_upload_k<6>(t.data(), f.data());
  vmult_upload_k<7>(t.data(), f.data());
  zm_upload_k<1>(t.data(), f.data());
  zm_upload_k<2>(t.data(), f.data());
}

void launch_vmult_args(Context& ctx, int level, int prec, const VmultArgs& a) {
  // k <= 2: the z-march kernel where its tiles fit the level, else the brick kernel
  if (ctx.cfg.degree == 1 && zm_vmult_launch_k<1>(ctx, level, prec, a)) return;
  if (ctx.cfg.degree == 2 && zm_vmult_launch_k<2>(ctx, level, prec, a)) return;
  switch (ctx.cfg.degree) {
    case 1: vmult_launch_k<1>(ctx, level, prec, a); break;
    case 2: vmult_launch_k<2>(ctx, level, prec, a); break;
    case 3: vmult_launch_k<3>(ctx, level, prec, a); break;
    case 4: vmult_launch_k<4>(ctx, level, prec, a); break;
    case 5: vmult_launch_k<5>(ctx, level, prec, a); break;
    case 6: vmult_launch_k<6>(ctx, level, prec, a); break;
    case 7: vmult_launch_k<7>(ctx, level, prec, a); break;
    default: throw std::invalid_argument("degree not supported by the vmult kernel (1..7)");
  }
}

void launch_vmult(Context& ctx, int level, int prec, void* y, const void* x, const void* b) {
  const int m = ctx.dev[0][level].lay.m;
  launch_vmult_args(ctx, level, prec, VmultArgs{y, x, b, false, 0, m, 0, m});
}

void launch_vmult_args_public(Context& ctx, int level, int prec, void* y, const void* x, const void* b, int zlo,
                              int zhi, int c0, int c1) {
  launch_vmult_args(ctx, level, prec, VmultArgs{y, x, b, true, zlo, zhi, c0, c1});
}

void launch_vmult_zrange(Context& ctx, int level, int prec, void* y, const void* x, const void* b, int z0, int z1) {
  const int m = ctx.dev[0][level].lay.m;
  launch_vmult_args(ctx, level, prec, VmultArgs{y, x, b, false, 0, m, z0, z1});
}

void launch_vmult_slab(Context& ctx, int level, int prec, void* y, const void* x, const void* b, int z0, int z1) {
  const int m = ctx.dev[0][level].lay.m;
  launch_vmult_args(ctx, level, prec, VmultArgs{y, x, b, true, std::max(z0 - 1, 0), std::min(z1 + 1, m), z0, z1});
}

}  // namespace smg
