// stokesmg_b200.hpp — C++ host side of the B200 hot path, behind the reference's operator / smoother /
// transfer interfaces. Header-only over the C ABI (include/smg_b200.h); no CUDA or torch types here.
//
// The reference defines these operations in SPEC.md (modules stokes_op, smoother, multigrid, solver)
// on BlockVector<dim,T> (proj/include/stokesmg/block_vector.hpp:15-93), signals errors with
// std::invalid_argument (mesh.hpp:31-34, fem1d.hpp:95-96) and drives them from v_cycle / fgmres
// (SPEC.md:459-467, 507-533). This header gives the same shapes:
//   StokesOperator<T>::vmult(dst, src)            apply_stokes
//   StokesOperator<T>::residual(r, b, x)          r = b - A x
//   VertexPatchSmoother<T>::smooth(x, b, zero)    smooth
//   Transfer<T>::prolongate_add / restrict        prolongate / restrict SPEC.md:441-458
//   MGPreconditioner<T>::vmult(x, b)              v_cycle
//   solve_mixed(...)                              fgmres + solve_mixed SPEC.md:507-533
// Vectors are either DeviceVector<T> (HBM-resident, the fast path) or any BlockVector-like type with
// `velocity[c]` and `pressure` std::vector members (the reference's stokesmg::BlockVector<3,T> fits
// as is); BlockVector pressure uses the DoFLayout cell-local numbering.
// A context is not re-entrant: one host thread per Context.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/smg_b200.h"

namespace stokesmg {
namespace b200 {

struct not_converged : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc, const smg_context* ctx) {
  if (rc == SMG_OK) return;
  const std::string msg = smg_last_error(ctx);
  if (rc == SMG_EINVAL) throw std::invalid_argument(msg);  // the reference's error type
  if (rc == SMG_ENOTCONV) throw not_converged(msg);
  if (rc == SMG_ENOMEM) throw std::bad_alloc();
  throw std::runtime_error("smg_b200 error " + std::to_string(rc) + ": " + msg);
}

template <class T>
constexpr int precision_of() {
  static_assert(std::is_same<T, double>::value || std::is_same<T, float>::value, "T must be double or float");
  return std::is_same<T, double>::value ? SMG_F64 : SMG_F32;
}

struct CgOptions {
  int max_iter = 30;     // patch Schur-CG cap
  double tol = 1e-8;     // relative tolerance
  bool fixed = false;    // exactly max_iter iterations (parity mode)
  bool precond = true;   // pressure-mass preconditioned inner CG
};

// One GPU context for a mesh hierarchy (build_hierarchy mesh.hpp:30-36 + all per-level setup).
class Context {
 public:
  Context(int degree, int max_level, int device = 0, CgOptions cg = {}) {
    smg_config cfg;
    smg_config_default(&cfg);
    cfg.degree = degree;
    cfg.max_level = max_level;
    cfg.device = device;
    cfg.cg_max_iter = cg.max_iter;
    cfg.cg_tol = cg.tol;
    cfg.cg_fixed = cg.fixed ? 1 : 0;
    cfg.cg_precond = cg.precond ? 1 : 0;
    check(smg_create(&cfg, &h_), nullptr);
    degree_ = degree;
    max_level_ = max_level;
  }
  ~Context() {
    if (h_) smg_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  smg_context* handle() const { return h_; }
  int degree() const { return degree_; }
  int max_level() const { return max_level_; }
  void set_stream(void* cuda_stream) { check(smg_set_stream(h_, cuda_stream), h_); }
  // block sizes of a level: [u_x, u_y, u_z, p, total] (BlockVector::resize arguments)
  std::vector<int64_t> sizes(int level) const {
    int64_t s[5];
    check(smg_level_sizes(degree_, level, s), h_);
    return std::vector<int64_t>(s, s + 5);
  }
  int64_t launches() const { return smg_launch_count(h_); }

 private:
  smg_context* h_ = nullptr;
  int degree_ = 0, max_level_ = 0;
};

// A level vector resident in HBM, stored layout [u_x | u_y | u_z | p].
template <class T>
class DeviceVector {
 public:
  DeviceVector(Context& ctx, int level) : ctx_(&ctx), level_(level) {
    check(smg_vec_alloc(ctx.handle(), level, precision_of<T>(), &ptr_), ctx.handle());
  }
  ~DeviceVector() {
    if (ptr_) smg_vec_free(ctx_->handle(), ptr_);
  }
  DeviceVector(DeviceVector&& o) noexcept : ctx_(o.ctx_), level_(o.level_), ptr_(std::exchange(o.ptr_, nullptr)) {}
  DeviceVector(const DeviceVector&) = delete;
  DeviceVector& operator=(const DeviceVector&) = delete;
  void* data() { return ptr_; }
  const void* data() const { return ptr_; }
  int level() const { return level_; }
  Context& context() const { return *ctx_; }

  // BlockVector <-> device (block_vector.hpp:17-18 layout, cell-local pressure)
  template <class BV>
  void upload(const BV& src) {
    const void* vel[3] = {src.velocity[0].data(), src.velocity[1].data(), src.velocity[2].data()};
    check_sizes(src);
    check(smg_vec_upload(ctx_->handle(), level_, precision_of<T>(), ptr_, vel, src.pressure.data()), ctx_->handle());
  }
  template <class BV>
  void download(BV& dst) const {
    resize_blocks(*ctx_, level_, dst);
    void* vel[3] = {dst.velocity[0].data(), dst.velocity[1].data(), dst.velocity[2].data()};
    check(smg_vec_download(ctx_->handle(), level_, precision_of<T>(), vel, dst.pressure.data(), ptr_),
          ctx_->handle());
  }
  double dot(const DeviceVector& o) const {  // fp64 accumulation (block_vector.hpp:53-61)
    double r = 0.0;
    check(smg_dot(ctx_->handle(), level_, precision_of<T>(), ptr_, o.ptr_, &r), ctx_->handle());
    return r;
  }
  void axpy(double alpha, const DeviceVector& x) {  // this += alpha x
    check(smg_axpy(ctx_->handle(), level_, precision_of<T>(), alpha, x.ptr_, ptr_), ctx_->handle());
  }
  template <class U>
  void copy_from(const DeviceVector<U>& o) {  // BlockVector::copy_from<U> (block_vector.hpp:39-49)
    check(smg_convert(ctx_->handle(), level_, precision_of<T>(), ptr_, precision_of<U>(), o.data()), ctx_->handle());
  }

  template <class BV>
  static void resize_blocks(const Context& ctx, int level, BV& v) {
    const std::vector<int64_t> s = ctx.sizes(level);
    for (int c = 0; c < 3; ++c) v.velocity[c].assign(static_cast<size_t>(s[c]), 0);
    v.pressure.assign(static_cast<size_t>(s[3]), 0);
  }

 private:
  template <class BV>
  void check_sizes(const BV& v) const {
    const std::vector<int64_t> s = ctx_->sizes(level_);
    for (int c = 0; c < 3; ++c)
      if (static_cast<int64_t>(v.velocity[c].size()) != s[c]) throw std::invalid_argument("velocity block size mismatch");
    if (static_cast<int64_t>(v.pressure.size()) != s[3]) throw std::invalid_argument("pressure block size mismatch");
  }
  Context* ctx_;
  int level_;
  void* ptr_ = nullptr;
};

// y = A x with A = [[A, B^T], [B, 0]] (apply_stokes).
template <class T>
class StokesOperator {
 public:
  StokesOperator(Context& ctx, int level) : ctx_(&ctx), level_(level) {}
  void vmult(DeviceVector<T>& dst, const DeviceVector<T>& src) const {
    check(smg_vmult(ctx_->handle(), level_, precision_of<T>(), dst.data(), src.data()), ctx_->handle());
  }
  void residual(DeviceVector<T>& r, const DeviceVector<T>& b, const DeviceVector<T>& x) const {
    check(smg_residual(ctx_->handle(), level_, precision_of<T>(), r.data(), b.data(), x.data()), ctx_->handle());
  }
  // host BlockVector path (copies included): drop-in for a CPU operator's vmult(BlockVector&, const BlockVector&)
  template <class BV>
  void vmult(BV& dst, const BV& src) const {
    DeviceVector<T>::resize_blocks(*ctx_, level_, dst);
    const void* xv[3] = {src.velocity[0].data(), src.velocity[1].data(), src.velocity[2].data()};
    void* yv[3] = {dst.velocity[0].data(), dst.velocity[1].data(), dst.velocity[2].data()};
    check(smg_vmult_host(ctx_->handle(), level_, precision_of<T>(), yv, dst.pressure.data(), xv, src.pressure.data()),
          ctx_->handle());
  }
  int level() const { return level_; }

 private:
  Context* ctx_;
  int level_;
};

// One multiplicative vertex-patch smoothing step (smooth SPEC.md:400-408).
template <class T>
class VertexPatchSmoother {
 public:
  VertexPatchSmoother(Context& ctx, int level) : ctx_(&ctx), level_(level) {}
  void smooth(DeviceVector<T>& x, const DeviceVector<T>& b, bool zero_init = false) const {
    check(smg_smooth(ctx_->handle(), level_, precision_of<T>(), x.data(), b.data(), zero_init ? 1 : 0), ctx_->handle());
  }

 private:
  Context* ctx_;
  int level_;
};

// Intergrid transfer between coarse_level and coarse_level + 1.
template <class T>
class Transfer {
 public:
  explicit Transfer(Context& ctx) : ctx_(&ctx) {}
  void prolongate_add(int coarse_level, DeviceVector<T>& fine, const DeviceVector<T>& coarse) const {
    check(smg_prolongate_add(ctx_->handle(), coarse_level, precision_of<T>(), fine.data(), coarse.data()),
          ctx_->handle());
  }
  void restrict_down(int coarse_level, DeviceVector<T>& coarse, const DeviceVector<T>& fine) const {
    check(smg_restrict(ctx_->handle(), coarse_level, precision_of<T>(), coarse.data(), fine.data()), ctx_->handle());
  }

 private:
  Context* ctx_;
};

// V-cycle preconditioner (v_cycle SPEC.md:459-467): x = V(b), zero initial guess.
template <class T>
class MGPreconditioner {
 public:
  MGPreconditioner(Context& ctx, int level) : ctx_(&ctx), level_(level) {}
  void vmult(DeviceVector<T>& x, const DeviceVector<T>& b) const {
    check(smg_vcycle(ctx_->handle(), level_, precision_of<T>(), x.data(), b.data()), ctx_->handle());
  }

 private:
  Context* ctx_;
  int level_;
};

struct SolveResult {
  int iterations = 0;
  std::vector<double> history;  // residual norms, history[0] = ||b||
};

// Right-preconditioned FGMRES on the fp64 operator with the V-cycle in fp32 (mixed)
// or fp64. Throws not_converged if rel_tol is not reached within max_iter.
inline SolveResult solve_mixed(Context& ctx, int level, DeviceVector<double>& x, const DeviceVector<double>& b,
                               double rel_tol, int max_iter, bool fp32_vcycle = true) {
  SolveResult r;
  r.history.assign(static_cast<size_t>(max_iter) + 1, 0.0);
  const int rc = smg_solve(ctx.handle(), level, x.data(), b.data(), rel_tol, max_iter, fp32_vcycle ? SMG_F32 : SMG_F64,
                           &r.iterations, r.history.data());
  r.history.resize(static_cast<size_t>(r.iterations) + 1);
  check(rc, ctx.handle());
  return r;
}

// ---- multi-GPU: one Context per GPU / rank over the C ABI's z-slab driver (smg_dist_*) ----
// The reference's seams for a partitioned mesh: DistOperator::vmult is apply_A of
// fgmres(apply_A, apply_P, ...), DistContext::vcycle is apply_P (v_cycle SPEC.md:459-467)
// and DistContext::solve runs the whole MG-preconditioned FGMRES over the slabs. Vectors are device
// buffers in the held layout (held() sizes: owned cells + 3 ghost layers per interior side).
class DistContext {
 public:
  // NCCL transport: rank 0 calls nccl_unique_id() and the caller distributes the 128 bytes
  static std::vector<char> nccl_unique_id() {
    std::vector<char> id(128);
    check(smg_nccl_unique_id(id.data()), nullptr);
    return id;
  }
  DistContext(Context& ctx, const std::vector<char>& nccl_id, int nranks, int rank) : ctx_(&ctx) {
    if (nccl_id.size() != 128) throw std::invalid_argument("NCCL unique id must be 128 bytes");
    check(smg_dist_init_nccl(ctx.handle(), nccl_id.data(), nranks, rank), ctx.handle());
  }
  // caller transport (MPI, a shared-memory mailbox, ...); `t` must stay valid while the context lives
  DistContext(Context& ctx, const smg_transport& t, int nranks, int rank) : ctx_(&ctx) {
    check(smg_dist_init_transport(ctx.handle(), &t, nranks, rank), ctx.handle());
  }
  struct Held {
    int z0, z1, zlo, zhi;        // owned and held cells
    std::vector<int64_t> sizes;  // block sizes of the held layout + total
  };
  Held held(int level) const {
    int cells[4];
    int64_t s[5];
    check(smg_dist_held(ctx_->handle(), level, cells, s), ctx_->handle());
    return Held{cells[0], cells[1], cells[2], cells[3], std::vector<int64_t>(s, s + 5)};
  }
  template <class T>
  void vmult(int level, void* y, void* x) const {
    check(smg_dist_vmult(ctx_->handle(), level, precision_of<T>(), y, x), ctx_->handle());
  }
  template <class T>
  void vcycle(void* x, const void* b) const {
    check(smg_dist_vcycle(ctx_->handle(), precision_of<T>(), x, b), ctx_->handle());
  }
  SolveResult solve(void* x, const void* b, double rel_tol, int max_iter, bool fp32_vcycle = true) const {
    SolveResult r;
    r.history.assign(static_cast<size_t>(max_iter) + 1, 0.0);
    const int rc = smg_dist_solve(ctx_->handle(), x, b, rel_tol, max_iter, fp32_vcycle ? SMG_F32 : SMG_F64,
                                  &r.iterations, r.history.data());
    r.history.resize(static_cast<size_t>(r.iterations) + 1);
    check(rc, ctx_->handle());
    return r;
  }

 private:
  Context* ctx_;
};

}  // namespace b200
}  // namespace stokesmg
