// Internal declarations shared by the CUDA translation units of libsmg_b200.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <set>
#include <new>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/smg_b200.h"
#include "setup1d.hpp"

namespace smg {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct not_converged : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define SMG_CUDA(call)                                                                             \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      throw ::smg::cuda_error(std::string(#call) + ": " + cudaGetErrorString(e_));                \
  } while (0)

// Stored layout of one level vector.
// A z-slab holds the cells [zlo, zhi) of the level (the whole level: [0, m)); each block keeps the
// global x/y extents and the node planes of those cells (u_z: planes zlo*H .. zhi*H inclusive).
struct LevelLayout {
  int k = 0, level = 0, m = 0, n = 0;
  int zlo = 0, zhi = 0;
  int64_t dims[3][3]{};  // dims[c][axis] of the held part
  int64_t plane[4]{};    // elements per z node plane of each block
  int64_t off[4]{};
  int64_t size[4]{};
  int64_t total = 0;
  LevelLayout() = default;
  LevelLayout(int kk, int lvl) : LevelLayout(kk, lvl, 0, 2 << lvl) {}
  LevelLayout(int kk, int lvl, int z_lo, int z_hi) : k(kk), level(lvl), zlo(z_lo), zhi(z_hi) {
    if (kk < 1) throw std::invalid_argument("degree must be >= 1");
    if (lvl < 0 || lvl > 12) throw std::invalid_argument("level out of range");
    m = 2 << lvl;
    n = m * (k + 1);
    if (zlo < 0 || zhi > m || zlo >= zhi) throw std::invalid_argument("slab cell range out of range");
    const int64_t nz = static_cast<int64_t>(zhi - zlo) * (k + 1);
    int64_t o = 0;
    for (int c = 0; c < 3; ++c) {
      for (int a = 0; a < 2; ++a) dims[c][a] = a == c ? n + 1 : n;
      dims[c][2] = c == 2 ? nz + 1 : nz;
      plane[c] = dims[c][0] * dims[c][1];
      off[c] = o;
      size[c] = dims[c][0] * dims[c][1] * dims[c][2];
      o += size[c];
    }
    off[3] = o;
    plane[3] = static_cast<int64_t>(n) * n;
    size[3] = plane[3] * nz;
    total = o + size[3];
  }
};

// operator launch on a (slab) level vector: held cells [zlo, zhi), owned (computed) cells [z0, z1)
struct VmultArgs {
  void* y;
  const void* x;
  const void* b;  // residual r = b - A x if not null
  bool slab;
  int zlo, zhi, z0, z1;
};

// Device-resident constant data of one level in one precision.
struct DevLevel {
  LevelLayout lay;
  void* ops = nullptr;      // N_OPS x 9 x (k+1) x (k+2) operator blocks
  void* patch = nullptr;    // packed patch tables (smoother)
  void* transfer = nullptr; // packed embedding tables (this level as the fine level)
  void* pweights = nullptr; // pressure node weights (k+1)
};

// A tensor map depends on the vector's address AND its layout (level, precision, held cells): the
// allocator may hand the same address to a vector of another layout, so all of them are in the key.
struct TmapKey {
  const void* ptr;
  int level, esize, zlo, zhi;
  bool operator<(const TmapKey& o) const {
    if (ptr != o.ptr) return ptr < o.ptr;
    if (level != o.level) return level < o.level;
    if (esize != o.esize) return esize < o.esize;
    if (zlo != o.zlo) return zlo < o.zlo;
    return zhi < o.zhi;
  }
};

struct DistState;                // dist.cu: z-slab multi-GPU state
void dist_destroy(DistState* d);

struct Context {
  smg_config cfg{};
  int device = 0;
  bool device_ready = false;  // set once smg_create validated the device: every entry point then pins it
  int num_sms = 0;            // SM count of `device` (persistent grids)
  cudaStream_t stream = nullptr;
  std::string last_error;
  int64_t launches = 0;
  std::vector<LevelTables> tables;      // per level
  std::vector<PatchTables> ptables;     // per level
  TransferTables ttab;
  std::vector<DevLevel> dev[2];         // [precision][level]
  // coarse solve: dense pseudo-inverse on the free DoFs of level 0
  std::vector<int64_t> coarse_free;
  void* coarse_pinv[2] = {nullptr, nullptr};
  void* coarse_free_dev = nullptr;
  // scratch
  void* dot_partials = nullptr;  // double[kDotBlocks]
  void* dot_host = nullptr;      // pinned double[kDotBlocks]
  void* smoother_stats = nullptr;  // unsigned long long[2]: patches solved, inner CG iterations
  void* multidot_partials = nullptr;  // double[kDotBlocks]: batched Gram-Schmidt partial sums
  void* krylov_ptrs = nullptr;        // device array of the Krylov basis pointers (kMaxKrylov)
  void* krylov_coef = nullptr;        // device double[3 kMaxKrylov]: h1 | h2 | norm^2 of an iteration
  double* krylov_host = nullptr;      // pinned mirror of krylov_coef
  std::vector<void*> allocations;
  // per-level work vectors for the smoother / V-cycle (allocated lazily): [prec][level]
  std::vector<void*> work_r[2], work_x[2], work_b[2];
  std::vector<void*> krylov;  // FGMRES basis pool (fp64, finest-level size)
  void* pstage[2] = {nullptr, nullptr};
  void* pstage_out[2] = {nullptr, nullptr};
  cudaStream_t s_capture = nullptr;  // private stream for CUDA-graph capture
  cudaStream_t s_in = nullptr, s_out = nullptr;  // host-path copy streams (created on first use)  // pressure staging for the BlockVector host path (finest level size)
  // TMA descriptors of input vectors (vmult.cu)
  void* tmap_dev = nullptr;
  std::map<TmapKey, int> tmap_slots;
  int tmap_next = 0;
  std::vector<bool> tmap_pinned;  // slots referenced by captured CUDA graphs: never recycled
  bool tmap_recording = false;    // during a graph capture: collect the slots the captured kernels use
  std::set<int> tmap_recorded;
  // captured V-cycle graphs: [prec][level] (smg_solve, fixed work-vector pointers)
  std::vector<cudaGraphExec_t> vgraph[2];
  std::vector<int64_t> vgraph_launches[2];
  DistState* dist = nullptr;  // multi-GPU set-up (smg_dist_init_*), owned
  void* dist_pw = nullptr;    // pressure node weights of the finest level (distributed mean projection)
  ~Context();
};

constexpr int kDotBlocks = 1184;  // 8 x 148 SMs
constexpr int kMaxKrylov = 256;   // FGMRES basis vectors per solve (max_iter + 1)
constexpr int kTmapSlots = 64;         // cached TMA descriptor sets (global memory)
constexpr int kTmapSlotBytes = 1024;   // up to 8 CUtensorMap (128 B each)

size_t elem_size(int precision);

// raise a kernel's dynamic shared-memory limit once per (device, kernel, size); thread-safe. The
// attribute is per device, so a process-wide "done" flag would skip it for a second device.
void ensure_smem_attr(const void* kernel, int device, size_t bytes);

// level-0 pseudo-inverse from the bordered (nf+1)^2 system K on the device (coarse.cu): fp64 and fp32
// nf x nf copies, owned by the context
void coarse_inverse_device(Context& c, const Dense& K, int nf, void** pinv64, void** pinv32);

void upload_reference_tables();  // __constant__ reference-cell blocks (vmult.cu)

// ---- launchers (stream-ordered) ----
void launch_vmult(Context& c, int level, int prec, void* y, const void* x, const void* b /*residual if !null*/);
// z-slab operator: x, y (, b) hold the cells [max(z0-1,0), min(z1+1,m)) in the slab layout; computes
// the rows of the owned cells [z0, z1) (ghost layers must be current in x)
void launch_vmult_slab(Context& c, int level, int prec, void* y, const void* x, const void* b, int z0, int z1);
// operator (residual if b) rows of the cells [c0, c1) on vectors holding the cells [zlo, zhi)
void launch_vmult_args_public(Context& c, int level, int prec, void* y, const void* x, const void* b, int zlo, int zhi,
                              int c0, int c1);
// operator rows of the cells [z0, z1) of a whole-level vector (bricks restricted to that z range)
void launch_vmult_zrange(Context& c, int level, int prec, void* y, const void* x, const void* b, int z0, int z1);
void launch_smooth_colour(Context& c, int level, int prec, int colour, void* x, const void* r);
// fused halo-residual colour (k <= 3): x_out (holding a copy of x_in) += corrections from b - A x_in
void launch_smooth_colour_fused(Context& c, int level, int prec, int colour, void* x_out, const void* x_in,
                                const void* b);
// one colour on vectors holding the cells [zlo, zhi): patches with vertex z planes in [vz0, vz1]
void launch_smooth_colour_held(Context& c, int level, int prec, int colour, void* x, const void* r, int zlo, int zhi,
                               int vz0, int vz1);
void launch_prolongate_add(Context& c, int coarse_level, int prec, void* xf, const void* xc);
void launch_restrict(Context& c, int coarse_level, int prec, void* rc, const void* rf);
// z-slab transfers: fine vectors hold fine cells [fzlo, fzhi), coarse [czlo, czhi); prolongation adds
// into the rows of fine cells [r0, r1), restriction writes the rows of coarse cells [r0, r1)
void launch_prolongate_add_held(Context& c, int coarse_level, int prec, void* xf, const void* xc, int fzlo, int fzhi,
                                int czlo, int czhi, int r0, int r1);
void launch_restrict_held(Context& c, int coarse_level, int prec, void* rc, const void* rf, int fzlo, int fzhi, int czlo,
                          int czhi, int r0, int r1);
void launch_coarse_apply(Context& c, int prec, void* x, const void* b);
double dot(Context& c, int64_t n, int prec, const void* a, const void* b);
double dot_ranges(Context& c, int prec, const void* a, const void* b, const int64_t* begin, const int64_t* len,
                  int nranges);
void launch_axpy(Context& c, int64_t n, int prec, double alpha, const void* x, void* y);
void launch_axpby(Context& c, int64_t n, int prec, double alpha, const void* x, double beta, void* y);
void launch_convert(Context& c, int64_t n, int dst_prec, void* dst, int src_prec, const void* src);
void launch_zero(Context& c, int64_t n, int prec, void* x);
void launch_scale(Context& c, int64_t n, int prec, double alpha, void* x);
void launch_add_scalar(Context& c, int64_t n, int prec, double alpha, void* x);  // x += alpha
// out_dev[i] = <V_i, w>, i < nv (fp64; V_dev: device array of nv device pointers); one launch pair
void launch_multidot(Context& c, int64_t n, const double* const* V_dev, int nv, const double* w, double* out_dev);
// w -= sum_i coef_dev[i] V_i
void launch_multi_axpy(Context& c, int64_t n, const double* const* V_dev, int nv, const double* coef_dev, double* w);
void launch_sub_pressure_mean(Context& c, int level, int prec, void* x);  // mass-weighted mean removal
// pressure block global lexicographic <-> cell-local (BlockVector / DoFLayout order)
void launch_pressure_permute(Context& c, int level, int prec, void* dst, const void* src, bool to_cell_local,
                             int z0 = 0, int z1 = -1, cudaStream_t stream = nullptr);

// next TMA descriptor slot (round robin over the unpinned slots); the caller re-keys it
inline int tmap_alloc_slot(Context& c) {
  if (c.tmap_pinned.size() != static_cast<size_t>(kTmapSlots)) c.tmap_pinned.assign(kTmapSlots, false);
  for (int tries = 0; tries < kTmapSlots; ++tries) {
    const int slot = c.tmap_next++ % kTmapSlots;
    if (!c.tmap_pinned[slot]) {
      for (auto e = c.tmap_slots.begin(); e != c.tmap_slots.end();)
        e = (e->second == slot) ? c.tmap_slots.erase(e) : std::next(e);
      return slot;
    }
  }
  throw std::runtime_error("all tensor-map slots are pinned by captured graphs");
}

// C-ABI plumbing shared by the entry-point files: map exceptions to status codes, pin the device
template <class F>
int guarded_call(smg_context* h, F&& f) {
  Context* c = reinterpret_cast<Context*>(h);
  try {
    if (c && c->device_ready) SMG_CUDA(cudaSetDevice(c->device));
    return f();
  } catch (const std::invalid_argument& e) {
    if (c) c->last_error = e.what();
    return SMG_EINVAL;
  } catch (const std::bad_alloc&) {
    if (c) c->last_error = "out of memory";
    return SMG_ENOMEM;
  } catch (const not_converged& e) {
    if (c) c->last_error = e.what();
    return SMG_ENOTCONV;
  } catch (const std::exception& e) {
    if (c) c->last_error = e.what();
    return SMG_ECUDA;
  }
}
inline Context& context_of(smg_context* h) {
  if (!h) throw std::invalid_argument("null context");
  return *reinterpret_cast<Context*>(h);
}

}  // namespace smg
