// C ABI of libsmg_b200.so (include/smg_b200.h): context setup, level vectors, operator / smoother /
// transfer entry points, and the caller side of the hot path — the V-cycle (v_cycle SPEC.md:459-467)
// and the mixed-precision flexible GMRES (fgmres / solve_mixed SPEC.md:507-533) — driving the sm_100a
// kernels from the host. No CPU fallback: every numeric operation runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <cstdlib>
#include <vector>
#include <mutex>
#include <set>
#include <tuple>

#include "smg_internal.cuh"

namespace smg {

std::vector<double> pack_patch_tables(const PatchTables& P);  // smoother.cu

namespace {

void* dev_upload(Context& c, const std::vector<double>& v, int prec) {
  void* d = nullptr;
  const size_t n = v.size();
  SMG_CUDA(cudaMalloc(&d, std::max<size_t>(n, 1) * elem_size(prec)));
  c.allocations.push_back(d);
  if (prec == SMG_F64) {
    SMG_CUDA(cudaMemcpy(d, v.data(), n * 8, cudaMemcpyHostToDevice));
  } else {
    std::vector<float> f(v.begin(), v.end());
    SMG_CUDA(cudaMemcpy(d, f.data(), n * 4, cudaMemcpyHostToDevice));
  }
  return d;
}

// Dense global 1D operator (rows x cols) from the cell-row blocks of LevelTables.
Dense global1d(const LevelTables& T, int op, bool par_rows, bool par_cols) {
  const int H = T.k + 1, n = T.m * H;
  const int rows = par_rows ? n + 1 : n, cols = par_cols ? n + 1 : n;
  const int nb = par_cols ? H + 1 : H;
  Dense A(rows, cols);
  LevelTables& W = const_cast<LevelTables&>(T);
  for (int e = 0; e < T.m; ++e) {
    const int var = e == 0 ? 0 : (e == T.m - 1 ? 2 : 1);
    for (int d = -1; d <= 1; ++d) {
      if (e + d < 0 || e + d >= T.m) continue;
      for (int a = 0; a < H; ++a)
        for (int b = 0; b < nb; ++b) A(e * H + a, (e + d) * H + b) += W.w(op, var, d, a, b);
    }
  }
  return A;
}

// Level-0 pseudo-inverse (coarse_solve SPEC.md:468-476): dense A_0 on the free DoFs from the
// Kronecker factors, then the leading block of the inverse of [[A, e],[e^T, 0]] with e the constant
// pressure vector — equal to A^+ for symmetric A with ker A = span(e).
void setup_coarse(Context& c) {
  if (c.coarse_pinv[0]) return;  // built on first use (dense inverse of the level-0 system)
  const LevelTables& T = c.tables[0];
  const LevelLayout lay(c.cfg.degree, 0);
  const int n = lay.n;
  const Dense MO = global1d(T, OP_MO, false, false), LO = global1d(T, OP_LO, false, false);
  const Dense MP = global1d(T, OP_MP, true, true), LP = global1d(T, OP_LP, true, true);
  const Dense D = global1d(T, OP_D, false, true);  // n x (n+1)
  std::vector<int64_t> fr;
  for (int comp = 0; comp < 3; ++comp)
    for (int64_t z = 0; z < lay.dims[comp][2]; ++z)
      for (int64_t y = 0; y < lay.dims[comp][1]; ++y)
        for (int64_t x = 0; x < lay.dims[comp][0]; ++x) {
          const int64_t g[3] = {x, y, z};
          if (g[comp] == 0 || g[comp] == n) continue;
          fr.push_back(lay.off[comp] + (z * lay.dims[comp][1] + y) * lay.dims[comp][0] + x);
        }
  for (int64_t i = 0; i < lay.size[3]; ++i) fr.push_back(lay.off[3] + i);
  const int nf = static_cast<int>(fr.size());
  // decode stored index -> (block, coords)
  auto decode = [&](int64_t idx, int& blk, int* g) {
    blk = 3;
    for (int b = 0; b < 3; ++b)
      if (idx >= lay.off[b] && idx < lay.off[b + 1]) blk = b;
    const int64_t l = idx - lay.off[blk];
    const int64_t d0 = blk < 3 ? lay.dims[blk][0] : n, d1 = blk < 3 ? lay.dims[blk][1] : n;
    g[0] = static_cast<int>(l % d0);
    g[1] = static_cast<int>((l / d0) % d1);
    g[2] = static_cast<int>(l / (d0 * d1));
  };
  Dense K(nf + 1, nf + 1);
  std::vector<int> blk(nf);
  std::vector<int> co(3 * nf);
  for (int i = 0; i < nf; ++i) decode(fr[i], blk[i], &co[3 * i]);
  const int band = 2 * (c.cfg.degree + 1) + 1;  // every 1D factor vanishes beyond one neighbour cell
#pragma omp parallel for schedule(dynamic, 64)
  for (int i = 0; i < nf; ++i)
    for (int j = 0; j < nf; ++j) {
      const int bi = blk[i], bj = blk[j];
      const int* gi = &co[3 * i];
      const int* gj = &co[3 * j];
      if (std::abs(gi[0] - gj[0]) > band || std::abs(gi[1] - gj[1]) > band || std::abs(gi[2] - gj[2]) > band) continue;
      double v = 0.0;
      if (bi < 3 && bj == bi) {
        // Kronecker sum: sum_d L_d (x) M_others, par factors along axis bi
        for (int d = 0; d < 3; ++d) {
          double t = 1.0;
          for (int a = 0; a < 3 && t != 0.0; ++a) {
            const bool par = (a == bi);
            const Dense& Mm = par ? MP : MO;
            const Dense& Ll = par ? LP : LO;
            t *= (a == d ? Ll : Mm)(gi[a], gj[a]);
          }
          v += t;
        }
      } else if (bi == 3 && bj < 3) {
        double t = 1.0;
        for (int a = 0; a < 3; ++a) t *= (a == bj ? D(gi[a], gj[a]) : MO(gi[a], gj[a]));
        v = t;
      } else if (bi < 3 && bj == 3) {
        double t = 1.0;
        for (int a = 0; a < 3; ++a) t *= (a == bi ? D(gj[a], gi[a]) : MO(gj[a], gi[a]));
        v = t;
      }
      K(i, j) = v;
    }
  for (int i = 0; i < nf; ++i)
    if (blk[i] == 3) K(i, nf) = K(nf, i) = 1.0;
  c.coarse_free = fr;
  coarse_inverse_device(c, K, nf, &c.coarse_pinv[0], &c.coarse_pinv[1]);
  void* d = nullptr;
  SMG_CUDA(cudaMalloc(&d, fr.size() * sizeof(int64_t)));
  c.allocations.push_back(d);
  SMG_CUDA(cudaMemcpy(d, fr.data(), fr.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  c.coarse_free_dev = d;
}

void* alloc_vec(Context& c, int level, int prec) {
  void* d = nullptr;
  SMG_CUDA(cudaMalloc(&d, c.dev[0][level].lay.total * elem_size(prec)));
  c.allocations.push_back(d);
  return d;
}

void ensure_work(Context& c, int prec) {
  if (!c.work_r[prec].empty()) return;
  const int L = c.cfg.max_level;
  c.work_r[prec].assign(L + 1, nullptr);
  c.work_x[prec].assign(L + 1, nullptr);
  c.work_b[prec].assign(L + 1, nullptr);
  for (int l = 0; l <= L; ++l) {
    c.work_r[prec][l] = alloc_vec(c, l, prec);
    c.work_x[prec][l] = alloc_vec(c, l, prec);
    c.work_b[prec][l] = alloc_vec(c, l, prec);
  }
}

void check_level(const Context& c, int level) {
  if (level < 0 || level > c.cfg.max_level) throw std::invalid_argument("level out of range");
}

// x_zero: x is known to be 0 (pre-smoothing on descent), so colour 0's residual is b itself
void smooth(Context& c, int level, int prec, void* x, const void* b, bool x_zero = false) {
  ensure_work(c, prec);
  if (c.cfg.smoother_fused && c.cfg.degree <= 3) {
    // fused halo residual: colour c reads the snapshot buf[c % 2] and writes buf[(c+1) % 2] (a copy of
    // the snapshot plus the colour's corrections) -- same-colour patches read each other's halos, so the
    // snapshot stays untouched; after the 8 colours the result is back in x
    void* buf[2] = {x, c.work_r[prec][level]};
    const size_t bytes = static_cast<size_t>(c.dev[0][level].lay.total) * elem_size(prec);
    for (int col = 0; col < 8; ++col) {
      SMG_CUDA(cudaMemcpyAsync(buf[(col + 1) & 1], buf[col & 1], bytes, cudaMemcpyDeviceToDevice, c.stream));
      launch_smooth_colour_fused(c, level, prec, col, buf[(col + 1) & 1], buf[col & 1], b);
    }
    return;
  }
  void* r = c.work_r[prec][level];
  for (int col = 0; col < 8; ++col) {
    if (col == 0 && x_zero) {  // r = b - A 0 on the patch rows (the gather reads patch DoFs only)
      launch_smooth_colour(c, level, prec, col, x, b);
      continue;
    }
    launch_vmult(c, level, prec, r, x, b);
    launch_smooth_colour(c, level, prec, col, x, r);
  }
}

void vcycle(Context& c, int level, int prec, void* x, const void* b) {
  if (level == 0) {
    setup_coarse(c);
    launch_coarse_apply(c, prec, x, b);
    return;
  }
  ensure_work(c, prec);
  const int64_t N = c.dev[0][level].lay.total;
  launch_zero(c, N, prec, x);
  smooth(c, level, prec, x, b, /*x_zero=*/true);
  void* r = c.work_r[prec][level];
  void* bc = c.work_b[prec][level - 1];
  void* xc = c.work_x[prec][level - 1];
  launch_vmult(c, level, prec, r, x, b);
  launch_restrict(c, level - 1, prec, bc, r);
  vcycle(c, level - 1, prec, xc, bc);
  launch_prolongate_add(c, level - 1, prec, x, xc);
  smooth(c, level, prec, x, b);
}

// V-cycle on the context's fixed work vectors (x = vx, b = vb of `level`) replayed from a CUDA graph:
// the ~36 launches per level (8 colours x (residual + patches) x 2 steps, transfers, coarse solve) are
// captured once per (level, precision) after a warm-up V-cycle has created every lazily built object
// (work vectors, coarse pseudo-inverse, TMA descriptors, whose slots are then pinned), and replayed
// with one cudaGraphLaunch. SMG_NO_GRAPH=1: plain launches.
void vcycle_graph(Context& c, int level, int prec, void* vx, const void* vb) {
  static const bool off = std::getenv("SMG_NO_GRAPH") != nullptr;
  const int L = c.cfg.max_level;
  if (c.vgraph[prec].empty()) {
    c.vgraph[prec].assign(L + 1, nullptr);
    c.vgraph_launches[prec].assign(L + 1, 0);
  }
  if (off) {
    vcycle(c, level, prec, vx, vb);
    return;
  }
  cudaGraphExec_t& ge = c.vgraph[prec][level];
  if (!ge) {
    vcycle(c, level, prec, vx, vb);  // warm-up: lazy set-up happens outside the capture
    SMG_CUDA(cudaStreamSynchronize(c.stream));
    // captured on a private stream (the caller's may be the legacy default stream, which cannot be
    // captured); the replay below is ordered on the caller's stream
    if (!c.s_capture) SMG_CUDA(cudaStreamCreateWithFlags(&c.s_capture, cudaStreamNonBlocking));
    const cudaStream_t user = c.stream;
    c.stream = c.s_capture;
    const int64_t l0 = c.launches;
    cudaGraph_t g = nullptr;
    c.tmap_recorded.clear();
    c.tmap_recording = true;
    SMG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      vcycle(c, level, prec, vx, vb);
    } catch (...) {
      cudaStreamEndCapture(c.stream, &g);
      if (g) cudaGraphDestroy(g);
      c.stream = user;
      c.tmap_recording = false;
      throw;
    }
    c.stream = user;
    c.tmap_recording = false;
    SMG_CUDA(cudaStreamEndCapture(c.s_capture, &g));
    SMG_CUDA(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    c.vgraph_launches[prec][level] = c.launches - l0;
    if (c.tmap_pinned.size() != static_cast<size_t>(kTmapSlots)) c.tmap_pinned.assign(kTmapSlots, false);
    for (int slot : c.tmap_recorded) c.tmap_pinned[slot] = true;  // the graph holds their addresses
    c.launches -= c.vgraph_launches[prec][level];  // counted on every replay
    // the warm-up cycle already produced this call's result (the capture executes nothing); order
    // the caller's stream after it and replay from the next call on
    cudaEvent_t done;
    SMG_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    SMG_CUDA(cudaEventRecord(done, c.s_capture));
    SMG_CUDA(cudaStreamWaitEvent(c.stream, done, 0));
    cudaEventDestroy(done);
    return;
  }
  SMG_CUDA(cudaGraphLaunch(ge, c.stream));
  c.launches += c.vgraph_launches[prec][level];
}

// FGMRES, right-preconditioned, no restart, x0 = 0; Gram-Schmidt twice per
// iteration as SPEC.md:550 asks (MGS + re-orthogonalisation with SMG_KRYLOV_MGS=1, else the batched
// classical form CGS2: one host sync per iteration instead of 2(j+1)+1); the V-cycle runs in `vp`
// precision with conversion at its boundary, replayed from a CUDA graph.
int fgmres(Context& c, int level, double* x, const double* b, double tol, int max_iter, int vp, int* iters,
           double* hist) {
  const int64_t N = c.dev[0][level].lay.total;
  std::vector<double*> V, Z;
  // Krylov basis vectors come from a per-context pool (finest-level size, grown on first use and
  // kept): no allocation inside the solve after the first call
  size_t used = 0;
  auto newvec = [&]() {
    if (used == c.krylov.size()) c.krylov.push_back(alloc_vec(c, c.cfg.max_level, SMG_F64));
    return static_cast<double*>(c.krylov[used++]);
  };
  void *vb = nullptr, *vx = nullptr;
  if (vp == SMG_F32) ensure_work(c, SMG_F32);
  std::vector<std::vector<double>> H(max_iter + 1, std::vector<double>(max_iter, 0.0));
  std::vector<double> cs(max_iter, 0.0), sn(max_iter, 0.0), g(max_iter + 1, 0.0);
  launch_zero(c, N, SMG_F64, x);
  const double beta = std::sqrt(dot(c, N, SMG_F64, b, b));
  if (hist) hist[0] = beta;
  int it = 0;
  if (beta == 0.0) {
    if (iters) *iters = 0;
    return SMG_OK;
  }
  if (max_iter + 1 >= kMaxKrylov) throw std::invalid_argument("max_iter exceeds the Krylov basis capacity (254)");
  static const bool mgs = std::getenv("SMG_KRYLOV_MGS") != nullptr;
  // basis vector i's pointer into the device pointer table (for the batched Gram-Schmidt kernels)
  auto publish = [&](int i, const double* p) {
    SMG_CUDA(cudaMemcpyAsync(static_cast<double**>(c.krylov_ptrs) + i, &p, sizeof(double*), cudaMemcpyHostToDevice,
                             c.stream));
  };
  V.push_back(newvec());
  launch_convert(c, N, SMG_F64, V[0], SMG_F64, b);
  launch_scale(c, N, SMG_F64, 1.0 / beta, V[0]);
  publish(0, V[0]);
  g[0] = beta;
  double* w = newvec();
  bool converged = false;
  for (; it < max_iter;) {
    const int j = it;
    Z.push_back(newvec());
    if (vp == SMG_F64) {
      vcycle(c, level, SMG_F64, Z[j], V[j]);
    } else {
      // fp64 -> fp32 at the V-cycle boundary; the top-level scratch of the fp32 hierarchy holds b and x
      vb = c.work_b[SMG_F32][level];
      vx = c.work_x[SMG_F32][level];
      launch_convert(c, N, SMG_F32, vb, SMG_F64, V[j]);
      vcycle_graph(c, level, SMG_F32, vx, vb);
      launch_convert(c, N, SMG_F64, Z[j], SMG_F32, vx);
    }
    launch_vmult(c, level, SMG_F64, w, Z[j], nullptr);
    double wn;
    if (mgs) {
      // SPEC-literal (SMG_KRYLOV_MGS=1): modified Gram-Schmidt + one re-orthogonalisation pass, one
      // host-synchronous dot per coefficient
      for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i <= j; ++i) {
          const double hij = dot(c, N, SMG_F64, w, V[i]);
          H[i][j] += hij;
          launch_axpy(c, N, SMG_F64, -hij, V[i], w);
        }
      wn = std::sqrt(dot(c, N, SMG_F64, w, w));
    } else {
      // classical Gram-Schmidt applied twice (CGS2): all coefficients of a pass in one batched dot,
      // the update in one kernel with the coefficients left on the device, one host sync per iteration
      const double* const* Vd = static_cast<const double* const*>(c.krylov_ptrs);
      double* coef = static_cast<double*>(c.krylov_coef);
      launch_multidot(c, N, Vd, j + 1, w, coef);
      launch_multi_axpy(c, N, Vd, j + 1, coef, w);
      launch_multidot(c, N, Vd, j + 1, w, coef + kMaxKrylov);
      launch_multi_axpy(c, N, Vd, j + 1, coef + kMaxKrylov, w);
      const double* wp = w;
      SMG_CUDA(cudaMemcpyAsync(static_cast<double**>(c.krylov_ptrs) + kMaxKrylov - 1, &wp, sizeof(double*),
                               cudaMemcpyHostToDevice, c.stream));
      launch_multidot(c, N, Vd + kMaxKrylov - 1, 1, w, coef + 2 * kMaxKrylov);
      SMG_CUDA(cudaMemcpyAsync(c.krylov_host, coef, 3 * kMaxKrylov * sizeof(double), cudaMemcpyDeviceToHost,
                               c.stream));
      SMG_CUDA(cudaStreamSynchronize(c.stream));
      for (int i = 0; i <= j; ++i) H[i][j] = c.krylov_host[i] + c.krylov_host[kMaxKrylov + i];
      wn = std::sqrt(c.krylov_host[2 * kMaxKrylov]);
    }
    H[j + 1][j] = wn;
    for (int i = 0; i < j; ++i) {
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
    if (std::fabs(g[j + 1]) <= tol * beta || wn == 0.0) {
      converged = true;
      break;
    }
    V.push_back(newvec());
    launch_convert(c, N, SMG_F64, V.back(), SMG_F64, w);
    launch_scale(c, N, SMG_F64, 1.0 / wn, V.back());
    publish(static_cast<int>(V.size()) - 1, V.back());
  }
  std::vector<double> y(it, 0.0);
  for (int i = it - 1; i >= 0; --i) {
    double s = g[i];
    for (int l = i + 1; l < it; ++l) s -= H[i][l] * y[l];
    y[i] = s / H[i][i];
  }
  for (int i = 0; i < it; ++i) launch_axpy(c, N, SMG_F64, y[i], Z[i], x);
  launch_sub_pressure_mean(c, level, SMG_F64, x);
  SMG_CUDA(cudaStreamSynchronize(c.stream));
  if (iters) *iters = it;
  return converged ? SMG_OK : SMG_ENOTCONV;
}

// BlockVector (host, reference DoFLayout: pressure cell-local) <-> device level vector
// (stored layout, pressure global lexicographic). Velocity blocks are copied as they are; the
// pressure goes through a staging buffer and the permutation kernel. Stream-ordered, asynchronous
// with respect to the host for pinned buffers.
char* pressure_stage(Context& c, int prec) {
  if (!c.pstage[prec]) c.pstage[prec] = alloc_vec(c, c.cfg.max_level, prec);
  return static_cast<char*>(c.pstage[prec]);
}

void upload_blocks(Context& c, int level, int prec, char* dst, const void* const vel[3], const void* p) {
  const LevelLayout& lay = c.dev[0][level].lay;
  const size_t es = elem_size(prec);
  for (int b = 0; b < 3; ++b)
    SMG_CUDA(cudaMemcpyAsync(dst + lay.off[b] * es, vel[b], lay.size[b] * es, cudaMemcpyHostToDevice, c.stream));
  char* st = pressure_stage(c, prec);
  SMG_CUDA(cudaMemcpyAsync(st, p, lay.size[3] * es, cudaMemcpyHostToDevice, c.stream));
  launch_pressure_permute(c, level, prec, dst + lay.off[3] * es, st, false);
}

void download_blocks(Context& c, int level, int prec, void* const vel[3], void* p, const char* src) {
  const LevelLayout& lay = c.dev[0][level].lay;
  const size_t es = elem_size(prec);
  for (int b = 0; b < 3; ++b)
    SMG_CUDA(cudaMemcpyAsync(vel[b], src + lay.off[b] * es, lay.size[b] * es, cudaMemcpyDeviceToHost, c.stream));
  char* st = pressure_stage(c, prec);
  launch_pressure_permute(c, level, prec, st, src + lay.off[3] * es, true);
  SMG_CUDA(cudaMemcpyAsync(p, st, lay.size[3] * es, cudaMemcpyDeviceToHost, c.stream));
}

// Host BlockVector apply, pipelined over z-chunks of the level: chunk k's copy in
// (stream s_in: velocity planes + cell-local pressure, then the pressure permutation), the operator
// rows of chunk k once chunks k and k+1 are resident (context stream; the kernel's z range), and
// chunk k's copy out (stream s_out: pressure permutation back, then the copies) overlap, so the
// PCIe transfers in both directions and the compute run concurrently.
void vmult_host_pipelined(Context& c, int level, int prec, void* const y_vel[3], void* y_p, const void* const x_vel[3],
                          const void* x_p) {
  ensure_work(c, prec);
  const LevelLayout& lay = c.dev[0][level].lay;
  const size_t es = elem_size(prec);
  const int H = c.cfg.degree + 1;
  char* dx = static_cast<char*>(c.work_x[prec][level]);
  char* dy = static_cast<char*>(c.work_b[prec][level]);
  char* pin = pressure_stage(c, prec);
  if (!c.pstage_out[prec]) c.pstage_out[prec] = alloc_vec(c, c.cfg.max_level, prec);
  char* pout = static_cast<char*>(c.pstage_out[prec]);
  if (!c.s_in) {
    SMG_CUDA(cudaStreamCreateWithFlags(&c.s_in, cudaStreamNonBlocking));
    SMG_CUDA(cudaStreamCreateWithFlags(&c.s_out, cudaStreamNonBlocking));
  }
  // z-chunks of at least 2 cells (a chunk that is not a multiple of the kernel's brick depth runs a
  // masked partial brick); SMG_HOST_CHUNKS overrides the target count
  const int m = lay.m;
  int nch_target = 16;
  if (const char* e = std::getenv("SMG_HOST_CHUNKS")) nch_target = std::max(1, std::atoi(e));
  int chunk = std::max(2, m / nch_target);
  if (m < 8) chunk = m;
  const int nchunk = (m + chunk - 1) / chunk;
  std::vector<cudaEvent_t> ev_in(nchunk), ev_comp(nchunk);
  for (int k = 0; k < nchunk; ++k) {
    SMG_CUDA(cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming));
    SMG_CUDA(cudaEventCreateWithFlags(&ev_comp[k], cudaEventDisableTiming));
  }
  struct EvGuard {
    std::vector<cudaEvent_t>* a;
    std::vector<cudaEvent_t>* b;
    ~EvGuard() {
      for (auto e : *a) cudaEventDestroy(e);
      for (auto e : *b) cudaEventDestroy(e);
    }
  } guard{&ev_in, &ev_comp};
  cudaEvent_t start;
  SMG_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  SMG_CUDA(cudaEventRecord(start, c.stream));  // the copies are ordered after earlier work on the context stream
  SMG_CUDA(cudaStreamWaitEvent(c.s_in, start, 0));
  SMG_CUDA(cudaStreamWaitEvent(c.s_out, start, 0));
  cudaEventDestroy(start);
  // byte range [a, b) of block blk for the node planes of cells [z0, z1) (+ the top u_z plane at the end)
  auto span = [&](int blk, int z0, int z1, int64_t& off, int64_t& len) {
    const int64_t plane = blk == 3 ? static_cast<int64_t>(lay.n) * lay.n : lay.dims[blk][0] * lay.dims[blk][1];
    const int64_t p0 = static_cast<int64_t>(z0) * H, p1 = static_cast<int64_t>(z1) * H + (blk == 2 && z1 == m ? 1 : 0);
    off = p0 * plane;
    len = (p1 - p0) * plane;
  };
  for (int k = 0; k < nchunk; ++k) {
    const int z0 = k * chunk, z1 = std::min(m, z0 + chunk);
    for (int blk = 0; blk < 4; ++blk) {
      int64_t off, len;
      span(blk, z0, z1, off, len);
      const char* src = static_cast<const char*>(blk < 3 ? x_vel[blk] : x_p) + off * es;
      char* dst = (blk < 3 ? dx + lay.off[blk] * es : pin) + off * es;
      SMG_CUDA(cudaMemcpyAsync(dst, src, len * es, cudaMemcpyHostToDevice, c.s_in));
    }
    SMG_CUDA(cudaEventRecord(ev_in[k], c.s_in));
  }
  // the copy streams carry copies only (a kernel between two copies of one stream leaves the copy
  // engine idle); the pressure permutations run on the compute stream, one chunk ahead of the vmult
  auto permute_in = [&](int k) {
    const int z0 = k * chunk, z1 = std::min(m, z0 + chunk);
    SMG_CUDA(cudaStreamWaitEvent(c.stream, ev_in[k], 0));
    launch_pressure_permute(c, level, prec, dx + lay.off[3] * es, pin, false, z0, z1, c.stream);
  };
  permute_in(0);
  for (int k = 0; k < nchunk; ++k) {
    const int z0 = k * chunk, z1 = std::min(m, z0 + chunk);
    if (k + 1 < nchunk) permute_in(k + 1);
    launch_vmult_zrange(c, level, prec, dy, dx, nullptr, z0, z1);
    launch_pressure_permute(c, level, prec, pout, dy + lay.off[3] * es, true, z0, z1, c.stream);
    SMG_CUDA(cudaEventRecord(ev_comp[k], c.stream));
    SMG_CUDA(cudaStreamWaitEvent(c.s_out, ev_comp[k], 0));
    for (int blk = 0; blk < 4; ++blk) {
      int64_t off, len;
      span(blk, z0, z1, off, len);
      const char* src = (blk < 3 ? dy + lay.off[blk] * es : pout) + off * es;
      char* dst = static_cast<char*>(blk < 3 ? y_vel[blk] : y_p) + off * es;
      SMG_CUDA(cudaMemcpyAsync(dst, src, len * es, cudaMemcpyDeviceToHost, c.s_out));
    }
  }
  SMG_CUDA(cudaStreamSynchronize(c.s_out));
  SMG_CUDA(cudaStreamSynchronize(c.stream));
}

// launches and allocations go to the context's device whatever device the caller made current
template <class F>
int guarded(smg_context* h, F&& f) {
  return guarded_call(h, std::forward<F>(f));
}

}  // namespace

void ensure_smem_attr(const void* kernel, int device, size_t bytes) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, size_t>> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({device, kernel, bytes})) return;
  SMG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  done.insert({device, kernel, bytes});
}

namespace {

Context& ctx_of(smg_context* h) {
  if (!h) throw std::invalid_argument("null context");
  return *reinterpret_cast<Context*>(h);
}

void check_prec(int p) {
  if (p != SMG_F64 && p != SMG_F32) throw std::invalid_argument("precision must be SMG_F64 or SMG_F32");
}

}  // namespace

// entry points of the single-GPU V-cycle for the z-slab driver (dist.cu): the replicated coarse levels
void vcycle_level(Context& c, int level, int prec, void* x, const void* b) { vcycle(c, level, prec, x, b); }

Context::~Context() {
  if (dist) dist_destroy(dist);
  if (dist_pw) cudaFree(dist_pw);
  if (s_in) cudaStreamDestroy(s_in);
  if (s_out) cudaStreamDestroy(s_out);
  if (s_capture) cudaStreamDestroy(s_capture);
  for (void* p : allocations) cudaFree(p);
  if (dot_host) cudaFreeHost(dot_host);
  if (krylov_host) cudaFreeHost(krylov_host);
  for (auto& g : vgraph)
    for (cudaGraphExec_t e : g)
      if (e) cudaGraphExecDestroy(e);
}

}  // namespace smg

using smg::Context;

extern "C" {

int smg_config_default(smg_config* cfg) {
  if (!cfg) return SMG_EINVAL;
  cfg->degree = 2;
  cfg->max_level = 3;
  cfg->device = 0;
  cfg->cg_max_iter = 30;
  cfg->cg_tol = 1e-8;
  cfg->cg_fixed = 0;
  cfg->cg_precond = 1;
  cfg->smoother_fused = 0;
  return SMG_OK;
}

int smg_level_sizes(int degree, int level, int64_t sizes[5]) {
  try {
    smg::LevelLayout l(degree, level);
    for (int i = 0; i < 4; ++i) sizes[i] = l.size[i];
    sizes[4] = l.total;
    return SMG_OK;
  } catch (...) {
    return SMG_EINVAL;
  }
}

int smg_pressure_node_weights(int degree, double* w) {
  if (degree < 1 || degree > 7 || !w) return SMG_EINVAL;
  const auto v = smg::pressure_node_weights(degree);
  for (int a = 0; a <= degree; ++a) w[a] = v[a];
  return SMG_OK;
}

static thread_local std::string g_create_error;

int smg_create(const smg_config* cfg, smg_context** out) {
  if (!cfg || !out) return SMG_EINVAL;
  *out = nullptr;
  Context* c = new (std::nothrow) Context();
  if (!c) return SMG_ENOMEM;
  int rc = smg::guarded(reinterpret_cast<smg_context*>(c), [&] {
    if (cfg->degree < 1 || cfg->degree > 7) throw std::invalid_argument("degree must be in 1..7");
    if (cfg->max_level < 0 || cfg->max_level > 10) throw std::invalid_argument("max_level must be in 0..10");
    if (cfg->cg_max_iter < 0) throw std::invalid_argument("cg_max_iter must be >= 0");
    c->cfg = *cfg;
    int ndev = 0;
    SMG_CUDA(cudaGetDeviceCount(&ndev));
    if (cfg->device < 0 || cfg->device >= ndev) throw smg::cuda_error("no such CUDA device");
    SMG_CUDA(cudaSetDevice(cfg->device));
    cudaDeviceProp prop{};
    SMG_CUDA(cudaGetDeviceProperties(&prop, cfg->device));
    if (prop.major < 10) throw smg::cuda_error("libsmg_b200 needs an sm_100 (Blackwell) device");
    c->device = cfg->device;
    c->num_sms = prop.multiProcessorCount;
    smg::upload_reference_tables();
    const int L = cfg->max_level;
    c->ttab = smg::build_transfer_tables(cfg->degree);
    std::vector<double> ttab;
    for (double v : c->ttab.Ec.a) ttab.push_back(v);
    for (double v : c->ttab.Ed.a) ttab.push_back(v);
    for (int p = 0; p < 2; ++p) c->dev[p].resize(L + 1);
    for (int l = 0; l <= L; ++l) {
      c->tables.push_back(smg::build_level_tables(cfg->degree, l));
      c->ptables.push_back(smg::build_patch_tables(c->tables.back()));
      const auto packed = smg::pack_patch_tables(c->ptables.back());
      const auto pw = smg::pressure_node_weights(cfg->degree);
      for (int p = 0; p < 2; ++p) {
        smg::DevLevel& d = c->dev[p][l];
        d.lay = smg::LevelLayout(cfg->degree, l);
        d.ops = smg::dev_upload(*c, c->tables.back().ops, p);
        d.patch = smg::dev_upload(*c, packed, p);
        d.transfer = smg::dev_upload(*c, ttab, p);
        d.pweights = smg::dev_upload(*c, pw, SMG_F64);
      }
    }
    SMG_CUDA(cudaMalloc(&c->dot_partials, (smg::kDotBlocks + 8) * sizeof(double)));
    c->allocations.push_back(c->dot_partials);
    SMG_CUDA(cudaMallocHost(&c->dot_host, 64));
    SMG_CUDA(cudaMalloc(&c->multidot_partials, smg::kDotBlocks * sizeof(double)));
    c->allocations.push_back(c->multidot_partials);
    SMG_CUDA(cudaMalloc(&c->krylov_ptrs, smg::kMaxKrylov * sizeof(double*)));
    c->allocations.push_back(c->krylov_ptrs);
    SMG_CUDA(cudaMalloc(&c->krylov_coef, 3 * smg::kMaxKrylov * sizeof(double)));
    c->allocations.push_back(c->krylov_coef);
    SMG_CUDA(cudaMallocHost(&c->krylov_host, 3 * smg::kMaxKrylov * sizeof(double)));
    SMG_CUDA(cudaMalloc(&c->smoother_stats, 2 * sizeof(unsigned long long)));
    c->allocations.push_back(c->smoother_stats);
    SMG_CUDA(cudaMemset(c->smoother_stats, 0, 2 * sizeof(unsigned long long)));
    SMG_CUDA(cudaMalloc(&c->tmap_dev, static_cast<size_t>(smg::kTmapSlots) * smg::kTmapSlotBytes));
    c->allocations.push_back(c->tmap_dev);
    c->device_ready = true;
    return SMG_OK;
  });
  if (rc != SMG_OK) {
    g_create_error = c->last_error;
    delete c;
    return rc;
  }
  *out = reinterpret_cast<smg_context*>(c);
  return SMG_OK;
}

int smg_destroy(smg_context* h) {
  if (!h) return SMG_EINVAL;
  delete reinterpret_cast<Context*>(h);
  return SMG_OK;
}

int smg_set_stream(smg_context* h, void* stream) {
  return smg::guarded(h, [&] {
    smg::ctx_of(h).stream = static_cast<cudaStream_t>(stream);
    return SMG_OK;
  });
}

const char* smg_last_error(const smg_context* h) {
  if (!h) return g_create_error.c_str();
  return reinterpret_cast<const Context*>(h)->last_error.c_str();
}

int64_t smg_launch_count(const smg_context* h) { return h ? reinterpret_cast<const Context*>(h)->launches : -1; }

int smg_vec_alloc(smg_context* h, int level, int precision, void** dptr) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!dptr) throw std::invalid_argument("null output pointer");
    SMG_CUDA(cudaMalloc(dptr, c.dev[0][level].lay.total * smg::elem_size(precision)));
    SMG_CUDA(cudaMemset(*dptr, 0, c.dev[0][level].lay.total * smg::elem_size(precision)));
    return SMG_OK;
  });
}

int smg_vec_free(smg_context* h, void* dptr) {
  return smg::guarded(h, [&] {
    SMG_CUDA(cudaFree(dptr));
    return SMG_OK;
  });
}

int smg_vmult(smg_context* h, int level, int precision, void* y, const void* x) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!x || !y || x == y) throw std::invalid_argument("vmult: x and y must be distinct non-null vectors");
    smg::launch_vmult(c, level, precision, y, x, nullptr);
    return SMG_OK;
  });
}

int smg_residual(smg_context* h, int level, int precision, void* r, const void* b, const void* x) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!r || !b || !x || r == x || r == b) throw std::invalid_argument("residual: r must differ from b and x");
    smg::launch_vmult(c, level, precision, r, x, b);
    return SMG_OK;
  });
}

int smg_smooth(smg_context* h, int level, int precision, void* x, const void* b, int zero_init) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (level < 1) throw std::invalid_argument("smooth: level 0 uses the coarse solver (SPEC.md:71)");
    if (zero_init) smg::launch_zero(c, c.dev[0][level].lay.total, precision, x);
    smg::smooth(c, level, precision, x, b, zero_init != 0);
    return SMG_OK;
  });
}

int smg_prolongate_add(smg_context* h, int coarse_level, int precision, void* xf, const void* xc) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, coarse_level + 1);
    smg::check_prec(precision);
    smg::launch_prolongate_add(c, coarse_level, precision, xf, xc);
    return SMG_OK;
  });
}

int smg_restrict(smg_context* h, int coarse_level, int precision, void* rc, const void* rf) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, coarse_level + 1);
    smg::check_prec(precision);
    smg::launch_restrict(c, coarse_level, precision, rc, rf);
    return SMG_OK;
  });
}

int smg_coarse_solve(smg_context* h, int precision, void* x, const void* b) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_prec(precision);
    smg::setup_coarse(c);
    smg::launch_coarse_apply(c, precision, x, b);
    return SMG_OK;
  });
}

int smg_vcycle(smg_context* h, int level, int precision, void* x, const void* b) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    smg::vcycle(c, level, precision, x, b);
    return SMG_OK;
  });
}

int smg_solve(smg_context* h, int level, void* x, const void* b, double rel_tol, int max_iter, int vp, int* iters,
              double* history) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(vp);
    if (!(rel_tol > 0.0 && rel_tol < 1.0)) throw std::invalid_argument("rel_tol must be in (0,1)");
    if (max_iter < 1) throw std::invalid_argument("max_iter must be >= 1");
    return smg::fgmres(c, level, static_cast<double*>(x), static_cast<const double*>(b), rel_tol, max_iter, vp,
                       iters, history);
  });
}

int smg_slab_sizes(int degree, int level, int z0, int z1, int64_t sizes[5]) {
  try {
    const int m = 2 << level;
    smg::LevelLayout l(degree, level, std::max(z0 - 1, 0), std::min(z1 + 1, m));
    if (z0 < 0 || z1 > m || z0 >= z1) return SMG_EINVAL;
    for (int i = 0; i < 4; ++i) sizes[i] = l.size[i];
    sizes[4] = l.total;
    return SMG_OK;
  } catch (...) {
    return SMG_EINVAL;
  }
}

int smg_vmult_slab(smg_context* h, int level, int precision, void* y, const void* x, int z0, int z1) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!x || !y || x == y) throw std::invalid_argument("vmult_slab: x and y must be distinct non-null vectors");
    smg::launch_vmult_slab(c, level, precision, y, x, nullptr, z0, z1);
    return SMG_OK;
  });
}

int smg_residual_slab(smg_context* h, int level, int precision, void* r, const void* b, const void* x, int z0, int z1) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!r || !b || !x || r == x || r == b) throw std::invalid_argument("residual_slab: r must differ from b and x");
    smg::launch_vmult_slab(c, level, precision, r, x, b, z0, z1);
    return SMG_OK;
  });
}

int smg_dot_slab(smg_context* h, int level, int precision, const void* a, const void* b, int z0, int z1, double* out) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!out) throw std::invalid_argument("dot_slab: null output");
    const int m = c.dev[0][level].lay.m, H = c.cfg.degree + 1;
    if (z0 < 0 || z1 > m || z0 >= z1) throw std::invalid_argument("dot_slab: owned range out of range");
    const smg::LevelLayout lay(c.cfg.degree, level, std::max(z0 - 1, 0), std::min(z1 + 1, m));
    int64_t beg[4], len[4];
    for (int blk = 0; blk < 4; ++blk) {
      // owned node planes of the block (u_z: plus the constrained top plane on the last slab)
      const int64_t p0 = static_cast<int64_t>(z0 - lay.zlo) * H;
      int64_t p1 = static_cast<int64_t>(z1 - lay.zlo) * H;
      if (blk == 2 && z1 == m) p1 += 1;
      beg[blk] = lay.off[blk] + p0 * lay.plane[blk];
      len[blk] = (p1 - p0) * lay.plane[blk];
    }
    *out = smg::dot_ranges(c, precision, a, b, beg, len, 4);
    return SMG_OK;
  });
}

int smg_held_sizes(int degree, int level, int zlo, int zhi, int64_t sizes[5]) {
  try {
    smg::LevelLayout l(degree, level, zlo, zhi);
    for (int i = 0; i < 4; ++i) sizes[i] = l.size[i];
    sizes[4] = l.total;
    return SMG_OK;
  } catch (...) {
    return SMG_EINVAL;
  }
}

int smg_residual_held(smg_context* h, int level, int precision, void* r, const void* b, const void* x, int zlo, int zhi,
                      int c0, int c1) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!r || !x || r == x || r == b) throw std::invalid_argument("residual_held: r must differ from b and x");
    smg::launch_vmult_args_public(c, level, precision, r, x, b, zlo, zhi, c0, c1);
    return SMG_OK;
  });
}

int smg_smooth_colour_held(smg_context* h, int level, int precision, int colour, void* x, const void* r, int zlo,
                           int zhi, int vz0, int vz1) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (level < 1 || colour < 0 || colour > 7) throw std::invalid_argument("smooth_colour_held: bad level / colour");
    smg::launch_smooth_colour_held(c, level, precision, colour, x, r, zlo, zhi, vz0, vz1);
    return SMG_OK;
  });
}

int smg_prolongate_add_held(smg_context* h, int coarse_level, int precision, void* xf, const void* xc, int fzlo,
                            int fzhi, int czlo, int czhi, int f0, int f1) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, coarse_level + 1);
    smg::check_prec(precision);
    smg::launch_prolongate_add_held(c, coarse_level, precision, xf, xc, fzlo, fzhi, czlo, czhi, f0, f1);
    return SMG_OK;
  });
}

int smg_restrict_held(smg_context* h, int coarse_level, int precision, void* rc, const void* rf, int fzlo, int fzhi,
                      int czlo, int czhi, int c0, int c1) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, coarse_level + 1);
    smg::check_prec(precision);
    smg::launch_restrict_held(c, coarse_level, precision, rc, rf, fzlo, fzhi, czlo, czhi, c0, c1);
    return SMG_OK;
  });
}

int smg_dot_held(smg_context* h, int level, int precision, const void* a, const void* b, int zlo, int zhi, int c0,
                 int c1, double* out) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!out) throw std::invalid_argument("dot_held: null output");
    const int m = c.dev[0][level].lay.m, H = c.cfg.degree + 1;
    if (c0 < zlo || c1 > zhi || c0 >= c1) throw std::invalid_argument("dot_held: rows outside the held cells");
    const smg::LevelLayout lay(c.cfg.degree, level, zlo, zhi);
    int64_t beg[4], len[4];
    for (int blk = 0; blk < 4; ++blk) {
      const int64_t p0 = static_cast<int64_t>(c0 - zlo) * H;
      int64_t p1 = static_cast<int64_t>(c1 - zlo) * H;
      if (blk == 2 && c1 == m) p1 += 1;
      beg[blk] = lay.off[blk] + p0 * lay.plane[blk];
      len[blk] = (p1 - p0) * lay.plane[blk];
    }
    *out = smg::dot_ranges(c, precision, a, b, beg, len, 4);
    return SMG_OK;
  });
}

int smg_dot(smg_context* h, int level, int precision, const void* a, const void* b, double* out) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    *out = smg::dot(c, c.dev[0][level].lay.total, precision, a, b);
    return SMG_OK;
  });
}

int smg_axpy(smg_context* h, int level, int precision, double alpha, const void* x, void* y) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    smg::launch_axpy(c, c.dev[0][level].lay.total, precision, alpha, x, y);
    return SMG_OK;
  });
}

int smg_convert(smg_context* h, int level, int dp, void* dst, int sp, const void* src) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(dp);
    smg::check_prec(sp);
    smg::launch_convert(c, c.dev[0][level].lay.total, dp, dst, sp, src);
    return SMG_OK;
  });
}

int smg_smoother_stats(smg_context* h, int reset, int64_t* patches, int64_t* cg_iterations) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    unsigned long long v[2];
    SMG_CUDA(cudaMemcpyAsync(v, c.smoother_stats, sizeof(v), cudaMemcpyDeviceToHost, c.stream));
    SMG_CUDA(cudaStreamSynchronize(c.stream));
    if (patches) *patches = static_cast<int64_t>(v[0]);
    if (cg_iterations) *cg_iterations = static_cast<int64_t>(v[1]);
    if (reset) SMG_CUDA(cudaMemsetAsync(c.smoother_stats, 0, sizeof(v), c.stream));
    return SMG_OK;
  });
}

int smg_scale(smg_context* h, int level, int precision, double alpha, void* x) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!x) throw std::invalid_argument("scale: null vector");
    smg::launch_scale(c, c.dev[0][level].lay.total, precision, alpha, x);
    return SMG_OK;
  });
}

int smg_subtract_from(smg_context* h, int level, int precision, const void* b, void* y) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!b || !y) throw std::invalid_argument("subtract_from: null vector");
    smg::launch_axpby(c, c.dev[0][level].lay.total, precision, 1.0, b, -1.0, y);  // y = b - y
    return SMG_OK;
  });
}

int smg_norm(smg_context* h, int level, int precision, const void* x, double* out) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!x || !out) throw std::invalid_argument("norm: null pointer");
    *out = std::sqrt(smg::dot(c, c.dev[0][level].lay.total, precision, x, x));
    return SMG_OK;
  });
}

int smg_project_zero_mean(smg_context* h, int level, int precision, void* x) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!x) throw std::invalid_argument("project_zero_mean: null vector");
    smg::launch_sub_pressure_mean(c, level, precision, x);
    return SMG_OK;
  });
}

int smg_vec_upload(smg_context* h, int level, int precision, void* dst, const void* const vel[3], const void* p) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!dst || !vel || !vel[0] || !vel[1] || !vel[2] || !p) throw std::invalid_argument("vec_upload: null pointer");
    smg::upload_blocks(c, level, precision, static_cast<char*>(dst), vel, p);
    SMG_CUDA(cudaStreamSynchronize(c.stream));
    return SMG_OK;
  });
}

int smg_vec_download(smg_context* h, int level, int precision, void* const vel[3], void* p, const void* src) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!src || !vel || !vel[0] || !vel[1] || !vel[2] || !p) throw std::invalid_argument("vec_download: null pointer");
    smg::download_blocks(c, level, precision, vel, p, static_cast<const char*>(src));
    SMG_CUDA(cudaStreamSynchronize(c.stream));
    return SMG_OK;
  });
}

int smg_vmult_host(smg_context* h, int level, int precision, void* const y_vel[3], void* y_p,
                   const void* const x_vel[3], const void* x_p) {
  return smg::guarded(h, [&] {
    Context& c = smg::ctx_of(h);
    smg::check_level(c, level);
    smg::check_prec(precision);
    if (!x_vel || !y_vel || !x_p || !y_p) throw std::invalid_argument("vmult_host: null pointer");
    smg::vmult_host_pipelined(c, level, precision, y_vel, y_p, x_vel, x_p);
    return SMG_OK;
  });
}

}  // extern "C"
