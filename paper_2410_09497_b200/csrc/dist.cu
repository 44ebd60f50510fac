// Multi-GPU driver behind the C ABI: z-slab partition of the cell
// array, one context per GPU / rank; the Stokes operator, the slab V-cycle and MG-preconditioned FGMRES
// over the slabs, with the ghost exchange and the reductions going through a transport:
//   * built-in NCCL (smg_dist_init_nccl): grouped ncclSend / ncclRecv of contiguous node-plane slices
//     per block and neighbour (NVLink / NVSwitch), ncclAllReduce for dots and the agglomerated coarse
//     levels -- all on the context's stream, so a caller may capture them in a CUDA graph;
//   * caller callbacks (smg_dist_init_transport), e.g. MPI, or torch.distributed in the tests.
// This is the C++ form of the reference's seams fgmres(apply_A, apply_P, ...) and
// v_cycle for a partitioned mesh; the semantics are those of smg_solve (single GPU):
// the level-by-level algorithm is identical, so the results equal the single-GPU ones to rounding.
//
// Partition: finest-level owned cells [z0, z1) of rank r from smg_dist_partition (contiguous, even,
// boundaries on multiples of 4 cells); level l owns [z0 >> (L-l), z1 >> (L-l)). MG vectors of level l
// hold GHOST = 3 cell layers beyond each interior end (smg_dist_sizes):
//   * smoothing, per colour: ghost exchange of x, residual on the rows of cells [z0-2, z1+1), then the
//     colour's patches with vertex planes z0..z1 (face patches computed identically on both sides);
//   * restriction reads fine cells 2c0-2 .. 2c1-1 (hence the residual rows from z0-2 and GHOST = 3);
//     prolongation adds into the owned fine rows;
//   * the finest level whose slabs are < 4 cells or do not nest is agglomerated: the owned rows of the
//     right-hand side are summed over the ranks into a full vector and the rest of the V-cycle runs
//     replicated on every rank (smg_vcycle), then each rank takes back its held rows.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "smg_internal.cuh"

namespace smg {

void vcycle_level(Context& c, int level, int prec, void* x, const void* b);  // api.cu

namespace {

constexpr int kGhost = 3;

// ---- NCCL through dlopen: the library has no link-time NCCL dependency, and inside a PyTorch process
// it binds to the libnccl.so.2 torch already loaded ----
struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, const char*, int) = nullptr;  // ncclUniqueId passed by value: 128 bytes
  int (*CommDestroy)(void*) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
};
struct UniqueId {
  char b[128];
};
NcclApi& nccl() {
  static NcclApi api;
  if (!api.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw cuda_error("NCCL not found (libnccl.so.2)");
    api.GetUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
    api.CommDestroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupEnd"));
    api.Send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(dlsym(h, "ncclSend"));
    api.Recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(dlsym(h, "ncclRecv"));
    api.AllReduce =
        reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(dlsym(h, "ncclAllReduce"));
    if (!api.GetUniqueId || !api.CommDestroy || !api.GroupStart || !api.GroupEnd || !api.Send || !api.Recv ||
        !api.AllReduce || !dlsym(h, "ncclCommInitRank"))
      throw cuda_error("NCCL symbols missing");
    api.h = h;
  }
  return api;
}
// ncclCommInitRank(ncclComm_t*, int nranks, ncclUniqueId id (by value), int rank)
int nccl_comm_init(void** comm, int nranks, const UniqueId& id, int rank) {
  using Fn = int (*)(void**, int, UniqueId, int);
  auto fn = reinterpret_cast<Fn>(dlsym(nccl().h, "ncclCommInitRank"));
  return fn(comm, nranks, id, rank);
}
constexpr int kNcclChar = 0, kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0;

struct Msg {
  void* ptr;
  size_t bytes;
  int peer;
};

}  // namespace

// per-context distributed state
struct DistState {
  int nranks = 1, rank = 0;
  std::vector<std::pair<int, int>> bounds;  // finest owned cells of every rank
  int L = 0, la = 0;                        // finest level, agglomeration level (levels > la partitioned)
  bool use_nccl = false;
  void* comm = nullptr;
  smg_transport tr{};
  // work vectors [prec][level] in the held layout (levels > la and la itself), full vectors at la
  std::vector<void*> x[2], r[2], b[2], full[2], fullx[2];
  std::vector<void*> krylov;  // fp64 finest held vectors (FGMRES basis)
  double* dscal = nullptr;    // device scratch for reductions
  cudaGraphExec_t vgraph[2] = {nullptr, nullptr};  // captured finest-level V-cycle per precision (NCCL)
  int64_t vgraph_launches[2] = {0, 0};
  bool graph_failed = false;
  ~DistState() {
    for (cudaGraphExec_t& e : vgraph)
      if (e) cudaGraphExecDestroy(e);
    if (use_nccl && comm) nccl().CommDestroy(comm);
    for (int p = 0; p < 2; ++p)
      for (auto* v : {&x[p], &r[p], &b[p], &full[p], &fullx[p]})
        for (void* q : *v) cudaFree(q);
    for (void* q : krylov) cudaFree(q);
    cudaFree(dscal);
  }
};

namespace {

DistState& dist(Context& c) {
  if (!c.dist) throw std::invalid_argument("the context has no distributed set-up (smg_dist_init_*)");
  return *c.dist;
}

// owned / held cells of rank r at level l
struct Slab {
  int m, z0, z1, zlo, zhi;
};
Slab slab_of(const DistState& D, int r, int l) {
  Slab s;
  s.m = 2 << l;
  s.z0 = D.bounds[r].first >> (D.L - l);
  s.z1 = D.bounds[r].second >> (D.L - l);
  s.zlo = std::max(s.z0 - kGhost, 0);
  s.zhi = std::min(s.z1 + kGhost, s.m);
  return s;
}

void* dalloc(size_t bytes) {
  void* p = nullptr;
  SMG_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  SMG_CUDA(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
  return p;
}

// ---- transport ----
void transport_exchange(Context& c, const std::vector<Msg>& sends, const std::vector<Msg>& recvs) {
  DistState& D = dist(c);
  if (sends.empty() && recvs.empty()) return;
  if (D.use_nccl) {
    NcclApi& N = nccl();
    if (N.GroupStart()) throw cuda_error("ncclGroupStart failed");
    for (const Msg& m : sends)
      if (N.Send(m.ptr, m.bytes, kNcclChar, m.peer, D.comm, c.stream)) throw cuda_error("ncclSend failed");
    for (const Msg& m : recvs)
      if (N.Recv(m.ptr, m.bytes, kNcclChar, m.peer, D.comm, c.stream)) throw cuda_error("ncclRecv failed");
    if (N.GroupEnd()) throw cuda_error("ncclGroupEnd failed");
    return;
  }
  std::vector<const void*> sp;
  std::vector<size_t> sb;
  std::vector<int> sr;
  std::vector<void*> rp;
  std::vector<size_t> rb;
  std::vector<int> rr;
  for (const Msg& m : sends) {
    sp.push_back(m.ptr);
    sb.push_back(m.bytes);
    sr.push_back(m.peer);
  }
  for (const Msg& m : recvs) {
    rp.push_back(m.ptr);
    rb.push_back(m.bytes);
    rr.push_back(m.peer);
  }
  if (D.tr.exchange(D.tr.user, static_cast<int>(sends.size()), sp.data(), sb.data(), sr.data(),
                    static_cast<int>(recvs.size()), rp.data(), rb.data(), rr.data(), c.stream) != 0)
    throw cuda_error("transport exchange callback failed");
}

void transport_allreduce(Context& c, void* dev, size_t count, int prec) {
  DistState& D = dist(c);
  if (D.nranks == 1) return;
  if (D.use_nccl) {
    if (nccl().AllReduce(dev, dev, count, prec == SMG_F64 ? kNcclFloat64 : kNcclFloat32, kNcclSum, D.comm, c.stream))
      throw cuda_error("ncclAllReduce failed");
    return;
  }
  if (D.tr.allreduce_sum(D.tr.user, dev, count, prec, c.stream) != 0)
    throw cuda_error("transport all-reduce callback failed");
}

// ghost exchange of a held vector of level l (> la): my owned cells inside a neighbour's held range go
// to it, its owned cells inside my held range come back; per block one contiguous slice of node planes
void exchange(Context& c, int l, int prec, void* v) {
  DistState& D = dist(c);
  const int k = c.cfg.degree, H = k + 1;
  const Slab S = slab_of(D, D.rank, l);
  const LevelLayout lay(k, l, S.zlo, S.zhi);
  const size_t es = elem_size(prec);
  std::vector<Msg> sends, recvs;
  for (int q : {D.rank - 1, D.rank + 1}) {
    if (q < 0 || q >= D.nranks) continue;
    const Slab T = slab_of(D, q, l);
    const int sa = std::max(S.z0, T.zlo), sb = std::min(S.z1, T.zhi);
    const int ra = std::max(S.zlo, T.z0), rb = std::min(S.zhi, T.z1);
    for (int blk = 0; blk < 4; ++blk) {
      char* base = static_cast<char*>(v) + lay.off[blk] * es;
      const int64_t pl = lay.plane[blk] * static_cast<int64_t>(es);
      if (sa < sb) sends.push_back({base + (sa - S.zlo) * H * pl, static_cast<size_t>((sb - sa) * H * pl), q});
      if (ra < rb) recvs.push_back({base + (ra - S.zlo) * H * pl, static_cast<size_t>((rb - ra) * H * pl), q});
    }
  }
  transport_exchange(c, sends, recvs);
}

// dot over the owned rows (fp64 accumulate) summed over the ranks
// (not `dot`: a qualified smg::dot would find the single-GPU dot declared directly in smg first)
double dist_dot(Context& c, int l, int prec, const void* a, const void* b) {
  DistState& D = dist(c);
  const int k = c.cfg.degree, H = k + 1;
  const Slab S = slab_of(D, D.rank, l);
  const LevelLayout lay(k, l, S.zlo, S.zhi);
  int64_t beg[4], len[4];
  for (int blk = 0; blk < 4; ++blk) {
    const int64_t p0 = static_cast<int64_t>(S.z0 - S.zlo) * H;
    int64_t p1 = static_cast<int64_t>(S.z1 - S.zlo) * H;
    if (blk == 2 && S.z1 == S.m) p1 += 1;
    beg[blk] = lay.off[blk] + p0 * lay.plane[blk];
    len[blk] = (p1 - p0) * lay.plane[blk];
  }
  double v = dot_ranges(c, prec, a, b, beg, len, 4);
  if (D.nranks == 1) return v;
  SMG_CUDA(cudaMemcpyAsync(D.dscal, &v, sizeof(double), cudaMemcpyHostToDevice, c.stream));
  transport_allreduce(c, D.dscal, 1, SMG_F64);
  SMG_CUDA(cudaMemcpyAsync(&v, D.dscal, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  SMG_CUDA(cudaStreamSynchronize(c.stream));
  return v;
}

int64_t held_total(Context& c, int l) {
  const Slab S = slab_of(dist(c), dist(c).rank, l);
  return LevelLayout(c.cfg.degree, l, S.zlo, S.zhi).total;
}

void ensure_dist_work(Context& c, int prec) {
  DistState& D = dist(c);
  if (!D.x[prec].empty()) return;
  const size_t es = elem_size(prec);
  D.x[prec].assign(D.L + 1, nullptr);
  D.r[prec].assign(D.L + 1, nullptr);
  D.b[prec].assign(D.L + 1, nullptr);
  D.full[prec].assign(D.L + 1, nullptr);
  D.fullx[prec].assign(D.L + 1, nullptr);
  for (int l = D.la; l <= D.L; ++l) {
    const size_t n = static_cast<size_t>(held_total(c, l)) * es;
    D.x[prec][l] = dalloc(n);
    D.r[prec][l] = dalloc(n);
    D.b[prec][l] = dalloc(n);
  }
  const size_t nf = static_cast<size_t>(c.dev[0][D.la].lay.total) * es;
  D.full[prec][D.la] = dalloc(nf);
  D.fullx[prec][D.la] = dalloc(nf);
}

// residual rows of the cells [z0 + c0, z1 + c1) (clipped to the level), held vectors of level l
void residual_rows(Context& c, int l, int prec, void* r, const void* b, const void* x, int c0, int c1) {
  const Slab S = slab_of(dist(c), dist(c).rank, l);
  const int a0 = std::max(S.z0 + c0, 0), a1 = std::min(S.z1 + c1, S.m);
  if (a0 < a1) launch_vmult_args_public(c, l, prec, r, x, b, S.zlo, S.zhi, a0, a1);
}

void smooth(Context& c, int l, int prec, void* x, const void* b, void* r) {
  const Slab S = slab_of(dist(c), dist(c).rank, l);
  for (int col = 0; col < 8; ++col) {
    exchange(c, l, prec, x);
    residual_rows(c, l, prec, r, b, x, -2, 1);
    launch_smooth_colour_held(c, l, prec, col, x, r, S.zlo, S.zhi, S.z0, S.z1);
  }
}

// owned planes of the held vector v (level l) -> full vector f at the same positions (block by block)
void copy_planes(Context& c, int l, int prec, void* dst, const void* src, bool to_full, int cz0, int cz1) {
  DistState& D = dist(c);
  const int k = c.cfg.degree, H = k + 1;
  const Slab S = slab_of(D, D.rank, l);
  const LevelLayout held(k, l, S.zlo, S.zhi), full(k, l);
  const size_t es = elem_size(prec);
  for (int blk = 0; blk < 4; ++blk) {
    const int64_t p0 = static_cast<int64_t>(cz0) * H;
    int64_t p1 = static_cast<int64_t>(cz1) * H;
    if (blk == 2 && cz1 == S.m) p1 += 1;
    const int64_t hoff = held.off[blk] + (p0 - static_cast<int64_t>(S.zlo) * H) * held.plane[blk];
    const int64_t foff = full.off[blk] + p0 * full.plane[blk];
    const size_t bytes = static_cast<size_t>((p1 - p0) * held.plane[blk]) * es;
    char* d = static_cast<char*>(dst) + (to_full ? foff : hoff) * es;
    const char* s = static_cast<const char*>(src) + (to_full ? hoff : foff) * es;
    SMG_CUDA(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, c.stream));
  }
}

void vcycle(Context& c, int l, int prec, void* x, const void* b) {
  DistState& D = dist(c);
  const size_t es = elem_size(prec);
  const Slab S = slab_of(D, D.rank, l);
  if (l == D.la) {
    // agglomeration: owned rows summed over the ranks into a full vector, V-cycle replicated
    void* full = D.full[prec][l];
    void* fx = D.fullx[prec][l];
    SMG_CUDA(cudaMemsetAsync(full, 0, c.dev[0][l].lay.total * es, c.stream));
    copy_planes(c, l, prec, full, b, true, S.z0, S.z1);
    transport_allreduce(c, full, c.dev[0][l].lay.total, prec);
    vcycle_level(c, l, prec, fx, full);
    copy_planes(c, l, prec, x, fx, false, S.zlo, S.zhi);
    return;
  }
  void* r = D.r[prec][l];
  SMG_CUDA(cudaMemsetAsync(x, 0, held_total(c, l) * es, c.stream));
  exchange(c, l, prec, const_cast<void*>(b));
  smooth(c, l, prec, x, b, r);
  exchange(c, l, prec, x);
  residual_rows(c, l, prec, r, b, x, -2, 1);
  const int lc = l - 1;
  const Slab Sc = slab_of(D, D.rank, lc);
  void* bc = D.b[prec][lc];
  void* xc = D.x[prec][lc];
  SMG_CUDA(cudaMemsetAsync(bc, 0, held_total(c, lc) * es, c.stream));
  launch_restrict_held(c, lc, prec, bc, r, S.zlo, S.zhi, Sc.zlo, Sc.zhi, Sc.z0, Sc.z1);
  vcycle(c, lc, prec, xc, bc);
  launch_prolongate_add_held(c, lc, prec, x, xc, S.zlo, S.zhi, Sc.zlo, Sc.zhi, S.z0, S.z1);
  smooth(c, l, prec, x, b, r);
}

void vmult(Context& c, int l, int prec, void* y, void* x) {
  exchange(c, l, prec, x);
  residual_rows(c, l, prec, y, nullptr, x, 0, 0);
}

// mass-weighted pressure mean over the owned rows (all ranks), subtracted from every held row
void project_mean(Context& c, int prec, void* x) {
  DistState& D = dist(c);
  const int k = c.cfg.degree, H = k + 1, l = D.L;
  const Slab S = slab_of(D, D.rank, l);
  const LevelLayout lay(k, l, S.zlo, S.zhi);
  const int n = lay.n;
  // the weighted sum is a dot of the owned pressure rows with the (separable) node weights of the whole
  // level's pressure block, built once per context
  if (!c.dist_pw) {
    const auto w1 = pressure_node_weights(k);
    std::vector<double> w(static_cast<size_t>(n) * n * n);
    for (int z = 0; z < n; ++z)
      for (int y = 0; y < n; ++y)
        for (int xx = 0; xx < n; ++xx) w[(static_cast<size_t>(z) * n + y) * n + xx] = w1[z % H] * w1[y % H] * w1[xx % H];
    c.dist_pw = dalloc(w.size() * sizeof(double));
    SMG_CUDA(cudaMemcpy(c.dist_pw, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  const int64_t pl = static_cast<int64_t>(n) * n;
  const int64_t beg = lay.off[3] + static_cast<int64_t>(S.z0 - S.zlo) * H * pl;
  const int64_t len = static_cast<int64_t>(S.z1 - S.z0) * H * pl;
  // dot of x's owned pressure rows with the weights at the same global planes
  const double* wg = static_cast<const double*>(c.dist_pw) + static_cast<int64_t>(S.z0) * H * pl;
  const size_t es = elem_size(prec);
  double s;
  if (prec == SMG_F64) {
    const int64_t b0[1] = {0}, l0[1] = {len};
    s = dot_ranges(c, SMG_F64, static_cast<const char*>(x) + beg * es, wg, b0, l0, 1);
  } else {
    throw std::invalid_argument("project_mean: fp64 only");
  }
  if (D.nranks > 1) {
    SMG_CUDA(cudaMemcpyAsync(D.dscal, &s, sizeof(double), cudaMemcpyHostToDevice, c.stream));
    transport_allreduce(c, D.dscal, 1, SMG_F64);
    SMG_CUDA(cudaMemcpyAsync(&s, D.dscal, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    SMG_CUDA(cudaStreamSynchronize(c.stream));
  }
  double ws = 0.0;
  for (double v : pressure_node_weights(k)) ws += v;
  const double mean = s / (ws * ws * ws * double(lay.m) * lay.m * lay.m);
  launch_add_scalar(c, lay.size[3], prec, -mean, static_cast<char*>(x) + lay.off[3] * es);  // every held row
}

// The finest-level fp32 V-cycle on the fixed work vectors, replayed from a CUDA graph when the
// transport is the in-library NCCL (its send / recv / all-reduce are stream-ordered and captured with
// the kernels); caller callbacks run on the host and cannot be captured, so they take plain launches.
// A failed capture (e.g. an NCCL build without graph support) falls back to plain launches for good.
void vcycle_maybe_graph(Context& c, int prec, void* vx, const void* vb) {
  DistState& D = dist(c);
  static const bool off = std::getenv("SMG_NO_GRAPH") != nullptr;
  if (off || !D.use_nccl || D.graph_failed) {
    vcycle(c, D.L, prec, vx, vb);
    return;
  }
  if (!D.vgraph[prec]) {
    vcycle(c, D.L, prec, vx, vb);  // warm-up: lazy set-up outside the capture
    SMG_CUDA(cudaStreamSynchronize(c.stream));
    if (!c.s_capture) SMG_CUDA(cudaStreamCreateWithFlags(&c.s_capture, cudaStreamNonBlocking));
    const cudaStream_t user = c.stream;
    c.stream = c.s_capture;
    c.tmap_recorded.clear();
    c.tmap_recording = true;
    const int64_t l0 = c.launches;
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      try {
        vcycle(c, D.L, prec, vx, vb);
      } catch (...) {
        ok = false;
      }
      ok = (cudaStreamEndCapture(c.stream, &g) == cudaSuccess) && ok && g;
    }
    c.stream = user;
    c.tmap_recording = false;
    if (ok && cudaGraphInstantiate(&D.vgraph[prec], g, 0) == cudaSuccess) {
      D.vgraph_launches[prec] = c.launches - l0;
      if (c.tmap_pinned.size() != static_cast<size_t>(kTmapSlots)) c.tmap_pinned.assign(kTmapSlots, false);
      for (int slot : c.tmap_recorded) c.tmap_pinned[slot] = true;
    } else {
      D.vgraph[prec] = nullptr;
      D.graph_failed = true;
      cudaGetLastError();  // clear a sticky capture error
    }
    if (g) cudaGraphDestroy(g);
    c.launches = l0;
    return;  // the warm-up cycle already produced this call's result (the capture executes nothing)
  }
  SMG_CUDA(cudaGraphLaunch(D.vgraph[prec], c.stream));
  c.launches += D.vgraph_launches[prec];
}

int fgmres(Context& c, double* x, const double* b, double tol, int max_iter, int vp, int* iters, double* hist) {
  DistState& D = dist(c);
  const int L = D.L;
  const int64_t N = held_total(c, L);
  size_t used = 0;
  auto newvec = [&]() {
    if (used == D.krylov.size()) D.krylov.push_back(dalloc(static_cast<size_t>(N) * 8));
    return static_cast<double*>(D.krylov[used++]);
  };
  if (vp == SMG_F32) ensure_dist_work(c, SMG_F32);
  ensure_dist_work(c, SMG_F64);
  std::vector<std::vector<double>> Hm(max_iter + 1, std::vector<double>(max_iter, 0.0));
  std::vector<double> cs(max_iter, 0.0), sn(max_iter, 0.0), g(max_iter + 1, 0.0);
  std::vector<double*> V, Z;
  launch_zero(c, N, SMG_F64, x);
  const double beta = std::sqrt(dist_dot(c, L, SMG_F64, b, b));
  if (hist) hist[0] = beta;
  if (beta == 0.0) {
    if (iters) *iters = 0;
    return SMG_OK;
  }
  V.push_back(newvec());
  launch_convert(c, N, SMG_F64, V[0], SMG_F64, b);
  launch_scale(c, N, SMG_F64, 1.0 / beta, V[0]);
  g[0] = beta;
  double* w = newvec();
  int it = 0;
  bool converged = false;
  for (; it < max_iter;) {
    const int j = it;
    Z.push_back(newvec());
    if (vp == SMG_F64) {
      vcycle(c, L, SMG_F64, Z[j], V[j]);
    } else {
      // fp64 -> fp32 at the V-cycle boundary; the finest fp32 b / x work vectors are not used by the
      // V-cycle of that level itself (it takes them as arguments)
      void* vb = D.b[SMG_F32][L];
      void* vx = D.x[SMG_F32][L];
      launch_convert(c, N, SMG_F32, vb, SMG_F64, V[j]);
      vcycle_maybe_graph(c, SMG_F32, vx, vb);
      launch_convert(c, N, SMG_F64, Z[j], SMG_F32, vx);
    }
    vmult(c, L, SMG_F64, w, Z[j]);
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i <= j; ++i) {
        const double hij = dist_dot(c, L, SMG_F64, w, V[i]);
        Hm[i][j] += hij;
        launch_axpy(c, N, SMG_F64, -hij, V[i], w);
      }
    const double wn = std::sqrt(dist_dot(c, L, SMG_F64, w, w));
    Hm[j + 1][j] = wn;
    for (int i = 0; i < j; ++i) {
      const double t = cs[i] * Hm[i][j] + sn[i] * Hm[i + 1][j];
      Hm[i + 1][j] = -sn[i] * Hm[i][j] + cs[i] * Hm[i + 1][j];
      Hm[i][j] = t;
    }
    const double den = std::hypot(Hm[j][j], Hm[j + 1][j]);
    cs[j] = Hm[j][j] / den;
    sn[j] = Hm[j + 1][j] / den;
    Hm[j][j] = den;
    Hm[j + 1][j] = 0.0;
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
  }
  std::vector<double> y(it, 0.0);
  for (int i = it - 1; i >= 0; --i) {
    double s = g[i];
    for (int l2 = i + 1; l2 < it; ++l2) s -= Hm[i][l2] * y[l2];
    y[i] = s / Hm[i][i];
  }
  for (int i = 0; i < it; ++i) launch_axpy(c, N, SMG_F64, y[i], Z[i], x);
  project_mean(c, SMG_F64, x);
  SMG_CUDA(cudaStreamSynchronize(c.stream));
  if (iters) *iters = it;
  return converged ? SMG_OK : SMG_ENOTCONV;
}

}  // namespace

void dist_destroy(DistState* d) { delete d; }

// owned cells [z0, z1) of `rank` among `nranks` on level `level`: contiguous, as even as possible,
// interior boundaries on multiples of 4 cells (2 or 1 when the level is too thin)
bool dist_partition(int level, int nranks, int rank, int* z0, int* z1) {
  const int m = 2 << level;
  for (int mult = 4; mult >= 1; mult /= 2) {
    if (m % mult != 0) continue;
    const int units = m / mult;
    if (units < nranks) continue;
    const int base = units / nranks, extra = units % nranks;
    int z = 0;
    for (int r = 0; r <= rank; ++r) {
      const int w = (base + (r < extra ? 1 : 0)) * mult;
      if (r == rank) {
        *z0 = z;
        *z1 = z + w;
      }
      z += w;
    }
    return true;
  }
  return false;
}

namespace {

void dist_setup(Context& c, int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("dist: bad rank / nranks");
  auto* D = new DistState();
  try {
    D->nranks = nranks;
    D->rank = rank;
    D->L = c.cfg.max_level;
    for (int r = 0; r < nranks; ++r) {
      int a = 0, b = 0;
      if (!dist_partition(D->L, nranks, r, &a, &b))
        throw std::invalid_argument("dist: the finest level has fewer cell layers than ranks");
      D->bounds.push_back({a, b});
    }
    // finest levels that stay partitioned: every slab nests and keeps >= 4 cells
    D->la = D->L;
    for (int l = D->L; l >= 1; --l) {
      const int s = 1 << (D->L - l);
      bool ok = true;
      for (auto& bz : D->bounds) ok = ok && bz.first % s == 0 && bz.second % s == 0 && (bz.second - bz.first) / s >= 4;
      if (!ok) break;
      D->la = l - 1;
    }
    if (D->la >= D->L) throw std::invalid_argument("dist: the finest level is too thin to partition (>= 4 cells per slab)");
    D->dscal = static_cast<double*>(dalloc(64));
  } catch (...) {
    delete D;
    throw;
  }
  if (c.dist) dist_destroy(c.dist);
  c.dist = D;
}

}  // namespace
}  // namespace smg

using smg::Context;

extern "C" {

int smg_nccl_unique_id(char id[128]) {
  try {
    if (!id) return SMG_EINVAL;
    if (smg::nccl().GetUniqueId(id) != 0) return SMG_ECUDA;
    return SMG_OK;
  } catch (...) {
    return SMG_ECUDA;
  }
}

int smg_dist_init_nccl(smg_context* h, const char id[128], int nranks, int rank) {
  return smg::guarded_call(h, [&] {
    Context& c = smg::context_of(h);
    if (!id) throw std::invalid_argument("dist: null NCCL id");
    smg::dist_setup(c, nranks, rank);
    smg::UniqueId u;
    std::memcpy(u.b, id, 128);
    if (smg::nccl_comm_init(&c.dist->comm, nranks, u, rank) != 0) throw smg::cuda_error("ncclCommInitRank failed");
    c.dist->use_nccl = true;
    return SMG_OK;
  });
}

int smg_dist_init_transport(smg_context* h, const smg_transport* t, int nranks, int rank) {
  return smg::guarded_call(h, [&] {
    Context& c = smg::context_of(h);
    if (!t || (nranks > 1 && (!t->exchange || !t->allreduce_sum)))
      throw std::invalid_argument("dist: the transport needs exchange and allreduce_sum callbacks");
    smg::dist_setup(c, nranks, rank);
    c.dist->tr = *t;
    return SMG_OK;
  });
}

int smg_dist_partition(int level, int nranks, int rank, int* z0, int* z1) {
  if (!z0 || !z1 || nranks < 1 || rank < 0 || rank >= nranks || level < 0 || level > 12) return SMG_EINVAL;
  return smg::dist_partition(level, nranks, rank, z0, z1) ? SMG_OK : SMG_EINVAL;
}

int smg_dist_held(smg_context* h, int level, int cells[4], int64_t sizes[5]) {
  return smg::guarded_call(h, [&] {
    Context& c = smg::context_of(h);
    smg::DistState& D = smg::dist(c);
    if (level <= D.la || level > D.L) throw std::invalid_argument("dist: level is not partitioned");
    const smg::Slab S = smg::slab_of(D, D.rank, level);
    if (cells) {
      cells[0] = S.z0;
      cells[1] = S.z1;
      cells[2] = S.zlo;
      cells[3] = S.zhi;
    }
    if (sizes) {
      const smg::LevelLayout lay(c.cfg.degree, level, S.zlo, S.zhi);
      for (int i = 0; i < 4; ++i) sizes[i] = lay.size[i];
      sizes[4] = lay.total;
    }
    return SMG_OK;
  });
}

int smg_dist_vmult(smg_context* h, int level, int precision, void* y, void* x) {
  return smg::guarded_call(h, [&] {
    Context& c = smg::context_of(h);
    smg::DistState& D = smg::dist(c);
    if (precision != SMG_F64 && precision != SMG_F32) throw std::invalid_argument("bad precision");
    if (level <= D.la || level > D.L) throw std::invalid_argument("dist: level is not partitioned");
    if (!x || !y || x == y) throw std::invalid_argument("dist_vmult: x and y must be distinct non-null vectors");
    smg::vmult(c, level, precision, y, x);
    return SMG_OK;
  });
}

int smg_dist_dot(smg_context* h, int level, int precision, const void* a, const void* b, double* out) {
  return smg::guarded_call(h, [&] {
    Context& c = smg::context_of(h);
    smg::DistState& D = smg::dist(c);
    if (level <= D.la || level > D.L || !out) throw std::invalid_argument("dist_dot: bad level / output");
    *out = smg::dist_dot(c, level, precision, a, b);
    return SMG_OK;
  });
}

int smg_dist_vcycle(smg_context* h, int precision, void* x, const void* b) {
  return smg::guarded_call(h, [&] {
    Context& c = smg::context_of(h);
    smg::DistState& D = smg::dist(c);
    if (precision != SMG_F64 && precision != SMG_F32) throw std::invalid_argument("bad precision");
    smg::ensure_dist_work(c, precision);
    smg::vcycle(c, D.L, precision, x, b);
    return SMG_OK;
  });
}

int smg_dist_solve(smg_context* h, void* x, const void* b, double rel_tol, int max_iter, int vp, int* iters,
                   double* history) {
  return smg::guarded_call(h, [&] {
    Context& c = smg::context_of(h);
    smg::dist(c);
    if (vp != SMG_F64 && vp != SMG_F32) throw std::invalid_argument("bad precision");
    if (!(rel_tol > 0.0 && rel_tol < 1.0)) throw std::invalid_argument("rel_tol must be in (0,1)");
    if (max_iter < 1) throw std::invalid_argument("max_iter must be >= 1");
    return smg::fgmres(c, static_cast<double*>(x), static_cast<const double*>(b), rel_tol, max_iter, vp, iters,
                       history);
  });
}

}  // extern "C"
