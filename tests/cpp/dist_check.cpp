// C++ caller of the multi-GPU driver (smg_dist_*) through the host wrapper: two ranks as two host
// threads with one Context each on device 0, exchanging through a shared-memory mailbox transport
// (the callbacks a reference-side MPI / NCCL integration would provide). The distributed V-cycle-
// preconditioned FGMRES must equal the single-GPU smg_solve. Built by tests/test_host_cpp.py.
#include <cuda_runtime.h>

#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <thread>
#include <tuple>
#include <vector>

#include "../../paper_2410_09497_b200/host/stokesmg_b200.hpp"

using namespace stokesmg::b200;

struct Mailbox {
  int nranks;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0, gen = 0;
  std::map<std::tuple<int, int, int>, std::vector<char>> msgs;  // (src, dst, seq) -> bytes
  std::vector<std::vector<char>> red;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int g = gen;
    if (++arrived == nranks) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
struct RankUser {
  Mailbox* box;
  int rank;
};

int exchange_cb(void* user, int ns, const void* const* sp, const size_t* sb, const int* speer, int nr,
                void* const* rp, const size_t* rb, const int* rpeer, void* stream) {
  auto* u = static_cast<RankUser*>(user);
  cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  std::map<int, int> seq;
  for (int i = 0; i < ns; ++i) {
    std::vector<char> h(sb[i]);
    cudaMemcpy(h.data(), sp[i], sb[i], cudaMemcpyDeviceToHost);
    std::lock_guard<std::mutex> lk(u->box->mu);
    u->box->msgs[{u->rank, speer[i], seq[speer[i]]++}] = std::move(h);
  }
  u->box->barrier();
  std::map<int, int> rseq;
  for (int i = 0; i < nr; ++i) {
    std::vector<char> h;
    {
      std::lock_guard<std::mutex> lk(u->box->mu);
      auto it = u->box->msgs.find({rpeer[i], u->rank, rseq[rpeer[i]]++});
      if (it == u->box->msgs.end() || it->second.size() != rb[i]) return 1;
      h = std::move(it->second);
      u->box->msgs.erase(it);
    }
    cudaMemcpy(rp[i], h.data(), rb[i], cudaMemcpyHostToDevice);
  }
  u->box->barrier();
  return 0;
}

int allreduce_cb(void* user, void* dev, size_t count, int prec, void* stream) {
  auto* u = static_cast<RankUser*>(user);
  cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  const size_t bytes = count * (prec == SMG_F64 ? 8 : 4);
  std::vector<char> h(bytes);
  cudaMemcpy(h.data(), dev, bytes, cudaMemcpyDeviceToHost);
  {
    std::lock_guard<std::mutex> lk(u->box->mu);
    u->box->red[u->rank] = h;
  }
  u->box->barrier();
  std::vector<char> sum(bytes, 0);
  for (int r = 0; r < u->box->nranks; ++r)
    for (size_t i = 0; i < count; ++i) {
      if (prec == SMG_F64) reinterpret_cast<double*>(sum.data())[i] += reinterpret_cast<const double*>(u->box->red[r].data())[i];
      else reinterpret_cast<float*>(sum.data())[i] += reinterpret_cast<const float*>(u->box->red[r].data())[i];
    }
  u->box->barrier();
  cudaMemcpy(dev, sum.data(), bytes, cudaMemcpyHostToDevice);
  return 0;
}

int main() {
  const int k = 2, L = 3, R = 2;
  // right-hand side b = A x_r for a random x_r (full level, host)
  Context ref(k, L, 0, CgOptions{10, 0.0, true, true});
  const std::vector<int64_t> fs = ref.sizes(L);
  std::vector<double> xr(fs[4]);
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (auto& v : xr) v = U(rng);
  DeviceVector<double> dx(ref, L), db(ref, L), dxs(ref, L);
  cudaMemcpy(dx.data(), xr.data(), fs[4] * 8, cudaMemcpyHostToDevice);
  StokesOperator<double>(ref, L).vmult(db, dx);
  std::vector<double> b(fs[4]);
  cudaMemcpy(b.data(), db.data(), fs[4] * 8, cudaMemcpyDeviceToHost);
  const SolveResult rs = solve_mixed(ref, L, dxs, db, 1e-8, 30, /*fp32_vcycle=*/false);
  std::vector<double> xs(fs[4]), xd(fs[4], 0.0);
  cudaMemcpy(xs.data(), dxs.data(), fs[4] * 8, cudaMemcpyDeviceToHost);

  const int H = k + 1, n = (2 << L) * H, m = 2 << L;
  const int64_t plane[4] = {int64_t(n + 1) * n, int64_t(n) * (n + 1), int64_t(n) * n, int64_t(n) * n};
  Mailbox box;
  box.nranks = R;
  box.red.resize(R);
  std::vector<int> iters(R, -1);
  std::vector<std::thread> th;
  for (int r = 0; r < R; ++r)
    th.emplace_back([&, r] {
      RankUser user{&box, r};
      smg_transport t{exchange_cb, allreduce_cb, &user};
      Context ctx(k, L, 0, CgOptions{10, 0.0, true, true});
      DistContext dist(ctx, t, R, r);
      const DistContext::Held hd = dist.held(L);
      // held vectors: block by block, node planes zlo H .. zhi H (+1 for u_z)
      std::vector<double> bh(hd.sizes[4]);
      int64_t fo = 0, ho = 0;
      for (int c = 0; c < 4; ++c) {
        const int64_t np = int64_t(hd.zhi - hd.zlo) * H + (c == 2 ? 1 : 0);
        std::memcpy(bh.data() + ho, b.data() + fo + int64_t(hd.zlo) * H * plane[c], np * plane[c] * 8);
        fo += fs[c];
        ho += hd.sizes[c];
      }
      void *dbh = nullptr, *dxh = nullptr;
      cudaMalloc(&dbh, bh.size() * 8);
      cudaMalloc(&dxh, bh.size() * 8);
      cudaMemcpy(dbh, bh.data(), bh.size() * 8, cudaMemcpyHostToDevice);
      const SolveResult res = dist.solve(dxh, dbh, 1e-8, 30, /*fp32_vcycle=*/false);
      iters[r] = res.iterations;
      std::vector<double> xh(bh.size());
      cudaMemcpy(xh.data(), dxh, xh.size() * 8, cudaMemcpyDeviceToHost);
      fo = 0;
      ho = 0;
      for (int c = 0; c < 4; ++c) {  // owned rows into the gathered solution
        const int64_t a = int64_t(hd.z0 - hd.zlo) * H, e = int64_t(hd.z1 - hd.zlo) * H + (c == 2 && hd.z1 == m ? 1 : 0);
        std::lock_guard<std::mutex> lk(box.mu);
        std::memcpy(xd.data() + fo + (int64_t(hd.zlo) * H + a) * plane[c], xh.data() + ho + a * plane[c],
                    (e - a) * plane[c] * 8);
        fo += fs[c];
        ho += hd.sizes[c];
      }
      cudaFree(dbh);
      cudaFree(dxh);
    });
  for (auto& t : th) t.join();
  double dmax = 0.0, xmax = 0.0;
  for (int64_t i = 0; i < fs[4]; ++i) {
    dmax = std::fmax(dmax, std::fabs(xd[i] - xs[i]));
    xmax = std::fmax(xmax, std::fabs(xs[i]));
  }
  std::printf("single-GPU iterations %d, distributed %d %d, max rel diff %.3e\n", rs.iterations, iters[0], iters[1],
              dmax / xmax);
  if (iters[0] != rs.iterations || iters[1] != rs.iterations || dmax > 1e-10 * xmax) {
    std::fprintf(stderr, "FAILED\n");
    return 1;
  }
  std::printf("dist ok\n");
  return 0;
}
