// loopback.cu — in-process communicator: G logical ranks (host threads, one context and
// stream each) on one device, exchanging through device memory.  It runs the sharded ALS
// driver (partition, local CSFs, all-reduce, all-gather) unchanged on a single GPU, so the
// multi-rank path is tested on hardware without G GPUs (SURVEY.md §8(e) "loopback").
// No kernel ever waits on another rank: each exchange is host barrier -> copies / a
// fixed-order reduction kernel on the caller's stream -> stream sync -> host barrier.
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <new>

#include "ctx.hpp"

struct splatt_loopback {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptrs;
  // false if the other ranks did not arrive within the timeout (a rank failed)
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; });
  }
};

namespace sb {

namespace {

struct PeerPtrs {
  const double* p[SPLATT_MAX_NMODES];
  int n;
};

// out[i] = op over ranks 0..n-1 of in_g[i], in rank order (deterministic).
__global__ void peer_reduce_kernel(PeerPtrs pp, size_t len, int is_max, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len;
       i += (size_t)gridDim.x * blockDim.x) {
    double acc = pp.p[0][i];
    for (int g = 1; g < pp.n; ++g) acc = is_max ? fmax(acc, pp.p[g][i]) : acc + pp.p[g][i];
    out[i] = acc;
  }
}

struct LoopbackComm final : Comm {
  splatt_loopback* grp = nullptr;
  void sync_ranks() {
    if (!grp->barrier()) fail(SPLATT_ERR_CUDA, "loopback: peer ranks did not arrive (timeout)");
  }
  void reduce(double* buf, size_t n, cudaStream_t s, int is_max) {
    SB_CUDA(cudaStreamSynchronize(s));
    grp->ptrs[rank] = buf;
    sync_ranks();
    DevBuf<double> tmp(n, s);
    PeerPtrs pp{};
    pp.n = nranks;
    for (int g = 0; g < nranks; ++g) pp.p[g] = static_cast<const double*>(grp->ptrs[g]);
    const int blocks = (int)std::min<size_t>(ceil_div(n, 256), 1024);
    peer_reduce_kernel<<<std::max(1, blocks), 256, 0, s>>>(pp, n, is_max, tmp.p);
    SB_CUDA(cudaGetLastError());
    SB_CUDA(cudaStreamSynchronize(s));
    sync_ranks();  // every rank has read every buffer
    SB_CUDA(cudaMemcpyAsync(buf, tmp.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    SB_CUDA(cudaStreamSynchronize(s));
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) override { reduce(buf, n, s, 0); }
  void allreduce_max(double* buf, size_t n, cudaStream_t s) override { reduce(buf, n, s, 1); }
  void allgatherv_rows(double* base, const std::vector<uint64_t>& b, int ld,
                       cudaStream_t s) override {
    SB_CUDA(cudaStreamSynchronize(s));
    grp->ptrs[rank] = base;
    sync_ranks();
    for (int g = 0; g < nranks; ++g) {
      if (g == rank || b[g + 1] == b[g]) continue;
      const double* src = static_cast<const double*>(grp->ptrs[g]) + b[g] * ld;
      SB_CUDA(cudaMemcpyAsync(base + b[g] * ld, src, (b[g + 1] - b[g]) * ld * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
    }
    SB_CUDA(cudaStreamSynchronize(s));
    sync_ranks();  // nobody overwrites its rows while a peer still copies them
  }
  bool shares_device() const override { return true; }
  // One device, one address space: the peers' slabs are addressable as they are.
  bool map_peers(void* base, size_t bytes, uint64_t gen, cudaStream_t s, void** peers) override {
    (void)bytes; (void)gen;
    SB_CUDA(cudaStreamSynchronize(s));  // this rank's factor initialisation is done
    grp->ptrs[rank] = base;
    sync_ranks();
    for (int g = 0; g < nranks; ++g) peers[g] = const_cast<void*>(grp->ptrs[g]);
    sync_ranks();  // every rank has read the table before a later exchange reuses it
    return true;
  }
};

}  // namespace

std::unique_ptr<Comm> make_loopback_comm(splatt_loopback* grp, int rank) {
  auto c = std::make_unique<LoopbackComm>();
  c->grp = grp;
  c->nranks = grp->n;
  c->rank = rank;
  return c;
}

}  // namespace sb

extern "C" {

splatt_status splatt_loopback_create(int32_t nranks, splatt_loopback** out) {
  if (!out || nranks < 1 || nranks > SPLATT_MAX_NMODES) return SPLATT_ERR_BADINPUT;
  auto* g = new (std::nothrow) splatt_loopback();
  if (!g) return SPLATT_ERR_NOMEM;
  g->n = nranks;
  g->ptrs.assign(nranks, nullptr);
  *out = g;
  return SPLATT_OK;
}

void splatt_loopback_destroy(splatt_loopback* g) { delete g; }

splatt_status splatt_ctx_set_comm_loopback(splatt_ctx* ctx, splatt_loopback* g, int32_t rank) {
  if (!ctx || !g || rank < 0 || rank >= g->n) return SPLATT_ERR_BADINPUT;
  if (ctx->own_stream == false && (ctx->stream == nullptr || ctx->stream == (cudaStream_t)1))
    return SPLATT_ERR_BADINPUT;  // each logical rank needs its own stream
  if (g->n == 1) {
    ctx->comm.reset();
    return SPLATT_OK;
  }
  ctx->comm = sb::make_loopback_comm(g, rank);
  return SPLATT_OK;
}

}  // extern "C"
