// comm.cu — NCCL collectives for the sharded ALS, loaded at run time.
//
// libnccl.so.2 is dlopen'ed on first use (the one torch already loaded is picked up by
// soname), so the library itself has no link-time NCCL dependency and loads on a
// CPU-only host.  Exchange per mode (§8(e) steps 4-5): the R x R partial Gram + fit inner
// product (summed) and the column maxima (maximised) in one all-gather of the ranks'
// statistics followed by a rank-ordered local reduction (allreduce_stats), and an
// all-gather of the owned factor rows with uneven counts as grouped broadcasts (NCCL has no
// allgatherv) unless the solve kernel already stored them into the peers (map_peers,
// SPLATT_XCHG_PEER).  All on the context stream, so they order with kernels.
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <cstring>

#include <mutex>

#include "ctx.hpp"

namespace sb {

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return;
#define SB_SYM(f, s) a.f = reinterpret_cast<decltype(a.f)>(dlsym(a.h, s))
    SB_SYM(GetUniqueId, "ncclGetUniqueId");
    SB_SYM(CommInitRank, "ncclCommInitRank");
    SB_SYM(CommDestroy, "ncclCommDestroy");
    SB_SYM(AllReduce, "ncclAllReduce");
    SB_SYM(Broadcast, "ncclBroadcast");
    SB_SYM(AllGather, "ncclAllGather");
    SB_SYM(GroupStart, "ncclGroupStart");
    SB_SYM(GroupEnd, "ncclGroupEnd");
    SB_SYM(GetErrorString, "ncclGetErrorString");
#undef SB_SYM
  });
  if (!a.h || !a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.Broadcast ||
      !a.GroupStart || !a.GroupEnd)
    fail(SPLATT_ERR_NCCL, "libnccl.so.2 could not be loaded");
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    fail(SPLATT_ERR_NCCL, std::string(what) + ": " + s);
  }
}

// What a rank publishes about its factor slab (SPLATT_XCHG_PEER): the CUDA IPC handle of
// the cudaMalloc allocation, its size, the owner's allocation generation (a new allocation
// at a recycled address must not be taken for the old one) and the owner's process id.
struct SlabRec {
  cudaIpcMemHandle_t handle;
  uint64_t bytes, gen;
  int64_t pid;
  int32_t ok;
  int32_t pad;
};

// out[i] = sum (i < nsum) or max (else) over the G gathered copies g[r * len + i], in rank
// order: every rank computes the same bits, whatever algorithm NCCL picked for the gather.
__global__ void gathered_reduce_kernel(const double* __restrict__ g, int G, size_t len,
                                       size_t nsum, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len;
       i += (size_t)gridDim.x * blockDim.x) {
    double acc = g[i];
    for (int r = 1; r < G; ++r) {
      const double v = g[(size_t)r * len + i];
      acc = i < nsum ? acc + v : fmax(acc, v);
    }
    out[i] = acc;
  }
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  // peers' slabs mapped into this process, reused while the owner keeps its allocation
  struct Mapping {
    SlabRec rec{};
    void* ptr = nullptr;
  };
  std::vector<Mapping> maps;
  void close_map(Mapping& m) {
    if (m.ptr && cudaIpcCloseMemHandle(m.ptr) != cudaSuccess) cudaGetLastError();
    m.ptr = nullptr;
  }
  ~NcclComm() override {
    for (Mapping& m : maps) close_map(m);
    if (comm && api().CommDestroy) api().CommDestroy(comm);
  }
  // Handles travel with one all-gather of SlabRec bytes; a second tiny all-reduce(max) of
  // the ranks' failure flags makes the outcome the same everywhere.  Two host syncs per call.
  bool map_peers(void* base, size_t bytes, uint64_t gen, cudaStream_t s, void** peers) override {
    if (nranks > kMaxPeerRanks || !api().AllGather) return false;  // same answer on every rank
    maps.resize(nranks);
    const size_t rec = sizeof(SlabRec);
    std::vector<SlabRec> all(nranks);
    SlabRec mine{};
    mine.bytes = bytes;
    mine.gen = gen;
    mine.pid = (int64_t)getpid();
    mine.ok = cudaIpcGetMemHandle(&mine.handle, base) == cudaSuccess ? 1 : 0;
    if (!mine.ok) cudaGetLastError();
    DevBuf<char> d((size_t)nranks * rec, s);
    DevBuf<double> flag(1, s);
    SB_CUDA(cudaMemcpyAsync(d.p + (size_t)rank * rec, &mine, rec, cudaMemcpyHostToDevice, s));
    check(api().AllGather(d.p + (size_t)rank * rec, d.p, rec, ncclChar, comm, s), "ncclAllGather");
    SB_CUDA(cudaMemcpyAsync(all.data(), d.p, (size_t)nranks * rec, cudaMemcpyDeviceToHost, s));
    SB_CUDA(cudaStreamSynchronize(s));
    double failed = mine.ok ? 0.0 : 1.0;
    for (int g = 0; g < nranks; ++g) {
      if (g == rank) {
        peers[g] = base;
        continue;
      }
      Mapping& m = maps[g];
      const SlabRec& r = all[g];
      if (!r.ok || r.bytes != bytes || r.pid == mine.pid) {  // IPC needs another process
        failed = 1.0;
        continue;
      }
      const bool same = m.ptr && m.rec.gen == r.gen && m.rec.pid == r.pid &&
                        m.rec.bytes == r.bytes &&
                        memcmp(&m.rec.handle, &r.handle, sizeof(r.handle)) == 0;
      if (!same) {
        close_map(m);
        if (cudaIpcOpenMemHandle(&m.ptr, r.handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          m.ptr = nullptr;
          failed = 1.0;
          continue;
        }
        m.rec = r;
      }
      peers[g] = m.ptr;
    }
    SB_CUDA(cudaMemcpyAsync(flag.p, &failed, sizeof(double), cudaMemcpyHostToDevice, s));
    allreduce_max(flag.p, 1, s);
    SB_CUDA(cudaMemcpyAsync(&failed, flag.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    SB_CUDA(cudaStreamSynchronize(s));
    return failed == 0.0;
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) override {
    check(api().AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm, s), "ncclAllReduce(sum)");
  }
  void allreduce_max(double* buf, size_t n, cudaStream_t s) override {
    check(api().AllReduce(buf, buf, n, ncclFloat64, ncclMax, comm, s), "ncclAllReduce(max)");
  }
  // One collective instead of two (the exchange is latency-bound: ~10 KB per rank): the
  // ranks' statistics are all-gathered and every rank reduces them in rank order.
  void allreduce_stats(double* buf, size_t nsum, size_t nmax, cudaStream_t s) override {
    if (!api().AllGather) return Comm::allreduce_stats(buf, nsum, nmax, s);
    const size_t len = nsum + nmax;
    DevBuf<double> g((size_t)nranks * len, s);
    check(api().AllGather(buf, g.p, len, ncclFloat64, comm, s), "ncclAllGather(stats)");
    const unsigned blocks = (unsigned)std::min<size_t>(ceil_div(len, (size_t)256), 64);
    gathered_reduce_kernel<<<std::max(1u, blocks), 256, 0, s>>>(g.p, nranks, len, nsum, buf);
    SB_CUDA(cudaGetLastError());
  }
  void allgatherv_rows(double* base, const std::vector<uint64_t>& b, int ld,
                       cudaStream_t s) override {
    check(api().GroupStart(), "ncclGroupStart");
    for (int g = 0; g < nranks; ++g) {
      const size_t cnt = (size_t)(b[g + 1] - b[g]) * ld;
      if (!cnt) continue;
      double* p = base + b[g] * ld;
      check(api().Broadcast(p, p, cnt, ncclFloat64, g, comm, s), "ncclBroadcast");
    }
    check(api().GroupEnd(), "ncclGroupEnd");
  }
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const void* id128, int nranks, int rank) {
  auto c = std::make_unique<NcclComm>();
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId id;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(&id, id128, sizeof(id));
  check(api().CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  return c;
}

void nccl_unique_id(void* id128) {
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(id128, &id, sizeof(id));
}

}  // namespace sb
