// comm.cu — NCCL collectives for the sharded ALS, loaded at run time.
//
// libnccl.so.2 is dlopen'ed on first use (the one torch already loaded is picked up by
// soname), so the library itself has no link-time NCCL dependency and loads on a
// CPU-only host.  Exchange per mode (§8(e) steps 4-5): all-reduce(sum) of the R x R
// partial Gram + fit inner product, all-reduce(max) of the column maxima, and an
// all-gather of the owned factor rows with uneven counts as grouped broadcasts
// (NCCL has no allgatherv).  All on the context stream, so they order with kernels.
#include <dlfcn.h>
#include <nccl.h>

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

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm && api().CommDestroy) api().CommDestroy(comm);
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) override {
    check(api().AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm, s), "ncclAllReduce(sum)");
  }
  void allreduce_max(double* buf, size_t n, cudaStream_t s) override {
    check(api().AllReduce(buf, buf, n, ncclFloat64, ncclMax, comm, s), "ncclAllReduce(max)");
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
