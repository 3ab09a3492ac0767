// ctx.hpp — the library context: device, stream, stream-ordered allocator, comm.
#pragma once
#include <chrono>
#include <cstdlib>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace sb {

// Collective interface used by the ALS driver when the path is sharded
// (SURVEY.md §8(e)).  Implemented over NCCL (comm.cu).
struct Comm {
  int nranks = 1, rank = 0;
  virtual ~Comm() = default;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_max(double* buf, size_t n, cudaStream_t s) = 0;
  // Rows [bounds[g], bounds[g+1]) of the I x ld matrix `base` are valid on rank g;
  // afterwards every rank holds all rows.
  virtual void allgatherv_rows(double* base, const std::vector<uint64_t>& bounds, int ld,
                               cudaStream_t s) = 0;
};

std::unique_ptr<Comm> make_nccl_comm(const void* id128, int nranks, int rank);
std::unique_ptr<Comm> make_loopback_comm(splatt_loopback* group, int rank);

}  // namespace sb

struct splatt_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  size_t l2_bytes = 0;
  std::string err;
  uint64_t kernel_launches = 0;
  uint64_t host_syncs = 0;       // blocking stream syncs issued by the library
  double host_sync_s = 0.0;      // host seconds spent in them
  std::vector<cudaEvent_t> ev_pool;      // timing events reused across calls (EventTimer)
  std::vector<cudaEvent_t> ev_pool_aux;  // same, for spans on the aux stream
  // Side stream for the R x R work that overlaps the MTTKRP (V^-1 of the next mode, the
  // fit) and two ordering events; created on first use, owned by the context.
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_aux = nullptr;
  std::unique_ptr<sb::Comm> comm;
  ~splatt_ctx() {
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_pool_aux) cudaEventDestroy(e);
    if (ev_ready) cudaEventDestroy(ev_ready);
    if (ev_aux) cudaEventDestroy(ev_aux);
    if (aux) cudaStreamDestroy(aux);
  }
  void ensure_aux() {
    if (aux) return;
    SB_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    SB_CUDA(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
    SB_CUDA(cudaEventCreateWithFlags(&ev_aux, cudaEventDisableTiming));
  }
};

namespace sb {

// RAII device buffer on the context's stream-ordered pool (cudaMallocAsync): frees
// are stream-ordered, so no host sync is needed between ALS phases.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) SB_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), stream));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
    return *this;
  }
  T* get() const { return p; }
};

// Spans of CUDA events recorded on one stream, read once at the end.  Events come from a
// per-context pool that lives as long as the context (no create/destroy per span), and a
// span that starts where the previous one ended reuses its end event.
struct EventTimer {
  struct Span { int a, b, cat; };
  std::vector<Span> spans;
  std::vector<cudaEvent_t>* pool = nullptr;
  size_t used = 0;
  cudaStream_t s = nullptr;
  bool on = false;
  int open_cat = -1, open_a = -1, last_end = -1;
  void init(std::vector<cudaEvent_t>* p, cudaStream_t stream, bool enabled) {
    pool = p;
    s = stream;
    on = enabled;
  }
  int record() {
    if (used == pool->size()) {
      cudaEvent_t e;
      SB_CUDA(cudaEventCreate(&e));
      pool->push_back(e);
    }
    SB_CUDA(cudaEventRecord((*pool)[used], s));
    return (int)used++;
  }
  void begin(int cat) {
    if (!on) return;
    open_a = (last_end >= 0) ? last_end : record();
    open_cat = cat;
  }
  void end() {
    if (!on) return;
    const int b = record();
    spans.push_back({open_a, b, open_cat});
    last_end = b;
  }
  // Any stream work between end() and the next begin() must not be attributed: call gap().
  void gap() { last_end = -1; }
  // Requires the stream to have completed.
  void collect(double* per_cat, int ncat) {
    for (auto& sp : spans) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, (*pool)[sp.a], (*pool)[sp.b]) == cudaSuccess && sp.cat < ncat)
        per_cat[sp.cat] += ms * 1e-3;
    }
  }
};

bool is_device_ptr(const void* p);

// Debug tracing (env SPLATT_TRACE=1): synchronises at every mark and prints the host
// wall time of each phase to stderr.  Off by default (no syncs, no output).
struct PhaseTrace {
  bool on = false;
  std::chrono::steady_clock::time_point t;
  cudaStream_t s = nullptr;
  const char* what = "";
  PhaseTrace(cudaStream_t stream, const char* w) : s(stream), what(w) {
    static const bool enabled = getenv("SPLATT_TRACE") != nullptr;
    on = enabled;
    if (on) { cudaStreamSynchronize(s); t = std::chrono::steady_clock::now(); }
  }
  void mark(const char* phase) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[splatt trace] %s %-14s %8.3f ms\n", what, phase,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Blocking wait on the context stream, counted and timed (splatt_stats host_syncs).
inline void host_sync(splatt_ctx* ctx) {
  const auto t0 = std::chrono::steady_clock::now();
  SB_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->host_sync_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  ++ctx->host_syncs;
}

}  // namespace sb
