// ctx.hpp — the library context: device, stream, stream-ordered allocator, comm.
#pragma once
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
  std::unique_ptr<sb::Comm> comm;
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

// Pairs of CUDA events recorded on one stream; durations read once at the end.
struct EventTimer {
  struct Span { cudaEvent_t a, b; int cat; };
  std::vector<Span> spans;
  cudaStream_t s = nullptr;
  bool on = false;
  int open_cat = -1;
  cudaEvent_t open_a = nullptr;
  void begin(int cat) {
    if (!on) return;
    SB_CUDA(cudaEventCreate(&open_a));
    SB_CUDA(cudaEventRecord(open_a, s));
    open_cat = cat;
  }
  void end() {
    if (!on) return;
    cudaEvent_t b;
    SB_CUDA(cudaEventCreate(&b));
    SB_CUDA(cudaEventRecord(b, s));
    spans.push_back({open_a, b, open_cat});
    open_a = nullptr;
  }
  // Requires the stream to have completed.
  void collect(double* per_cat, int ncat) {
    for (auto& sp : spans) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess && sp.cat < ncat)
        per_cat[sp.cat] += ms * 1e-3;
    }
  }
  ~EventTimer() {
    for (auto& sp : spans) { cudaEventDestroy(sp.a); cudaEventDestroy(sp.b); }
    if (open_a) cudaEventDestroy(open_a);
  }
};

bool is_device_ptr(const void* p);

}  // namespace sb
