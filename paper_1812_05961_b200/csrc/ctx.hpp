// ctx.hpp — the library context: device, stream, stream-ordered allocator, comm.
#pragma once
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace sb {

struct Arena;

// Collective interface used by the ALS driver when the path is sharded
// (SURVEY.md §8(e)).  Implemented over NCCL (comm.cu).
struct Comm {
  int nranks = 1, rank = 0;
  virtual ~Comm() = default;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_max(double* buf, size_t n, cudaStream_t s) = 0;
  // Ranks that are threads on ONE device (loopback): device-wide settings are left alone.
  virtual bool shares_device() const { return false; }
  // The per-mode statistics in one exchange: buf[0, nsum) summed and buf[nsum, nsum + nmax)
  // maximised over the ranks, the same bits on every rank.
  virtual void allreduce_stats(double* buf, size_t nsum, size_t nmax, cudaStream_t s) {
    allreduce_sum(buf, nsum, s);
    allreduce_max(buf + nsum, nmax, s);
  }
  // Rows [bounds[g], bounds[g+1]) of the I x ld matrix `base` are valid on rank g;
  // afterwards every rank holds all rows.
  virtual void allgatherv_rows(double* base, const std::vector<uint64_t>& bounds, int ld,
                               cudaStream_t s) = 0;
  // SPLATT_XCHG_PEER: make the `bytes`-long cudaMalloc allocation starting at `base`
  // (generation `gen`: bumped by the owner whenever it reallocates) addressable by every
  // rank; peers[g] = rank g's allocation as seen from this device (peers[rank] = base).
  // Collective, stream-ordered behind the work already enqueued on `s` on every rank and
  // complete on return (it is the barrier between the factor initialisation and the first
  // remote store).  Returns false on EVERY rank if any rank could not map some peer.
  virtual bool map_peers(void* base, size_t bytes, uint64_t gen, cudaStream_t s, void** peers) {
    (void)base; (void)bytes; (void)gen; (void)s; (void)peers;
    return false;
  }
};
constexpr int kMaxPeerRanks = 8;  // SPLATT_XCHG_PEER: ranks whose factor copies a solve stores to

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
  int part_mode = SPLATT_PART_AUTO;    // sharded path: P1 / P2 per mode (SPLATT_PART_*)
  int exchange = SPLATT_XCHG_COLLECTIVE;  // sharded path: how solved rows reach the peers
  // SPLATT_XCHG_PEER: the factor matrices of a sharded call live in this cudaMalloc slab
  // (IPC handles need a whole allocation), kept across calls and grown on demand.
  char* peer_slab = nullptr;
  size_t peer_slab_cap = 0;
  uint64_t peer_slab_gen = 0;
  double leaf_tile_frac = -1.0;        // ROOT MTTKRP leaf tiling (0 = off, < 0 = auto)
  bool deterministic = false;          // ROOT MTTKRP seams: fixed-order sums, no atomics
  // While a cpd_als call builds trees that only run ROOT traversals (policy ALL): the padded
  // rank their second-generation ROOT plans are for; the builder then forms the plan from the
  // sorted coordinates it already holds (root2.cu, root_plan_from_levels).  0 = no plan.
  int build_plan_ld = 0;
  // ROOT gather cache policy chosen by an earlier cpd_als call, keyed by the
  // tree's shape (order, rank padding, nonzeros, node counts, tiles): a repeated call on the
  // same tensor skips the timing iterations and their host sync.
  std::map<std::vector<uint64_t>, int> l1a_memo;
  // During an ALS call with tol > 0: device int, the iteration at which the fit stopped
  // improving (0 = still running).  Kernels of the loop return at once when it is set, so
  // the host enqueues iterations ahead without a sync per iteration (nullptr otherwise).
  const int* d_conv = nullptr;
  uint64_t host_syncs = 0;       // blocking stream syncs issued by the library
  double host_sync_s = 0.0;      // host seconds spent in them
  sb::Arena* arena_call = nullptr;       // per-call buffers of cpd_als (see sb::Arena)
  sb::Arena* arena_scratch = nullptr;    // CSF-build temporaries, reused tree to tree
  std::vector<cudaEvent_t> ev_pool;      // timing events reused across calls (EventTimer)
  std::vector<cudaEvent_t> ev_pool_aux;  // same, for spans on the aux stream
  // Side stream for the R x R work that overlaps the MTTKRP (V^-1 of the next mode, the
  // fit) and two ordering events; created on first use, owned by the context.
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_aux = nullptr, ev_solved = nullptr;
  // Host-staged COO values: uploaded on `copy` (overlapping the index upload and the sort);
  // ev_vals marks the end of the upload while vals_pending (sb::wait_vals).
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_copy_start = nullptr, ev_vals = nullptr;
  bool vals_pending = false;
  std::unique_ptr<sb::Comm> comm;
  // Pinned host staging for the call's small device->host results (status words, fit
  // history): async copies, so the host can collect timings while the device finishes.
  char* h_pinned = nullptr;
  size_t h_pinned_bytes = 0;
  char* pinned(size_t bytes) {
    if (bytes > h_pinned_bytes) {
      if (h_pinned) cudaFreeHost(h_pinned);
      h_pinned = nullptr;
      h_pinned_bytes = 0;
      const size_t want = std::max<size_t>(bytes, 4096);
      if (cudaHostAlloc((void**)&h_pinned, want, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      h_pinned_bytes = want;
    }
    return h_pinned;
  }
  ~splatt_ctx() {
    comm.reset();  // closes its mappings of the peers' slabs before ours goes
    if (peer_slab) cudaFree(peer_slab);
    if (h_pinned) cudaFreeHost(h_pinned);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_pool_aux) cudaEventDestroy(e);
    if (ev_ready) cudaEventDestroy(ev_ready);
    if (ev_aux) cudaEventDestroy(ev_aux);
    if (ev_solved) cudaEventDestroy(ev_solved);
    if (aux) cudaStreamDestroy(aux);
    if (ev_copy_start) cudaEventDestroy(ev_copy_start);
    if (ev_vals) cudaEventDestroy(ev_vals);
    if (copy) cudaStreamDestroy(copy);
    delete_arenas();
  }
  void delete_arenas();
  void ensure_copy() {
    if (copy) return;
    SB_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    SB_CUDA(cudaEventCreateWithFlags(&ev_copy_start, cudaEventDisableTiming));
    SB_CUDA(cudaEventCreateWithFlags(&ev_vals, cudaEventDisableTiming));
  }
  void ensure_aux() {
    if (aux) return;
    SB_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    SB_CUDA(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
    SB_CUDA(cudaEventCreateWithFlags(&ev_aux, cudaEventDisableTiming));
    SB_CUDA(cudaEventCreateWithFlags(&ev_solved, cudaEventDisableTiming));
  }
};

namespace sb {

// Bump arena for the device memory of one library call.  Offsets are virtual: an
// allocation that does not fit the current capacity falls back to the stream-ordered pool
// but still advances the offset, and the peak seen is the capacity the arena grows to at
// the start of the next call — so repeated calls allocate nothing.  Scopes nest LIFO
// (ArenaScope restores the offset), which lets a CSF build reuse one scratch region for
// every tree.  Work on the context stream is stream-ordered, so reusing a region after a
// scope closes is safe; the call ends with a host sync before the next call resets it.
struct Arena {
  char* base = nullptr;
  size_t cap = 0, off = 0, peak = 0;
  ~Arena() { if (base) cudaFree(base); }
  // At the start of a call (no live allocations): grow to the last call's peak.
  void reset() {
    off = 0;
    if (peak > cap) {
      if (base) cudaFree(base);
      base = nullptr;
      cap = 0;
      const size_t want = peak + peak / 16;
      // the overflow of the previous call sits in the stream-ordered pool: hand it back
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolTrimTo(pool, 0);
      if (cudaMalloc((void**)&base, want) == cudaSuccess) cap = want;
      else cudaGetLastError();  // keep working from the pool
    }
    peak = 0;
  }
  void* take(size_t bytes) {
    const size_t a = (off + 255) & ~(size_t)255;
    off = a + bytes;
    peak = std::max(peak, off);
    return (off <= cap) ? base + a : nullptr;
  }
};

}  // namespace sb

inline void splatt_ctx::delete_arenas() {
  delete arena_call;
  delete arena_scratch;
  arena_call = arena_scratch = nullptr;
}

namespace sb {

// The arena DevBuf allocations come from on this thread (nullptr: the stream-ordered pool).
inline Arena*& current_arena() {
  static thread_local Arena* a = nullptr;
  return a;
}

// Make `a` current for the scope; on exit restore the previous arena and release (LIFO)
// everything `a` handed out inside the scope if `release` is set.
struct ArenaScope {
  Arena* a;
  Arena* prev;
  size_t mark;
  bool release;
  ArenaScope(Arena* arena, bool release_on_exit)
      : a(arena), prev(current_arena()), mark(arena ? arena->off : 0), release(release_on_exit) {
    current_arena() = arena;
  }
  ~ArenaScope() {
    if (a && release) a->off = mark;
    current_arena() = prev;
  }
};

// RAII device buffer: from the current arena if one is set (release is then a no-op; the
// scope reclaims it), else on the context's stream-ordered pool (cudaMallocAsync): frees
// are stream-ordered, so no host sync is needed between ALS phases.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool pooled = false;  // true: cudaMallocAsync memory owned by this buffer
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (!count) return;
    if (Arena* a = current_arena()) p = static_cast<T*>(a->take(count * sizeof(T)));
    if (!p) {
      SB_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), stream));
      pooled = true;
    }
  }
  void release() {
    if (p && pooled && cudaFreeAsync(p, s) != cudaSuccess) cudaGetLastError();  // no stale error
    p = nullptr;
    n = 0;
    pooled = false;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), pooled(o.pooled) {
    o.p = nullptr;
    o.n = 0;
    o.pooled = false;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s; pooled = o.pooled;
      o.p = nullptr; o.n = 0; o.pooled = false;
    }
    return *this;
  }
  T* get() const { return p; }
  // Non-owning view of memory someone else frees.
  void adopt(T* ptr, size_t count) {
    release();
    p = ptr;
    n = count;
  }
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
  // Spans complete in enqueue order (one stream): collect_ready() adds those whose end event
  // has completed (non-blocking; callable while the device still runs), collect() the rest
  // (requires the stream to have completed).
  size_t cursor = 0;
  void collect_ready(double* per_cat, int ncat) {
    for (; cursor < spans.size(); ++cursor) {
      const Span& sp = spans[cursor];
      if (cudaEventQuery((*pool)[sp.b]) != cudaSuccess) {
        cudaGetLastError();  // cudaErrorNotReady is not an error
        return;
      }
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, (*pool)[sp.a], (*pool)[sp.b]) == cudaSuccess && sp.cat < ncat)
        per_cat[sp.cat] += ms * 1e-3;
    }
  }
  void collect(double* per_cat, int ncat) {
    for (; cursor < spans.size(); ++cursor) {
      const Span& sp = spans[cursor];
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
// Order the context stream after a pending host->device upload of the COO values (no-op
// otherwise).  Called right before the first kernel that reads the values.
inline void wait_vals(splatt_ctx* ctx) {
  if (!ctx->vals_pending) return;
  SB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_vals, 0));
  ctx->vals_pending = false;
}

inline void host_sync(splatt_ctx* ctx) {
  const auto t0 = std::chrono::steady_clock::now();
  SB_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->host_sync_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  ++ctx->host_syncs;
}

}  // namespace sb
