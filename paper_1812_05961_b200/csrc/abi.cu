// abi.cu — the extern "C" boundary (include/splatt_b200.h).  Argument checks, host<->
// device staging, status mapping.  No arithmetic of the method happens here.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <new>

#include "als.hpp"
#include "csf.hpp"
#include "dense.hpp"
#include "mttkrp.hpp"

using namespace sb;

namespace sb {

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace sb

namespace {

thread_local std::string g_noctx_err;

// After a failed call, wait for whatever the call had enqueued: the next call may reuse
// the context's arena memory (sb::Arena) that this work still touches.
void quiesce(splatt_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->aux) cudaStreamSynchronize(ctx->aux);
}

template <typename F>
splatt_status guard(splatt_ctx* ctx, F&& f) {
  try {
    if (ctx) ctx->err.clear();
    // A non-sticky error left by an earlier runtime call outside the library (or an ignored
    // status) must not be reported by this call's first launch check.
    const cudaError_t pending = cudaGetLastError();
    if (pending != cudaSuccess && getenv("SPLATT_DEBUG_ERRORS"))
      fprintf(stderr, "[splatt] pending CUDA error at call entry: %s\n", cudaGetErrorString(pending));
    f();
    if (getenv("SPLATT_DEBUG_ERRORS")) {
      const cudaError_t left = cudaGetLastError();
      if (left != cudaSuccess)
        fprintf(stderr, "[splatt] CUDA error left by the call: %s\n", cudaGetErrorString(left));
    }
    return SPLATT_OK;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.what(); else g_noctx_err = e.what();
    quiesce(ctx);
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "host allocation failed";
    quiesce(ctx);
    return SPLATT_ERR_NOMEM;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    quiesce(ctx);
    return SPLATT_ERR_CUDA;
  }
}

void check_coo(const splatt_coo* coo) {
  SB_REQUIRE(coo != nullptr, "coo is NULL");
  SB_REQUIRE(coo->nmodes >= 3 && coo->nmodes <= SPLATT_MAX_NMODES, "nmodes must be in [3, 8]");
  SB_REQUIRE(coo->nnz >= 1, "no nonzeros");
  SB_REQUIRE(coo->vals != nullptr, "vals is NULL");
  for (int m = 0; m < coo->nmodes; ++m) {
    SB_REQUIRE(coo->dims[m] >= 1 && coo->dims[m] < (1ull << 32), "dims must be in [1, 2^32)");
    SB_REQUIRE(coo->ind[m] != nullptr, "ind[m] is NULL");
  }
  if (coo->nnz >= (1ull << 31)) fail(SPLATT_ERR_UNSUPPORTED, "nnz >= 2^31 not supported");
}

// Device view of a caller COO; host arrays are uploaded into owned buffers.  Host values
// go up on the context's copy stream, so their upload overlaps the index upload, the
// validation and the sort; the first kernel that reads them waits (sb::wait_vals).
struct StagedCoo {
  DevCoo view;
  DevBuf<uint32_t> ind[SPLATT_MAX_NMODES];
  DevBuf<double> vals;
  splatt_ctx* ctx_ = nullptr;
  ~StagedCoo() { if (ctx_) { try { wait_vals(ctx_); } catch (...) {} } }  // before the free
  StagedCoo(splatt_ctx* ctx, const splatt_coo* coo) : ctx_(ctx) {
    view.N = coo->nmodes;
    view.nnz = coo->nnz;
    for (int m = 0; m < coo->nmodes; ++m) {
      view.dims[m] = coo->dims[m];
      if (is_device_ptr(coo->ind[m])) {
        view.ind[m] = coo->ind[m];
      } else {
        ind[m].alloc(coo->nnz, ctx->stream);
        SB_CUDA(cudaMemcpyAsync(ind[m].p, coo->ind[m], coo->nnz * 4, cudaMemcpyHostToDevice,
                                ctx->stream));
        view.ind[m] = ind[m].p;
      }
    }
    if (is_device_ptr(coo->vals)) {
      view.vals = coo->vals;
    } else {
      vals.alloc(coo->nnz, ctx->stream);
      ctx->ensure_copy();
      SB_CUDA(cudaEventRecord(ctx->ev_copy_start, ctx->stream));  // after the allocation
      SB_CUDA(cudaStreamWaitEvent(ctx->copy, ctx->ev_copy_start, 0));
      SB_CUDA(cudaMemcpyAsync(vals.p, coo->vals, coo->nnz * 8, cudaMemcpyHostToDevice,
                              ctx->copy));
      SB_CUDA(cudaEventRecord(ctx->ev_vals, ctx->copy));
      ctx->vals_pending = true;
      view.vals = vals.p;
    }
    if (getenv("SPLATT_DEBUG_STAGING")) {
      cudaPointerAttributes at;
      cudaPointerGetAttributes(&at, coo->vals);
      auto t0 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(ctx->stream);
      auto t1 = std::chrono::steady_clock::now();
      fprintf(stderr, "[splatt] staging: vals memtype=%d, sync after enqueue %.3f ms\n",
              (int)at.type, std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
  }
};

}  // namespace

extern "C" {

const char* splatt_version(void) { return "splatt_b200 0.1 (sm_100a, fp64)"; }

splatt_status splatt_ctx_create(splatt_ctx** out, int device, void* cuda_stream) {
  if (!out) return SPLATT_ERR_BADINPUT;
  splatt_ctx* ctx = new (std::nothrow) splatt_ctx();
  if (!ctx) return SPLATT_ERR_NOMEM;
  splatt_status st = guard(ctx, [&] {
    int n = 0;
    SB_CUDA(cudaGetDeviceCount(&n));
    SB_REQUIRE(device >= 0 && device < n, "no such CUDA device");
    SB_CUDA(cudaSetDevice(device));
    ctx->device = device;
    SB_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    int l2 = 0;
    SB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
    ctx->l2_bytes = (size_t)l2;
    if (cuda_stream) {
      ctx->stream = (cudaStream_t)cuda_stream;
    } else {
      SB_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
    // Keep freed blocks in the stream-ordered pool (no re-mapping between ALS calls).
    cudaMemPool_t pool;
    SB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    SB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  });
  if (st != SPLATT_OK) {
    g_noctx_err = ctx->err;
    delete ctx;
    return st;
  }
  *out = ctx;
  return SPLATT_OK;
}

void splatt_ctx_destroy(splatt_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->comm.reset();
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

splatt_status splatt_ctx_sync(splatt_ctx* ctx) {
  if (!ctx) return SPLATT_ERR_BADINPUT;
  return guard(ctx, [&] {
    SB_CUDA(cudaStreamSynchronize(ctx->stream));
    SB_CUDA(cudaGetLastError());
  });
}

const char* splatt_last_error(const splatt_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_noctx_err.c_str();
}

splatt_status splatt_comm_unique_id(void* id128) {
  if (!id128) return SPLATT_ERR_BADINPUT;
  return guard(nullptr, [&] { nccl_unique_id(id128); });
}

splatt_status splatt_ctx_set_comm(splatt_ctx* ctx, const void* id128, int nranks, int rank) {
  if (!ctx) return SPLATT_ERR_BADINPUT;
  return guard(ctx, [&] {
    SB_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad nranks/rank");
    SB_CUDA(cudaSetDevice(ctx->device));
    if (id128 == nullptr) {  // no communicator: the unsharded single-GPU path
      SB_REQUIRE(nranks == 1, "id128 is NULL");
      ctx->comm.reset();
      return;
    }
    ctx->comm = make_nccl_comm(id128, nranks, rank);
  });
}

splatt_status splatt_ctx_set_deterministic(splatt_ctx* ctx, int32_t on) {
  if (!ctx) return SPLATT_ERR_BADINPUT;
  ctx->deterministic = on != 0;
  return SPLATT_OK;
}

splatt_status splatt_ctx_set_leaf_tiling(splatt_ctx* ctx, double l2_fraction) {
  if (!ctx || !(l2_fraction >= 0.0 || l2_fraction == SPLATT_LEAF_TILING_AUTO) ||
      l2_fraction > 4.0)
    return SPLATT_ERR_BADINPUT;
  ctx->leaf_tile_frac = l2_fraction;
  return SPLATT_OK;
}

splatt_status splatt_ctx_set_partition(splatt_ctx* ctx, int32_t mode) {
  if (!ctx || (mode != SPLATT_PART_SLICES && mode != SPLATT_PART_NNZ && mode != SPLATT_PART_AUTO))
    return SPLATT_ERR_BADINPUT;
  ctx->part_mode = mode;
  return SPLATT_OK;
}

splatt_status splatt_ctx_set_exchange(splatt_ctx* ctx, int32_t mode) {
  if (!ctx || (mode != SPLATT_XCHG_COLLECTIVE && mode != SPLATT_XCHG_PEER))
    return SPLATT_ERR_BADINPUT;
  ctx->exchange = mode;
  return SPLATT_OK;
}

splatt_status splatt_partition_nnz(const uint64_t* w, uint64_t S, int32_t G, int32_t rank,
                                   uint64_t* row_bounds, uint64_t* split, uint64_t* nsplit,
                                   splatt_nnz_share* share) {
  if (G < 1 || rank < 0 || rank >= G || (S > 0 && !w)) return SPLATT_ERR_BADINPUT;
  NnzPart np;
  host_partition_nnz(w, S, G, rank, np);
  if (row_bounds) for (int g = 0; g <= G; ++g) row_bounds[g] = np.rowb[g];
  if (split) for (size_t k = 0; k < np.slots.size(); ++k) split[k] = np.slots[k];
  if (nsplit) *nsplit = np.slots.size();
  if (share) {
    share->full_lo = np.full_lo;
    share->full_hi = np.full_hi;
    share->npart = np.npart;
    for (int q = 0; q < 2; ++q) {
      share->part_slice[q] = np.pslice[q];
      share->part_begin[q] = np.pa[q];
      share->part_end[q] = np.pb[q];
    }
  }
  return SPLATT_OK;
}

splatt_status splatt_partition(const uint64_t* w, uint64_t S, int32_t G, uint64_t* bounds) {
  if (!bounds || G < 1 || (S > 0 && !w)) return SPLATT_ERR_BADINPUT;
  host_partition(w, S, G, bounds);
  return SPLATT_OK;
}

splatt_status splatt_csf_build(splatt_ctx* ctx, const splatt_coo* coo, int32_t nmodes,
                               const uint64_t* dims, int32_t policy, splatt_csf** out) {
  if (!ctx || !out) return SPLATT_ERR_BADINPUT;
  return guard(ctx, [&] {
    check_coo(coo);
    SB_REQUIRE(nmodes == coo->nmodes, "nmodes disagrees with coo->nmodes");
    SB_REQUIRE(dims != nullptr, "dims is NULL");
    for (int m = 0; m < nmodes; ++m) SB_REQUIRE(dims[m] == coo->dims[m], "dims disagree with coo");
    SB_REQUIRE(policy == SPLATT_CSF_ALL || policy == SPLATT_CSF_ONE || policy == SPLATT_CSF_TWO,
               "unknown CSF policy");
    SB_CUDA(cudaSetDevice(ctx->device));
    StagedCoo X(ctx, coo);
    if (!validate_coo_device(ctx, X.view.ind, X.view.nnz, nmodes, X.view.dims))
      fail(SPLATT_ERR_BADINPUT, "index out of range for its mode");
    auto c = std::make_unique<splatt_csf>();
    c->N = nmodes;
    c->policy = policy;
    c->ctx = ctx;
    for (int m = 0; m < nmodes; ++m) c->dims[m] = coo->dims[m];
    int roots[SPLATT_MAX_NMODES];
    csf_policy(nmodes, c->dims, policy, &c->ncsf, roots, c->mode_csf, c->mode_level);
    DevCsf* outs[SPLATT_MAX_NMODES];
    for (int k = 0; k < c->ncsf; ++k) {
      c->csf[k] = std::make_unique<DevCsf>();
      outs[k] = c->csf[k].get();
    }
    build_csf_set(ctx, X.view.ind, X.view.vals, X.view.nnz, nmodes, X.view.dims, roots, c->ncsf,
                  outs);
    for (int m = 0; m < nmodes; ++m)
      if (c->mode_level[m] > 0) c->csf[c->mode_csf[m]]->nonroot = true;
    *out = c.release();
  });
}

splatt_status splatt_csf_info(const splatt_csf* csf, int32_t which, int32_t* nmodes,
                              int32_t* mode_perm, uint64_t* n_nodes) {
  if (!csf || which < 0 || which >= csf->ncsf) return SPLATT_ERR_BADINPUT;
  const DevCsf& c = *csf->csf[which];
  if (nmodes) *nmodes = c.N;
  for (int l = 0; l < c.N; ++l) {
    if (mode_perm) mode_perm[l] = c.perm[l];
    if (n_nodes) n_nodes[l] = c.nodes[l];
  }
  return SPLATT_OK;
}

splatt_status splatt_csf_export(const splatt_csf* csf, int32_t which, int32_t level,
                                uint32_t* ids, uint32_t* ptr, double* vals) {
  if (!csf || which < 0 || which >= csf->ncsf) return SPLATT_ERR_BADINPUT;
  splatt_ctx* ctx = csf->ctx;
  return guard(ctx, [&] {
    const DevCsf& c = *csf->csf[which];
    SB_REQUIRE(level >= 0 && level < c.N, "level out of range");
    cudaStream_t s = ctx->stream;
    if (ids)
      SB_CUDA(cudaMemcpyAsync(ids, c.ids[level].p, c.nodes[level] * 4, cudaMemcpyDeviceToHost, s));
    if (ptr && level < c.N - 1)
      SB_CUDA(cudaMemcpyAsync(ptr, c.ptr[level].p, (c.nodes[level] + 1) * 4,
                              cudaMemcpyDeviceToHost, s));
    if (vals && level == c.N - 1)
      SB_CUDA(cudaMemcpyAsync(vals, c.vals.p, c.nnz * 8, cudaMemcpyDeviceToHost, s));
    SB_CUDA(cudaStreamSynchronize(s));
  });
}

void splatt_csf_free(splatt_csf* csf) {
  if (!csf) return;
  if (csf->ctx) cudaSetDevice(csf->ctx->device);
  delete csf;
}

splatt_status splatt_csf_dispatch(const splatt_csf* csf, int32_t mode, int32_t* ncsf,
                                  int32_t* which, int32_t* level) {
  if (!csf) return SPLATT_ERR_BADINPUT;
  if ((which || level) && (mode < 0 || mode >= csf->N)) return SPLATT_ERR_BADINPUT;
  if (ncsf) *ncsf = csf->ncsf;
  if (which) *which = csf->mode_csf[mode];
  if (level) *level = csf->mode_level[mode];
  return SPLATT_OK;
}

namespace {

// MTTKRP of `mode` on CSF `which`: the kernel kind is the level of `mode` in that tree.
void mttkrp_on(splatt_ctx* ctx, const splatt_csf* csf, int which, int mode,
               const double* const* factors, int rank, int ld, double* out) {
  SB_REQUIRE(csf != nullptr && factors != nullptr && out != nullptr, "NULL argument");
  SB_REQUIRE(mode >= 0 && mode < csf->N, "mode out of range");
  SB_REQUIRE(which >= 0 && which < csf->ncsf, "CSF index out of range");
  SB_REQUIRE(rank >= 1 && rank <= SPLATT_MAX_RANK, "rank must be in [1, 128]");
  SB_REQUIRE(ld >= rank, "ld < rank");
  const int N = csf->N;
  for (int m = 0; m < N; ++m)
    if (m != mode) SB_REQUIRE(factors[m] != nullptr, "factor pointer is NULL");
  SB_CUDA(cudaSetDevice(ctx->device));
  DevCsf& c = *csf->csf[which];
  int level = 0;
  while (c.perm[level] != mode) ++level;
  cudaStream_t s = ctx->stream;
  const int ldi = padded_ld(rank);
  bool direct = (ld == ldi) && ((uintptr_t)out % 32 == 0);
  for (int m = 0; m < N; ++m)
    if (m != mode) direct = direct && ((uintptr_t)factors[m] % 32 == 0);
  if (direct) {
    mttkrp_level(ctx, c, level, factors, out, csf->dims[mode], ld, rank);
    return;
  }
  // Staging path: pack factors to the internal padded layout, then copy out.
  std::vector<DevBuf<double>> F(N);
  const double* fp[SPLATT_MAX_NMODES] = {nullptr};
  for (int m = 0; m < N; ++m) {
    if (m == mode) continue;
    F[m].alloc(csf->dims[m] * ldi, s);
    SB_CUDA(cudaMemsetAsync(F[m].p, 0, csf->dims[m] * ldi * 8, s));
    SB_CUDA(cudaMemcpy2DAsync(F[m].p, ldi * 8, factors[m], (size_t)ld * 8, (size_t)rank * 8,
                              csf->dims[m], cudaMemcpyDeviceToDevice, s));
    fp[m] = F[m].p;
  }
  DevBuf<double> O(csf->dims[mode] * ldi, s);
  mttkrp_level(ctx, c, level, fp, O.p, csf->dims[mode], ldi, rank);
  SB_CUDA(cudaMemsetAsync(out, 0, csf->dims[mode] * (size_t)ld * 8, s));
  SB_CUDA(cudaMemcpy2DAsync(out, (size_t)ld * 8, O.p, ldi * 8, (size_t)rank * 8, csf->dims[mode],
                            cudaMemcpyDeviceToDevice, s));
}

}  // namespace

splatt_status splatt_mttkrp(splatt_ctx* ctx, const splatt_csf* csf, int32_t mode,
                            const double* const* factors, int32_t rank, int32_t ld,
                            double* out) {
  if (!ctx) return SPLATT_ERR_BADINPUT;
  return guard(ctx, [&] {
    SB_REQUIRE(csf != nullptr, "NULL argument");
    SB_REQUIRE(mode >= 0 && mode < csf->N, "mode out of range");
    mttkrp_on(ctx, csf, csf->mode_csf[mode], mode, factors, rank, ld, out);
  });
}

splatt_status splatt_mttkrp_csf(splatt_ctx* ctx, const splatt_csf* csf, int32_t which,
                                int32_t mode, const double* const* factors, int32_t rank,
                                int32_t ld, double* out) {
  if (!ctx) return SPLATT_ERR_BADINPUT;
  return guard(ctx, [&] { mttkrp_on(ctx, csf, which, mode, factors, rank, ld, out); });
}

splatt_status splatt_cpd_als_ex(splatt_ctx* ctx, const splatt_coo* coo, int32_t rank,
                                int32_t max_iters, double tol, uint64_t seed,
                                const double* const* init_factors, int32_t policy,
                                splatt_kruskal* out, splatt_stats* stats) {
  if (!ctx) return SPLATT_ERR_BADINPUT;
  const auto t0 = std::chrono::steady_clock::now();
  return guard(ctx, [&] {
    check_coo(coo);
    SB_REQUIRE(rank >= 1 && rank <= SPLATT_MAX_RANK, "rank must be in [1, 128]");
    SB_REQUIRE(max_iters >= 1, "max_iters must be >= 1");
    SB_REQUIRE(tol >= 0.0, "tol must be >= 0");
    SB_REQUIRE(policy == SPLATT_CSF_ALL || policy == SPLATT_CSF_ONE || policy == SPLATT_CSF_TWO,
               "unknown CSF policy");
    if (ctx->comm && policy != SPLATT_CSF_ALL)
      fail(SPLATT_ERR_UNSUPPORTED, "a sharded context requires policy ALL");
    SB_REQUIRE(out != nullptr && out->lambda != nullptr, "NULL output");
    for (int m = 0; m < coo->nmodes; ++m) SB_REQUIRE(out->factors[m] != nullptr, "NULL factor out");
    if (init_factors)
      for (int m = 0; m < coo->nmodes; ++m) SB_REQUIRE(init_factors[m] != nullptr, "NULL init");
    SB_CUDA(cudaSetDevice(ctx->device));
    if (stats) std::memset(stats, 0, sizeof(*stats));
    StagedCoo X(ctx, coo);
    AlsOut o{};
    for (int m = 0; m < coo->nmodes; ++m) o.factors[m] = out->factors[m];
    o.lambda = out->lambda;
    o.fit = &out->fit;
    o.iters = &out->iters;
    o.fit_history = out->fit_history;
    static const bool trace = getenv("SPLATT_TRACE") != nullptr;
    const auto t1 = std::chrono::steady_clock::now();
    cpd_als_device(ctx, X.view, rank, max_iters, tol, seed, init_factors, policy, o, stats);
    if (trace)
      fprintf(stderr, "[splatt trace] cpd_als host: staging %.3f ms, driver %.3f ms\n",
              std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1)
                  .count());
  });
}

splatt_status splatt_cpd_als_csf(splatt_ctx* ctx, const splatt_csf* csf, int32_t rank,
                                 int32_t max_iters, double tol, uint64_t seed,
                                 const double* const* init_factors, splatt_kruskal* out,
                                 splatt_stats* stats) {
  if (!ctx) return SPLATT_ERR_BADINPUT;
  return guard(ctx, [&] {
    SB_REQUIRE(csf != nullptr && csf->ncsf >= 1, "NULL CSF");
    SB_REQUIRE(rank >= 1 && rank <= SPLATT_MAX_RANK, "rank must be in [1, 128]");
    SB_REQUIRE(max_iters >= 1, "max_iters must be >= 1");
    SB_REQUIRE(tol >= 0.0, "tol must be >= 0");
    SB_REQUIRE(out != nullptr && out->lambda != nullptr, "NULL output");
    for (int m = 0; m < csf->N; ++m) SB_REQUIRE(out->factors[m] != nullptr, "NULL factor out");
    if (init_factors)
      for (int m = 0; m < csf->N; ++m) SB_REQUIRE(init_factors[m] != nullptr, "NULL init");
    if (ctx->comm)
      fail(SPLATT_ERR_UNSUPPORTED, "a prebuilt CSF set runs on an unsharded context only");
    SB_CUDA(cudaSetDevice(ctx->device));
    if (stats) std::memset(stats, 0, sizeof(*stats));
    DevCoo X;
    X.N = csf->N;
    X.nnz = csf->csf[0]->nnz;
    for (int m = 0; m < csf->N; ++m) X.dims[m] = csf->dims[m];
    AlsOut o{};
    for (int m = 0; m < csf->N; ++m) o.factors[m] = out->factors[m];
    o.lambda = out->lambda;
    o.fit = &out->fit;
    o.iters = &out->iters;
    o.fit_history = out->fit_history;
    cpd_als_device(ctx, X, rank, max_iters, tol, seed, init_factors, csf->policy, o, stats, csf);
  });
}

splatt_status splatt_cpd_als(splatt_ctx* ctx, const splatt_coo* coo, int32_t rank,
                             int32_t max_iters, double tol, uint64_t seed, splatt_kruskal* out) {
  return splatt_cpd_als_ex(ctx, coo, rank, max_iters, tol, seed, nullptr, SPLATT_CSF_ALL, out,
                           nullptr);
}

}  // extern "C"
