// als.cu — the CP-ALS driver (Algorithm 1).
//
// Host loop over iterations and modes; every step is a kernel on the context stream,
// there is no host round trip inside an iteration (the only device->host read per
// iteration is the fit, and only when tol > 0).  With a communicator the path is
// sharded: per mode the root slices are cut into contiguous ranges
// balanced on nnz (C-14), each rank builds the CSF of its own nonzeros, solves its own
// rows, and the Gram/inner/colmax statistics and the updated rows are exchanged.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>

#include "als.hpp"
#include "csf.hpp"
#include "dense.hpp"
#include "mttkrp.hpp"

namespace sb {

namespace {

enum Cat { kMttkrp = 0, kBuild, kAta, kNorm, kFit, kInverse, kComm, kLoop, kNumCat };

__global__ void histogram_kernel(const uint32_t* __restrict__ ind, uint64_t nnz,
                                 unsigned long long* __restrict__ cnt) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ind[j]], 1ull);
}

__global__ void owned_flags_kernel(const uint32_t* __restrict__ ind, uint64_t nnz, uint32_t lo,
                                   uint32_t hi, uint32_t* __restrict__ flag) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x)
    flag[j] = (ind[j] >= lo && ind[j] < hi) ? 1u : 0u;
}

__global__ void eq_flags_kernel(const uint32_t* __restrict__ ind, uint64_t nnz, uint32_t v,
                                uint32_t* __restrict__ flag) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x)
    flag[j] = (ind[j] == v) ? 1u : 0u;
}

// P2 share of this rank: whole slices [lo, hi) plus, for up to two partial slices ps[j], the
// nonzeros whose rank within the slice (input order, rk[j] = exclusive scan of "in slice")
// lies in [a[j], b[j]).
struct NnzShare {
  uint32_t lo, hi;
  int np;
  uint32_t ps[2];
  const uint32_t* rk[2];
  uint64_t a[2], b[2];
};
__global__ void nnz_share_flags_kernel(const uint32_t* __restrict__ ind, uint64_t nnz, NnzShare sh,
                                       uint32_t* __restrict__ flag) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = ind[j];
    bool take = (i >= sh.lo && i < sh.hi);
    for (int q = 0; q < sh.np; ++q)
      if (i == sh.ps[q]) {
        const uint64_t r = sh.rk[q][j];
        take = take || (r >= sh.a[q] && r < sh.b[q]);
      }
    flag[j] = take ? 1u : 0u;
  }
}

struct Compact {
  const uint32_t* src[SPLATT_MAX_NMODES];
  uint32_t* dst[SPLATT_MAX_NMODES];
  int N;
};

// Stable compaction: flag[j] (0/1) and its exclusive scan pos[j].
__global__ void compact_kernel(Compact c, const double* __restrict__ vin, double* __restrict__ vout,
                               const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                               uint64_t nnz) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    if (flag[j]) {
      const uint32_t k = pos[j];
      for (int m = 0; m < c.N; ++m) c.dst[m][k] = c.src[m][j];
      vout[k] = vin[j];
    }
  }
}

int blocks_for(splatt_ctx* ctx, uint64_t n) {
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n, 256), (uint64_t)ctx->num_sms * 16));
}

}  // namespace

void host_partition(const uint64_t* w, uint64_t S, int G, uint64_t* bounds) {
  // C-14 reading: smallest feasible cap by bisection, then
  // leftmost-greedy boundaries under it.
  auto feasible = [&](uint64_t cap) {
    int parts = 1;
    uint64_t cur = 0;
    for (uint64_t s = 0; s < S; ++s) {
      if (w[s] > cap) return false;
      if (cur + w[s] > cap) { ++parts; cur = 0; }
      cur += w[s];
    }
    return parts <= G;
  };
  uint64_t lo = 0, hi = 0;
  for (uint64_t s = 0; s < S; ++s) { lo = std::max(lo, w[s]); hi += w[s]; }
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (feasible(mid)) hi = mid; else lo = mid + 1;
  }
  uint64_t s = 0;
  bounds[0] = 0;
  for (int g = 0; g < G; ++g) {
    uint64_t cur = 0;
    while (s < S && cur + w[s] <= lo) { cur += w[s]; ++s; }
    bounds[g + 1] = s;
  }
  bounds[G] = S;
}

void host_partition_nnz(const uint64_t* w, uint64_t S, int G, int me, NnzPart& out) {
  std::vector<uint64_t> P(S + 1, 0);  // P[s] = position of slice s's first nonzero
  for (uint64_t t = 0; t < S; ++t) P[t + 1] = P[t] + w[t];
  const uint64_t nnz = P[S];
  auto cut = [&](int g) { return (uint64_t)((unsigned __int128)nnz * (unsigned)g / (unsigned)G); };
  out = NnzPart{};
  out.rowb.assign(G + 1, S);
  out.rowb[0] = 0;
  for (int g = 1; g < G; ++g)  // first slice starting at or after k_g
    out.rowb[g] = (uint64_t)(std::lower_bound(P.begin(), P.begin() + S, cut(g)) - P.begin());
  for (int g = 1; g < G; ++g) {  // slices strictly containing a cut (ascending, distinct)
    const uint64_t k = cut(g);
    if (k == 0 || k >= nnz) continue;
    const uint64_t sl = (uint64_t)(std::upper_bound(P.begin(), P.begin() + S + 1, k) - P.begin()) - 1;
    if (P[sl] < k && (out.slots.empty() || out.slots.back() != sl)) out.slots.push_back(sl);
  }
  const uint64_t k0 = cut(me), k1 = cut(me + 1);
  if (k1 <= k0) { out.full_lo = out.full_hi = 0; return; }
  // slices holding this rank's first and last nonzero
  const uint64_t s0 = (uint64_t)(std::upper_bound(P.begin(), P.begin() + S + 1, k0) - P.begin()) - 1;
  const uint64_t s1 = (uint64_t)(std::upper_bound(P.begin(), P.begin() + S + 1, k1 - 1) - P.begin()) - 1;
  auto slot_of = [&](uint64_t sl) {
    for (size_t j = 0; j < out.slots.size(); ++j)
      if (out.slots[j] == sl) return (int)j;
    return -1;
  };
  out.full_lo = s0;
  out.full_hi = s1 + 1;
  const bool first_partial = P[s0] < k0 || P[s0 + 1] > k1;
  if (first_partial) {
    out.pslice[out.npart] = s0;
    out.pa[out.npart] = k0 - P[s0];
    out.pb[out.npart] = std::min(P[s0 + 1], k1) - P[s0];
    out.pslot[out.npart] = slot_of(s0);
    ++out.npart;
    out.full_lo = s0 + 1;
  }
  if (s1 != s0 && P[s1 + 1] > k1) {
    out.pslice[out.npart] = s1;
    out.pa[out.npart] = 0;
    out.pb[out.npart] = k1 - P[s1];
    out.pslot[out.npart] = slot_of(s1);
    ++out.npart;
    out.full_hi = s1;
  }
  if (out.full_hi < out.full_lo) out.full_hi = out.full_lo;
}

void cpd_als_device(splatt_ctx* ctx, const DevCoo& X, int R, int max_iters, double tol,
                    uint64_t seed, const double* const* init, int policy, const AlsOut& out,
                    splatt_stats* st, const splatt_csf* prebuilt) {
  cudaStream_t s = ctx->stream;
  const int N = X.N;
  const int ld = padded_ld(R);
  const int G = ctx->comm ? ctx->comm->nranks : 1;
  const int me = ctx->comm ? ctx->comm->rank : 0;
  const bool sharded = ctx->comm != nullptr;  // also a 1-rank communicator (path tests)
  EventTimer tm, tma;  // main-stream and aux-stream spans
  tm.init(&ctx->ev_pool, s, st != nullptr);
  ctx->ensure_aux();
  cudaStream_t aux = ctx->aux;
  tma.init(&ctx->ev_pool_aux, aux, st != nullptr);
  const auto h_start = std::chrono::steady_clock::now();
  // Every device buffer of this call comes from the context's arenas (grown to the previous
  // call's peak, so a repeated call allocates nothing; see sb::Arena).
  if (!ctx->arena_call) ctx->arena_call = new Arena();
  if (!ctx->arena_scratch) ctx->arena_scratch = new Arena();
  ctx->arena_call->reset();
  ctx->arena_scratch->reset();
  ArenaScope call_scope(ctx->arena_call, false);
  // Leaf tiling AUTO (splatt_ctx_set_leaf_tiling): half-L2 tiles for runs of >= 10
  // iterations, where the one-time split pays for itself; restored on return.
  struct TileMode {
    splatt_ctx* c;
    double saved;
    ~TileMode() { c->leaf_tile_frac = saved; }
  } tile_mode{ctx, ctx->leaf_tile_frac};
  if (ctx->leaf_tile_frac < 0.0) ctx->leaf_tile_frac = max_iters >= 10 ? 0.5 : 0.0;
  uint64_t launches0 = ctx->kernel_launches;
  const uint64_t syncs0 = ctx->host_syncs;
  const double sync_s0 = ctx->host_sync_s;
  cudaEvent_t call_a = nullptr, call_b = nullptr;
  if (st) {
    SB_CUDA(cudaEventCreate(&call_a));
    SB_CUDA(cudaEventCreate(&call_b));
    SB_CUDA(cudaEventRecord(call_a, s));
  }

  // ---------------------------------------------------------------- validate
  tm.begin(kBuild);
  PhaseTrace tr(s, "cpd_als");
  DevBuf<int> bad(1, s);
  SB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
  if (!prebuilt) validate_coo_enqueue(ctx, X.ind, X.nnz, N, X.dims, bad.p);
  DevBuf<double> normx(1, s);
  // ||X||^2 from the COO values, or from the leaf values of a prebuilt tree (the same
  // numbers in another order: the sum differs by rounding only).  Unsharded with host-staged
  // values, it is taken after the build instead (the upload overlaps the sort) and checked
  // at the end of the call (EMPTY then takes precedence over the other statuses).
  const bool late_norm = !sharded && !prebuilt && ctx->vals_pending;
  double h_normx = 0.0;
  int h_bad = 0;
  if (!late_norm) {
    wait_vals(ctx);
    norm_sq(ctx, prebuilt ? prebuilt->csf[0]->vals.p : X.vals, X.nnz, normx.p);
    SB_CUDA(cudaMemcpyAsync(&h_normx, normx.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  SB_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  host_sync(ctx);
  if (h_bad) fail(SPLATT_ERR_BADINPUT, "index out of range for its mode");
  tr.mark("validate");
  if (!late_norm && !(h_normx > 0.0)) fail(SPLATT_ERR_EMPTY, "||X|| = 0");

  // ------------------------------------------- partition + CSF build per mode
  // Unsharded: the policy's CSFs (ALL / ONE / TWO); mode n runs its MTTKRP on
  // csf[mode_csf[n]] at level mode_level[n].  Sharded: ALL, one local CSF per mode.
  if (sharded && policy != SPLATT_CSF_ALL)
    fail(SPLATT_ERR_UNSUPPORTED, "a sharded context requires policy ALL");
  int ncsf = 0, roots[SPLATT_MAX_NMODES], mode_csf[SPLATT_MAX_NMODES], mode_level[SPLATT_MAX_NMODES];
  if (prebuilt) {
    ncsf = prebuilt->ncsf;
    for (int n = 0; n < N; ++n) {
      mode_csf[n] = prebuilt->mode_csf[n];
      mode_level[n] = prebuilt->mode_level[n];
    }
  } else {
    csf_policy(N, X.dims, policy, &ncsf, roots, mode_csf, mode_level);
  }
  std::vector<std::vector<uint64_t>> bounds(N);
  std::vector<NnzPart> nnzpart(N);  // P2 modes only
  std::vector<bool> used_p2(N, false);
  size_t max_slots = 0;
  std::vector<std::unique_ptr<DevCsf>> owned(std::max(N, ncsf));  // trees built by this call
  std::vector<DevCsf*> csf(std::max(N, ncsf), nullptr);
  if (prebuilt) {
    for (int n = 0; n < N; ++n) bounds[n] = {0, X.dims[n]};
    for (int k = 0; k < ncsf; ++k) csf[k] = prebuilt->csf[k].get();
  } else if (!sharded) {
    for (int n = 0; n < N; ++n) bounds[n] = {0, X.dims[n]};
    for (int k = 0; k < ncsf; ++k) {
      owned[k] = std::make_unique<DevCsf>();
      csf[k] = owned[k].get();
    }
    struct PlanScope {  // ROOT plans formed during the build (policy ALL: every tree ROOT)
      splatt_ctx* c;
      ~PlanScope() { c->build_plan_ld = 0; }
    } plan_scope{ctx};
    ctx->build_plan_ld = (policy == SPLATT_CSF_ALL) ? ld : 0;
    build_csf_set(ctx, X.ind, X.vals, X.nnz, N, X.dims, roots, ncsf, csf.data());
    ctx->build_plan_ld = 0;
    for (int n = 0; n < N; ++n)
      if (mode_level[n] > 0) csf[mode_csf[n]]->nonroot = true;
    if (late_norm) {
      wait_vals(ctx);  // (the build's decode already did)
      norm_sq(ctx, X.vals, X.nnz, normx.p);
    }
  }
  for (int n = 0; n < N && sharded; ++n) {
    owned[n] = std::make_unique<DevCsf>();
    csf[n] = owned[n].get();
    // this mode's selection / compaction temporaries live in the scratch arena; the local
    // tree is built into the call arena (build_csf nests its own scratch scope above ours)
    Arena* const call_arena = current_arena();
    ArenaScope tmp_scope(call_arena ? ctx->arena_scratch : nullptr, true);
    DevBuf<unsigned long long> cnt(X.dims[n], s);
    SB_CUDA(cudaMemsetAsync(cnt.p, 0, X.dims[n] * 8, s));
    histogram_kernel<<<blocks_for(ctx, X.nnz), 256, 0, s>>>(X.ind[n], X.nnz, cnt.p);
    SB_CHECK_LAUNCH(ctx);
    std::vector<uint64_t> hc(X.dims[n]);
    SB_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, X.dims[n] * 8, cudaMemcpyDeviceToHost, s));
    host_sync(ctx);
    DevBuf<uint32_t> flag(X.nnz, s), pos(X.nnz, s);
    uint64_t local = 0;
    std::vector<DevBuf<uint32_t>> rk(2);
    bool use_p2 = ctx->part_mode == SPLATT_PART_NNZ;
    if (ctx->part_mode == SPLATT_PART_AUTO) {
      // P2 only where the best whole-slice cut leaves a rank with enough excess nonzeros to
      // outweigh the extra small all-reduce per mode
      std::vector<uint64_t> b1(G + 1);
      host_partition(hc.data(), X.dims[n], G, b1.data());
      uint64_t mx = 0;
      for (int g = 0; g < G; ++g) {
        uint64_t load = 0;
        for (uint64_t i = b1[g]; i < b1[g + 1]; ++i) load += hc[i];
        mx = std::max(mx, load);
      }
      const double mean = (double)X.nnz / G;
      use_p2 = (double)mx - mean > std::max(0.01 * mean, (double)(1u << 18));
    }
    used_p2[n] = use_p2;
    if (use_p2) {  // P2: equal leaf ranges, slices may split
      host_partition_nnz(hc.data(), X.dims[n], G, me, nnzpart[n]);
      const NnzPart& np = nnzpart[n];
      bounds[n] = np.rowb;
      NnzShare sh{};
      sh.lo = (uint32_t)np.full_lo;
      sh.hi = (uint32_t)np.full_hi;
      sh.np = np.npart;
      for (uint64_t i = np.full_lo; i < np.full_hi; ++i) local += hc[i];
      for (int q = 0; q < np.npart; ++q) {
        rk[q].alloc(X.nnz, s);
        eq_flags_kernel<<<blocks_for(ctx, X.nnz), 256, 0, s>>>(X.ind[n], X.nnz,
                                                               (uint32_t)np.pslice[q], flag.p);
        SB_CHECK_LAUNCH(ctx);
        size_t tb = 0;
        SB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, rk[q].p, (int)X.nnz, s));
        DevBuf<uint8_t> temp(tb, s);
        SB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, flag.p, rk[q].p, (int)X.nnz, s));
        sh.ps[q] = (uint32_t)np.pslice[q];
        sh.rk[q] = rk[q].p;
        sh.a[q] = np.pa[q];
        sh.b[q] = np.pb[q];
        local += np.pb[q] - np.pa[q];
      }
      nnz_share_flags_kernel<<<blocks_for(ctx, X.nnz), 256, 0, s>>>(X.ind[n], X.nnz, sh, flag.p);
      SB_CHECK_LAUNCH(ctx);
      max_slots = std::max(max_slots, np.slots.size());
    } else {  // P1 (C-14): contiguous whole-slice ranges balanced on nnz
      bounds[n].assign(G + 1, 0);
      host_partition(hc.data(), X.dims[n], G, bounds[n].data());
      const uint32_t lo = (uint32_t)bounds[n][me], hi = (uint32_t)bounds[n][me + 1];
      owned_flags_kernel<<<blocks_for(ctx, X.nnz), 256, 0, s>>>(X.ind[n], X.nnz, lo, hi, flag.p);
      SB_CHECK_LAUNCH(ctx);
      for (uint64_t i = lo; i < hi; ++i) local += hc[i];
    }
    size_t tb = 0;
    SB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, pos.p, (int)X.nnz, s));
    DevBuf<uint8_t> temp(tb, s);
    SB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, flag.p, pos.p, (int)X.nnz, s));
    if (local == 0) {  // a rank with no nonzeros of this mode: empty CSF
      csf[n]->N = N;
      csf[n]->nnz = 0;
      continue;
    }
    DevBuf<uint32_t> lind[SPLATT_MAX_NMODES];
    DevBuf<double> lval(local, s);
    Compact c{};
    c.N = N;
    for (int m = 0; m < N; ++m) {
      lind[m].alloc(local, s);
      c.src[m] = X.ind[m];
      c.dst[m] = lind[m].p;
    }
    compact_kernel<<<blocks_for(ctx, X.nnz), 256, 0, s>>>(c, X.vals, lval.p, flag.p, pos.p, X.nnz);
    SB_CHECK_LAUNCH(ctx);
    const uint32_t* lp[SPLATT_MAX_NMODES];
    for (int m = 0; m < N; ++m) lp[m] = lind[m].p;
    ArenaScope back(call_arena, false);
    ctx->build_plan_ld = ld;  // sharded: every local tree runs ROOT
    try {
      build_csf(ctx, lp, lval.p, local, N, X.dims, n, *csf[n]);
    } catch (...) {
      ctx->build_plan_ld = 0;
      throw;
    }
    ctx->build_plan_ld = 0;
  }
  for (int n = 0; n < N; ++n)  // chunk tables / hot ids before the loop (no syncs inside it)
    mttkrp_prepare(ctx, *csf[sharded ? n : mode_csf[n]], sharded ? 0 : mode_level[n], ld);
  // The loop's MTTKRPs share each tree's chunk counter, zeroed once here (DevCsf::work_seq);
  // the sequence ends with the call, also on an error.
  struct WorkSeq {
    std::vector<DevCsf*> trees;
    ~WorkSeq() { for (DevCsf* t : trees) { t->work_seq = false; } }
  } work_seq;
  for (int k = 0; k < (sharded ? N : ncsf); ++k) {
    DevCsf* c = csf[k];
    if (!c || !c->nnz) continue;
    std::vector<DevCsf*> ts{c};
    for (auto& t : c->tiles) ts.push_back(t.get());
    for (DevCsf* t : ts) {
      ArenaScope own(t->arena, false);
      if (t->work.n < 1) t->work.alloc(1, s);
      SB_CUDA(cudaMemsetAsync(t->work.p, 0, sizeof(unsigned), s));
      t->work_base = 0;
      t->work_seq = true;
      work_seq.trees.push_back(t);
    }
  }
  tm.end();
  tr.mark("csf builds");

  // -------------------------------------------------------------- factors
  std::vector<DevBuf<double>> A(N);
  uint64_t maxI = 0, base = 0;
  // SPLATT_XCHG_PEER: the factors live in the context's cudaMalloc slab (one IPC handle maps
  // all of them into the peers), at offsets every rank computes alike.
  // (also with a one-rank communicator: no peers, but the mapping exchange runs)
  const bool want_peer = sharded && G <= kMaxPeerRanks && ctx->exchange == SPLATT_XCHG_PEER;
  size_t slab_off[SPLATT_MAX_NMODES + 1] = {0};
  for (int n = 0; n < N; ++n)
    slab_off[n + 1] = slab_off[n] + ((X.dims[n] * ld * sizeof(double) + 255) & ~(size_t)255);
  if (want_peer && slab_off[N] > ctx->peer_slab_cap) {
    // (every remote store into the old slab landed before the previous call returned: its
    // last solve was followed by an all-reduce on every rank)
    if (ctx->peer_slab) SB_CUDA(cudaFree(ctx->peer_slab));
    ctx->peer_slab = nullptr;
    ctx->peer_slab_cap = 0;
    SB_CUDA(cudaMalloc((void**)&ctx->peer_slab, slab_off[N]));
    ctx->peer_slab_cap = slab_off[N];
    ++ctx->peer_slab_gen;
  }
  for (int n = 0; n < N; ++n) {
    if (want_peer) A[n].adopt(reinterpret_cast<double*>(ctx->peer_slab + slab_off[n]), X.dims[n] * ld);
    else A[n].alloc(X.dims[n] * ld, s);
    maxI = std::max(maxI, X.dims[n]);
    if (init) {
      SB_CUDA(cudaMemsetAsync(A[n].p, 0, X.dims[n] * ld * sizeof(double), s));
      SB_CUDA(cudaMemcpy2DAsync(A[n].p, ld * sizeof(double), init[n], R * sizeof(double),
                                R * sizeof(double), X.dims[n], cudaMemcpyDefault, s));
    } else {
      init_factor(ctx, A[n].p, X.dims[n], R, ld, seed, base);   // C-2
    }
    base += X.dims[n] * (uint64_t)R;
  }
  const double* fac[SPLATT_MAX_NMODES] = {nullptr};
  for (int n = 0; n < N; ++n) fac[n] = A[n].p;
  const size_t RR = (size_t)R * R;
  DevBuf<double> Gall(N * RR, s), stats(stats_len(R), s), Vinv((size_t)ld * ld, s), lambda(R, s),
      inner(1, s), M(maxI * ld, s), fit_hist(max_iters, s), nu(R, s), sig((size_t)N * R, s),
      tau(R, s);
  DevBuf<int> status(1, s);
  DevBuf<unsigned> ticket(1, s);
  DevBuf<double> xslots(std::max<size_t>(1, max_slots) * ld, s);  // P2 split-row exchange
  SB_CUDA(cudaMemsetAsync(status.p, 0, sizeof(int), s));
  SB_CUDA(cudaMemsetAsync(ticket.p, 0, sizeof(unsigned), s));
  // The factors stay unnormalised in memory: A_n = stored_n * diag(sig_n);
  // MTTKRP runs on the stored rows and the solve maps the result back with tau.
  fill(ctx, sig.p, (size_t)N * R, 1.0);
  SB_CUDA(cudaMemsetAsync(fit_hist.p, 0, max_iters * sizeof(double), s));
  tm.gap();
  tm.begin(kAta);
  for (int n = 0; n < N; ++n) {   // initial Grams (C-4); factors are replicated
    rows_solve_stats(ctx, nullptr, A[n].p, 0, X.dims[n], R, ld, nullptr, nullptr, false, false,
                     nullptr, stats.p);
    gram_from_stats(ctx, stats.p, R, Gall.p + n * RR);
  }
  tm.end();

  // A/B knob, off by default (SPLATT_L2_PERSIST=<MB of set-aside>): the factor matrices as a
  // persisting L2 window around the loop.  It showed that the streamed tree records evict
  // gathered rows (c5: 2.394 -> 2.325 ms per launch); the kernels' evict-first hint on the
  // record stream (root2.cuh, SB_ROOT2_EVICT) removes the cause instead (2.240 ms, the window
  // adds nothing on top) without a device-wide limit, a host sync, or the set-aside's cost to
  // the CSF build (profiles/ab_r02/l2p/, evict/).
  struct L2Window {
    cudaStream_t s = nullptr;
    bool on = false;
    ~L2Window() {
      if (!on) return;
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.num_bytes = 0;
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
      cudaCtxResetPersistingL2Cache();
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
      cudaGetLastError();
    }
  } l2win;
  {
    const char* e = getenv("SPLATT_L2_PERSIST");
    const char* lo = reinterpret_cast<const char*>(A[0].p);
    const char* hi = lo;
    for (int n = 0; n < N; ++n) {
      lo = std::min(lo, reinterpret_cast<const char*>(A[n].p));
      hi = std::max(hi, reinterpret_cast<const char*>(A[n].p + X.dims[n] * ld));
    }
    const size_t win = (size_t)(hi - lo);
    int maxwin = 0, maxpersist = 0;
    cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
    cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
    size_t aside = 0;
    bool want = false;
    if (e) {
      want = atoi(e) > 0 && win <= (size_t)maxwin;
      aside = (size_t)atoi(e) << 20;
    }
    if (want) {
      host_sync(ctx);  // the build is done: the set-aside must not shrink its L2
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = const_cast<char*>(lo);
      v.accessPolicyWindow.num_bytes = win;
      v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)aside / (float)win);
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, aside) == cudaSuccess &&
          cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess) {
        l2win.s = s;
        l2win.on = true;
      } else {
        cudaGetLastError();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
        cudaGetLastError();
      }
    }
    if (e && getenv("SPLATT_TRACE"))
      fprintf(stderr, "[splatt] L2 persisting window: factors %zu bytes, set-aside %zu (max %d), %s\n",
              win, aside, maxpersist, l2win.on ? "on" : "off");
  }

  // Peer exchange: map the slabs after the factor initialisation and the initial Grams are
  // enqueued (the exchange of handles is stream-ordered behind them on every rank: no rank
  // stores into a peer's matrix before the peer has initialised and read it).
  PeerRows peer_rows[SPLATT_MAX_NMODES] = {};
  bool peer_x = false;
  if (want_peer) {
    void* bases[kMaxPeerRanks] = {nullptr};
    tm.begin(kComm);
    // (the slab's capacity, not this call's extent: it is what the handle covers, and
    // ranks given the same tensor hold the same capacity)
    peer_x = ctx->comm->map_peers(ctx->peer_slab, ctx->peer_slab_cap, ctx->peer_slab_gen, s, bases);
    ++ctx->host_syncs;
    tm.end();
    for (int n = 0; n < N && peer_x; ++n)
      for (int g = 0; g < G; ++g)
        if (g != me)
          peer_rows[n].p[peer_rows[n].n++] =
              reinterpret_cast<double*>(static_cast<char*>(bases[g]) + slab_off[n]);
  }

  // ----------------------------------------------------------------- loop
  DevBuf<double> rpart(rows_partials_cap(ctx, R), s);  // per-CTA solve partials (RowsReduce)
  double mttkrp_bytes = 0.0, mttkrp_min = 0.0;
  uint64_t mttkrp_launches = 0;
  // Rows of each mode a launch can reference, for the compulsory-traffic figure: the root
  // node count of the mode's own (whole-tensor) tree, else min(I_m, nodes at its level).
  auto min_bytes = [&](const DevCsf& c, int level) {
    uint64_t distinct[SPLATT_MAX_NMODES] = {0};
    for (int l = 0; l < N; ++l) {
      const int m = c.perm[l];
      uint64_t d = l == 0 ? c.nodes[0] : std::min<uint64_t>(c.dims[l], c.nodes[l]);
      if (!sharded)
        for (int k = 0; k < ncsf; ++k)
          if (csf[k]->perm[0] == m) d = std::min<uint64_t>(d, csf[k]->nodes[0]);
      distinct[m] = d;
    }
    return mttkrp_min_bytes(c, R, level, distinct);
  };
  std::vector<double> h_hist(max_iters, 0.0);
  int it_done = 0;
  cudaEvent_t loop_a = nullptr, loop_b = nullptr;
  SB_CUDA(cudaEventCreate(&loop_a));
  SB_CUDA(cudaEventCreate(&loop_b));
  SB_CUDA(cudaEventRecord(loop_a, s));
  // The R x R steps that do not feed the MTTKRP run on the aux stream, overlapped with
  // it: V^-1 of mode n is formed as soon as the Grams it needs are final (after mode
  // n-1's Gram refresh) while the main stream scales A_{n-1} and runs MTTKRP_n; the fit
  // of an iteration runs there too.  Ordering: ev_ready (main -> aux) after each Gram
  // refresh, ev_aux (aux -> main) before each solve.  Buffers shared by the two streams
  // (Vinv, Gall, lambda, inner, status) are written by one side only after the other
  // side's reads are ordered before it by these two events.
  // Convergence (C-11) without a host round trip per iteration: with tol > 0 the fit kernel
  // marks the iteration at which |fit_it - fit_{it-1}| < tol in a device word, every loop
  // kernel returns at once when it is set (splatt_ctx::d_conv), and the host reads it only
  // every kCheck iterations — the state is the converged one, the extra iterations are
  // no-ops.
  constexpr int kCheck = 8;
  const bool check = tol > 0.0;
  DevBuf<int> conv(1, s);
  SB_CUDA(cudaMemsetAsync(conv.p, 0, sizeof(int), s));
  struct ConvScope {
    splatt_ctx* c;
    ~ConvScope() { c->d_conv = nullptr; }
  } conv_scope{ctx};
  ctx->d_conv = check ? conv.p : nullptr;
  auto launch_aux = [&](int next, bool with_fit, int it) {
    SB_CUDA(cudaEventRecord(ctx->ev_ready, s));
    SB_CUDA(cudaStreamWaitEvent(aux, ctx->ev_ready, 0));
    if (with_fit) {
      tma.begin(kFit);
      fit(ctx, Gall.p, N, R, lambda.p, inner.p, normx.p, fit_hist.p + (it - 1), it, tol,
          check ? conv.p : nullptr, aux);  // line 13
      tma.end();
    }
    if (next >= 0) {
      tma.begin(kInverse);
      hadamard_inverse(ctx, Gall.p, N, next, R, ld, Vinv.p, status.p, sig.p, tau.p,
                       aux);  // lines 4/7/10
      tma.end();
    }
    SB_CUDA(cudaEventRecord(ctx->ev_aux, aux));
  };
  launch_aux(0, false, 0);
  // ROOT gather cache policy per tree: iteration 1 warms up, iteration 2
  // runs L1-allocating and iteration 3 L1::no_allocate gathers, timed with events (iteration
  // 1 is not a fair sample: its MTTKRPs ran ~3% faster than the same kernel in steady state
  // on c2); one host sync after iteration 3 picks the faster per tree for the rest (and for
  // later calls on the same trees).  Results do not depend on the choice.
  struct TuneEvents {
    cudaEvent_t e[SPLATT_MAX_NMODES][4] = {};
    ~TuneEvents() {
      for (auto& m : e)
        for (auto& x : m)
          if (x) cudaEventDestroy(x);
    }
  } tev_own;
  auto& tev = tev_own.e;
  bool tune[SPLATT_MAX_NMODES] = {false};
  bool tuning = false;
  auto memo_key = [&](const DevCsf& c) {
    std::vector<uint64_t> k{(uint64_t)c.N, (uint64_t)ld, c.nnz, (uint64_t)c.tiles.size()};
    for (int l = 0; l < c.N; ++l) {
      k.push_back((uint64_t)c.perm[l]);
      k.push_back(c.dims[l]);
      k.push_back(c.nodes[l]);
    }
    return k;
  };
  for (int n = 0; n < N; ++n) {  // a policy an earlier call timed on the same tree shape
    DevCsf& cn = *csf[mode_csf[n]];
    if (mode_level[n] == 0 && cn.l1a < 0) {
      auto it = ctx->l1a_memo.find(memo_key(cn));
      if (it != ctx->l1a_memo.end()) cn.l1a = it->second;
    }
  }
  if (max_iters >= 5 && !getenv("SPLATT_L1_ALLOC")) {
    for (int n = 0; n < N; ++n) {
      const DevCsf& cn = *csf[mode_csf[n]];
      // (the second-generation ROOT kernel has one gather policy: nothing to time)
      tune[n] = mode_level[n] == 0 && cn.l1a < 0 && cn.nnz >= (1u << 20) &&
                !root2_eligible(ctx, cn, ld);
      if (tune[n]) {
        tuning = true;
        for (int e = 0; e < 4; ++e) SB_CUDA(cudaEventCreate(&tev[n][e]));
      }
    }
  }
  for (int it = 1; it <= max_iters; ++it) {
    for (int n = 0; n < N; ++n) {
      const uint64_t lo = bounds[n][me], hi = bounds[n][me + 1];
      DevCsf& cn = *csf[mode_csf[n]];
      if (cn.nnz) {
        // iteration 1 warms up (L1-allocating, the usual winner, untimed); 2 times
        // L1-allocating, 3 no_allocate
        const bool timed = tune[n] && (it == 2 || it == 3);
        const int slot = it == 2 ? 1 : 0;  // tev[n][0..1]: no_allocate, [2..3]: L1-allocating
        if (timed) SB_CUDA(cudaEventRecord(tev[n][2 * slot], s));
        mttkrp_level(ctx, cn, mode_level[n], fac, M.p, X.dims[n], ld, R, &tm, kMttkrp,
                     timed ? slot : (tune[n] && it == 1 ? 1 : -1));  // 5/8/11
        if (timed) SB_CUDA(cudaEventRecord(tev[n][2 * slot + 1], s));
        mttkrp_bytes += mttkrp_alg_bytes(cn, R, mode_level[n]);
        mttkrp_min += min_bytes(cn, mode_level[n]);
        ++mttkrp_launches;
      } else {
        SB_CUDA(cudaMemsetAsync(M.p, 0, X.dims[n] * ld * sizeof(double), s));
      }
      if (sharded && used_p2[n] && !nnzpart[n].slots.empty()) {
        // P2: rows of slices split across ranks are summed into their owners' M rows
        const NnzPart& np = nnzpart[n];
        const size_t nsl = np.slots.size();
        tm.gap();
        tm.begin(kComm);
        SB_CUDA(cudaMemsetAsync(xslots.p, 0, nsl * ld * sizeof(double), s));
        for (int q = 0; q < np.npart; ++q)
          SB_CUDA(cudaMemcpyAsync(xslots.p + (size_t)np.pslot[q] * ld, M.p + np.pslice[q] * ld,
                                  ld * sizeof(double), cudaMemcpyDeviceToDevice, s));
        ctx->comm->allreduce_sum(xslots.p, nsl * ld, s);
        for (size_t k = 0; k < nsl; ++k)
          if (np.slots[k] >= np.rowb[me] && np.slots[k] < np.rowb[me + 1])
            SB_CUDA(cudaMemcpyAsync(M.p + np.slots[k] * ld, xslots.p + k * ld, ld * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
        tm.end();
      }
      // V^-1 of mode n is ready (no stream work: the solve's span starts where the MTTKRP's
      // ended, and includes any wait for the side stream)
      SB_CUDA(cudaStreamWaitEvent(s, ctx->ev_aux, 0));
      // M V^-1 + statistics; single rank: the reduction kernel also forms lambda, G_n, sig
      // (line 6); sharded: the statistics are all-reduced first.
      const LambdaOut lo_fused{it == 1, lambda.p, Gall.p + n * RR, inner.p, sig.p + (size_t)n * R,
                               ticket.p};
      // single rank: the reduction + lambda step runs on the side stream, overlapping the
      // next mode's MTTKRP (which reads the stored factor rows, not lambda or the Grams)
      const RowsReduce rr{aux, ctx->ev_solved, rpart.p, rpart.n, &tma, kNorm};
      tm.begin(kInverse);
      rows_solve_stats(ctx, M.p, A[n].p, lo, hi, R, ld, Vinv.p, tau.p, true, n == N - 1,
                       status.p, stats.p, sharded ? nullptr : &lo_fused,
                       sharded ? nullptr : &rr, peer_x ? &peer_rows[n] : nullptr);
      tm.end();
      if (sharded) {
        tm.begin(kComm);
        ctx->comm->allreduce_stats(stats.p, stats_sum_len(R), (size_t)R, s);  // max part follows
        // (peer exchange: the solve already stored the rows on every rank, and the
        // all-reduces above cannot complete before every rank's solve has)
        if (!peer_x) ctx->comm->allgatherv_rows(A[n].p, bounds[n], ld, s);
        tm.end();
        tm.begin(kNorm);
        lambda_gram(ctx, stats.p, R, it == 1, lambda.p, Gall.p + n * RR, inner.p,
                    sig.p + (size_t)n * R);  // line 6
        tm.end();
      }
      const bool last = (n == N - 1);
      const bool more = !(last && it == max_iters);
      launch_aux(more ? (n + 1) % N : -1, last, it);
    }
    it_done = it;
    if (tuning && it == 3) {
      host_sync(ctx);
      for (int n = 0; n < N; ++n) {
        if (!tune[n]) continue;
        float t0 = 0.f, t1 = 0.f;
        SB_CUDA(cudaEventElapsedTime(&t0, tev[n][0], tev[n][1]));
        SB_CUDA(cudaEventElapsedTime(&t1, tev[n][2], tev[n][3]));
        csf[mode_csf[n]]->l1a = (t1 < t0) ? 1 : 0;
        ctx->l1a_memo[memo_key(*csf[mode_csf[n]])] = csf[mode_csf[n]]->l1a;
        if (getenv("SPLATT_TRACE"))
          fprintf(stderr, "[splatt] mode %d ROOT gathers: no_allocate %.3f ms, L1-allocating %.3f ms\n",
                  n, t0, t1);
      }
      tuning = false;
    }
    if (check && it % kCheck == 0 && it < max_iters) {
      int h_conv = 0;
      SB_CUDA(cudaStreamWaitEvent(s, ctx->ev_aux, 0));  // after this iteration's fit
      SB_CUDA(cudaMemcpyAsync(&h_conv, conv.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      host_sync(ctx);
      if (h_conv) break;                                                     // C-11
    }
  }
  SB_CUDA(cudaStreamWaitEvent(s, ctx->ev_aux, 0));  // the aux stream's last work
  SB_CUDA(cudaEventRecord(loop_b, s));

  // ------------------------------------------------------------- finalise (C-12)
  // Enqueued before the status is read (one host sync per call end); on SINGULAR the
  // caller's outputs are unspecified.
  for (int n = 0; n < N; ++n) {
    fold_norms(ctx, Gall.p + n * RR, R, lambda.p, nu.p, sig.p + (size_t)n * R);
    scale_columns(ctx, A[n].p, 0, X.dims[n], R, ld, nu.p);
    SB_CUDA(cudaMemcpy2DAsync(out.factors[n], R * sizeof(double), A[n].p, ld * sizeof(double),
                              R * sizeof(double), X.dims[n], cudaMemcpyDefault, s));
  }
  SB_CUDA(cudaMemcpyAsync(out.lambda, lambda.p, R * sizeof(double), cudaMemcpyDefault, s));
  // Small results go through pinned staging (asynchronous copies), so that with stats the
  // host turns the recorded spans into times while the device finishes (collect_ready)
  // instead of after the final sync (~0.5 ms of event queries per c2 call).
  int h_status = 0, h_conv = 0;
  char* pin = ctx->pinned(2 * sizeof(double) + max_iters * sizeof(double));
  int* p_sc = pin ? reinterpret_cast<int*>(pin) : nullptr;
  double* p_hist = pin ? reinterpret_cast<double*>(pin + 2 * sizeof(double)) : nullptr;
  SB_CUDA(cudaMemcpyAsync(p_sc ? p_sc : &h_status, status.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SB_CUDA(cudaMemcpyAsync(p_sc ? p_sc + 1 : &h_conv, conv.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  double* p_normx = pin ? reinterpret_cast<double*>(pin + sizeof(double)) : &h_normx;
  if (late_norm)
    SB_CUDA(cudaMemcpyAsync(p_normx, normx.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  SB_CUDA(cudaMemcpyAsync(p_hist ? p_hist : h_hist.data(), fit_hist.p, max_iters * sizeof(double),
                          cudaMemcpyDeviceToHost, s));
  if (st) SB_CUDA(cudaEventRecord(call_b, s));
  const auto h_enq = std::chrono::steady_clock::now();
  double t_cat[kNumCat] = {0}, ta_cat[kNumCat] = {0};
  if (st) {
    while (cudaStreamQuery(s) == cudaErrorNotReady) {
      const size_t c0 = tm.cursor + tma.cursor;
      tm.collect_ready(t_cat, kNumCat);
      tma.collect_ready(ta_cat, kNumCat);
      if (tm.cursor + tma.cursor == c0) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    cudaGetLastError();
  }
  host_sync(ctx);
  const auto h_done = std::chrono::steady_clock::now();
  if (p_sc) {
    h_status = p_sc[0];
    h_conv = p_sc[1];
    std::copy(p_hist, p_hist + max_iters, h_hist.begin());
  }
  if (late_norm) h_normx = *p_normx;
  float loop_ms = 0.f;
  cudaEventElapsedTime(&loop_ms, loop_a, loop_b);
  cudaEventDestroy(loop_a);
  cudaEventDestroy(loop_b);
  float call_ms = 0.f;
  if (st) {
    cudaEventElapsedTime(&call_ms, call_a, call_b);
    cudaEventDestroy(call_a);
    cudaEventDestroy(call_b);
  }
  if (late_norm && !(h_normx > 0.0)) fail(SPLATT_ERR_EMPTY, "||X|| = 0");
  if (h_status) fail(SPLATT_ERR_SINGULAR, "Gram Hadamard product is singular (after ridge)");
  if (h_conv) it_done = h_conv;  // later enqueued iterations were no-ops
  *out.fit = h_hist[it_done - 1];
  *out.iters = it_done;
  if (out.fit_history)
    for (int i = 0; i < it_done; ++i) out.fit_history[i] = h_hist[i];

  if (st) {
    double* t = t_cat;
    double* ta = ta_cat;
    tm.collect(t, kNumCat);
    tma.collect(ta, kNumCat);
    st->t_aux_inverse = ta[kInverse];
    st->t_aux_fit = ta[kFit];
    st->t_mttkrp = t[kMttkrp];
    st->t_build = t[kBuild];
    st->t_ata = t[kAta];
    st->t_norm = t[kNorm] + ta[kNorm];  // single rank: on the side stream (overlapped)
    st->t_fit = t[kFit];
    st->t_inverse = t[kInverse];
    st->t_comm = t[kComm];
    st->t_loop = loop_ms * 1e-3;
    st->mttkrp_alg_bytes = mttkrp_bytes;
    st->mttkrp_min_bytes = mttkrp_min;
    st->mttkrp_launches = mttkrp_launches;
    st->kernel_launches = ctx->kernel_launches - launches0;
    for (int k = 0; k < (sharded ? N : ncsf); ++k)
      for (int l = 0; l < N; ++l) st->csf_nodes[k][l] = csf[k]->nodes[l];
    st->iters = it_done;
    st->nranks = G;
    st->exchange = peer_x ? SPLATT_XCHG_PEER : SPLATT_XCHG_COLLECTIVE;
    st->t_call = call_ms * 1e-3;
    st->host_syncs = (int32_t)(ctx->host_syncs - syncs0);
    st->t_host_sync = ctx->host_sync_s - sync_s0;
  }
  static const bool trace = getenv("SPLATT_TRACE") != nullptr;
  if (trace)
    fprintf(stderr, "[splatt trace] driver: enqueue-to-end %.3f ms (host %.3f ms ahead of the "
            "device at the final sync), epilogue %.3f ms\n",
            std::chrono::duration<double, std::milli>(h_enq - h_start).count(),
            std::chrono::duration<double, std::milli>(h_done - h_enq).count(),
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h_done)
                .count());
}

}  // namespace sb
