// root2.cu — the second-generation ROOT MTTKRP (root2.cuh): its per-tree plan and launch.
//
// RootPlan (built once per tree and rank padding, on the context stream, no host sync):
//   1. a sampled histogram of the ids every non-root level gathers (leaf ids, and the ids
//      of every internal level below the root: one factor row per node);
//   2. the K most frequent (level, id) pairs, by a descending radix sort of the counts,
//      become the shared-memory row slots (K from the kernel's shared-memory budget);
//   3. coded ids (slot | kHot, or the row id) for the leaves and internal levels, and the
//      per-leaf record {leaf code | d << 29, code of the fiber closing here, value} with d
//      the shallowest level whose node ends at this leaf (N-1: none), found by walking each
//      node's last child down to its last leaf.
// Integer work only: the plan is a pure function of the tree (the hot set only decides
// where a row is read from, never what is computed).
#include <algorithm>

#include "mttkrp.hpp"
#include "root2.cuh"

#ifndef SB_ROOT2_TABLE
#define SB_ROOT2_TABLE 256  // leaves per chunk-table entry of a tree run by this kernel
#endif
#ifndef SB_ROOT2_UNIT
#define SB_ROOT2_UNIT 6  // table chunks per big work unit (6 x 256 = 1536 leaves)
#endif
#ifndef SB_ROOT2_TAIL
#define SB_ROOT2_TAIL 2  // table chunks per group handed out one by one at the end
#endif

namespace sb {

#ifndef SB_ROOT2_HOT_MAX
#define SB_ROOT2_HOT_MAX 2
#endif
// Hot rows held in shared memory (at most; SPLATT_ROOT2_HOT overrides).  Only the very top
// rows pay: a power-law tensor sends ~1/H of a level's gathers to its hottest row, and those
// reads then skip the L1TEX/L2 round trip (per-CTA replicas of the same rows in global memory,
// which would relieve an L2 hot spot, ran as K = 0); rows further down the list are read by
// different groups of a warp in one instruction and cost shared-memory bank conflicts instead
// (c5 sweep: K = 0 2.66, 2 2.39, 8 2.45, 32 2.50, 248 (the capacity) 2.56 ms;
// profiles/ab_r02/README.md).
uint32_t root2_hot_rows() {
  if (const char* e = getenv("SPLATT_ROOT2_HOT")) return (uint32_t)atoi(e);
  return SB_ROOT2_HOT_MAX;
}

int root2_table_chunk() {
  if (const char* e = getenv("SPLATT_CHUNK")) {
    const int v = atoi(e);
    if (v >= 32 && v % 32 == 0) return v;
  }
  return SB_ROOT2_TABLE;
}

namespace {

using r2::kHot;
using r2::kIdMask;

inline int grid_n(splatt_ctx* ctx, uint64_t n) {
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n, 256), (uint64_t)ctx->num_sms * 16));
}

#ifndef SB_PLAN_SAMPLE
#define SB_PLAN_SAMPLE 256
#endif
constexpr uint32_t kSample = SB_PLAN_SAMPLE;  // histogram: every kSample-th node / leaf

__global__ void sampled_hist_kernel(const uint32_t* __restrict__ ids, uint64_t n, uint32_t step,
                                    uint32_t* __restrict__ cnt) {
  for (uint64_t j = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * step; j < n;
       j += (uint64_t)gridDim.x * blockDim.x * step)
    atomicAdd(&cnt[ids[j]], 1u);
}

__global__ void iota_u32_kernel(uint32_t* __restrict__ p, uint64_t n) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    p[j] = (uint32_t)j;
}

struct LevelOffsets {
  uint64_t off[SPLATT_MAX_NMODES + 1];  // concatenated count arrays of levels 1..N-1
  int N;
};

// c -> ~c: an ascending stable sort of the complements is the descending stable sort of the
// counts (equal counts keep the (level, id) order).
__global__ void complement_kernel(uint32_t* __restrict__ c, uint64_t n) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    c[j] = ~c[j];
}

// Slot s <- the s-th most frequent (level, id) if it was sampled at least twice
// (cnt_sorted: complemented counts in ascending order).
__global__ void hot_slots_kernel(const uint32_t* __restrict__ cnt_sorted,
                                 const uint32_t* __restrict__ gidx_sorted, uint64_t total,
                                 uint32_t K, LevelOffsets lo, uint32_t* __restrict__ hot,
                                 uint32_t* __restrict__ slotmap) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= K) return;
  if (s >= total || ~cnt_sorted[s] < 2u) { hot[s] = ~0u; return; }
  const uint32_t g = gidx_sorted[s];
  int l = 1;
  while (l + 1 < lo.N && g >= lo.off[l + 1]) ++l;
  hot[s] = ((uint32_t)l << 28) | (uint32_t)(g - lo.off[l]);
  slotmap[g] = s;
}

// Row code (root2.cuh): byte offset into the shared-memory table or into the factor.
__device__ __forceinline__ uint32_t code_of(const uint32_t* __restrict__ slotmap, uint64_t off,
                                            uint32_t id, uint32_t ldb) {
  const uint32_t s = slotmap[off + id];
  return s != ~0u ? (kHot | (s * ldb + ((s & 1u) << 4))) : id * ldb;
}

// Leaf records, with d = N-1 (no node ends here) until the level passes below.
__global__ void leaf_records_kernel(const uint32_t* __restrict__ leaf, const double* __restrict__ vals,
                                    uint64_t nnz, const uint32_t* __restrict__ slotmap,
                                    uint64_t off, uint32_t ldb, uint32_t dnone,
                                    uint4* __restrict__ rec) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t code = code_of(slotmap, off, leaf[k], ldb);
    const double v = vals[k];
    rec[k] = make_uint4(code | (dnone << r2::kDShift), 0u, (uint32_t)__double2loint(v),
                        (uint32_t)__double2hiint(v));
  }
}

struct PtrChain {
  const uint32_t* ptr[SPLATT_MAX_NMODES];
  int N;
};

// Level l (launched N-2 first, then upwards, so the shallowest level is written last): the
// last leaf of every level-l node gets d = l; level N-2 also writes the fiber's code.
__global__ void close_level_kernel(PtrChain pc, int l, uint64_t nodes,
                                   const uint32_t* __restrict__ ids_l,
                                   const uint32_t* __restrict__ slotmap, uint64_t off,
                                   uint32_t ldb, uint4* __restrict__ rec) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nodes;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = j;
    for (int m = l; m <= pc.N - 2; ++m) c = pc.ptr[m][c + 1] - 1u;  // last child, down to a leaf
    uint32_t* w = reinterpret_cast<uint32_t*>(rec + c);
    w[0] = (w[0] & ~(7u << r2::kDShift)) | ((uint32_t)l << r2::kDShift);
    if (l == pc.N - 2) w[1] = code_of(slotmap, off, ids_l[j], ldb);
  }
}

__global__ void code_level_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                  const uint32_t* __restrict__ slotmap, uint64_t off,
                                  uint32_t ldb, uint32_t* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = code_of(slotmap, off, ids[j], ldb);
}

struct CoordSet {
  const uint32_t* c[SPLATT_MAX_NMODES];  // level-order sorted coordinates (nnz each)
  int N;
};

// Every kSample-th leaf: its id, and the id of every internal node (levels 1..N-2) that
// starts there — a level-l node starts at j when a coordinate of levels 0..l differs from
// leaf j-1 (each node has one start, so nodes are sampled at the same 1/kSample rate).
__device__ __forceinline__ void add_aggregated(uint32_t* cnt, uint32_t a) {
  // equal addresses of a warp add once (power-law ids: the hot rows' counters are contended)
  const uint32_t peers = __match_any_sync(0xffffffffu, a);
  if (a != ~0u && (peers & ((1u << (threadIdx.x & 31u)) - 1u)) == 0u)
    atomicAdd(&cnt[a], (uint32_t)__popc(peers));
}
__global__ void sampled_hist_coords_kernel(CoordSet cs, uint64_t nnz, LevelOffsets lo,
                                           uint32_t* __restrict__ cnt) {
  const int N = cs.N;
  const uint64_t lane = threadIdx.x & 31u;
  // warp-uniform loop (every lane takes part in the aggregation)
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u);
       base * kSample < nnz; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = (base + lane) * kSample;
    const bool valid = k < nnz;
    add_aggregated(cnt, valid ? (uint32_t)(lo.off[N - 1] + cs.c[N - 1][k]) : ~0u);
    int ds = 0;  // first level whose coordinate differs from leaf k-1
    if (valid && k > 0) {
      ds = N - 1;
      for (int l = N - 2; l >= 0; --l)
        if (cs.c[l][k] != cs.c[l][k - 1]) ds = l;
    }
    for (int l = 1; l <= N - 2; ++l)
      add_aggregated(cnt, (valid && ds <= l) ? (uint32_t)(lo.off[l] + cs.c[l][k]) : ~0u);
  }
}

template <int G>
uint32_t plan_capacity(int N, int ld) {
  return N == 3 ? r2::hot_capacity<G, r2::Threads<3>::k>(ld)
                : r2::hot_capacity<G, r2::Threads<4>::k>(ld);
}

}  // namespace

// Lane-group width of the ROOT kernels for a padded rank (as launch_g: next pow2 of ld/4,
// packed 3 x 10 for ld/4 in {9, 10}).
int root2_group_width(int ld) {
  const int slots = ld / 4;
  if (slots <= 2) return 2;
  if (slots <= 4) return 4;
  if (slots == 9 || slots == 10) return 10;
  if (slots <= 8) return 8;
  if (slots <= 16) return 16;
  return 32;
}

uint32_t root2_hot_capacity(int N, int ld) {
  switch (root2_group_width(ld)) {
    case 2: return plan_capacity<2>(N, ld);
    case 4: return plan_capacity<4>(N, ld);
    case 8: return plan_capacity<8>(N, ld);
    case 10: return plan_capacity<10>(N, ld);
    case 16: return plan_capacity<16>(N, ld);
    default: return plan_capacity<32>(N, ld);
  }
}

bool root2_eligible(const splatt_ctx* ctx, const DevCsf& c, int ld) {
  // Default: 4-mode trees.  On 3-mode trees the first-generation kernel is as fast (c2) or
  // faster (c3 -9%, c4 -15%: its 24 resident warps and packed record phase beat the staged
  // records there; profiles/ab_r02/).  SPLATT_ROOT2=0 forces the first-generation kernel,
  // SPLATT_ROOT2=3 also runs this one on 3-mode trees (A/B runs and tests).
  const char* e = getenv("SPLATT_ROOT2");
  if ((e && *e == '0') || ctx->deterministic) return false;
  const bool n3 = e && *e == '3';
  if (c.N != 4 && !(c.N == 3 && n3)) return false;
  // row codes are byte offsets below 2^28 (factors of up to 256 MiB)
  for (int l = 1; l < c.N; ++l)
    if ((uint64_t)c.dims[l] * (uint64_t)ld * 8u >= (uint64_t)kHot) return false;
  return true;
}

void ensure_root_plan(splatt_ctx* ctx, DevCsf& c, int ld) {
  if (c.plan && c.plan->ld == ld && c.plan->ready) return;
  cudaStream_t st = ctx->stream;
  const int N = c.N;
  ArenaScope own(c.arena, false);  // lives as long as the tree
  auto plan = std::make_unique<RootPlan>();
  plan->ld = ld;
  plan->K = root2_hot_capacity(N, ld);
  plan->K = std::min<uint32_t>(plan->K, root2_hot_rows());
  const uint32_t ldb = (uint32_t)ld * 8u;
  LevelOffsets lo{};
  lo.N = N;
  uint64_t total = 0;
  for (int l = 1; l < N; ++l) { lo.off[l] = total; total += c.dims[l]; }
  lo.off[N] = total;
  plan->rec.alloc(c.nnz, st);
  // one padding entry each (the kernel loads one node ahead without a bounds test)
  for (int l = 0; l <= N - 3; ++l) {
    plan->cid[l].alloc(c.nodes[l] + 1, st);
    SB_CUDA(cudaMemsetAsync(plan->cid[l].p + c.nodes[l], 0, 4, st));
  }
  SB_CUDA(cudaMemcpyAsync(plan->cid[0].p, c.ids[0].p, c.nodes[0] * 4, cudaMemcpyDeviceToDevice, st));
  plan->hot.alloc(std::max<uint32_t>(1, plan->K), st);
  {
    // scratch: counts, sort pairs, slot map (released with the scope below when the tree
    // comes from an arena; pooled otherwise)
    ArenaScope tmp(current_arena(), true);
    DevBuf<uint32_t> cnt(total, st), cnt2(total, st), gidx(total, st), gidx2(total, st),
        slotmap(total, st);
    SB_CUDA(cudaMemsetAsync(cnt.p, 0, total * 4, st));
    SB_CUDA(cudaMemsetAsync(slotmap.p, 0xff, total * 4, st));
    for (int l = 1; l < N; ++l) {
      const uint64_t n = c.nodes[l];
      sampled_hist_kernel<<<grid_n(ctx, ceil_div(n, kSample)), 256, 0, st>>>(
          c.ids[l].p, n, kSample, cnt.p + lo.off[l]);
      SB_CHECK_LAUNCH(ctx);
    }
    iota_u32_kernel<<<grid_n(ctx, total), 256, 0, st>>>(gidx.p, total);
    SB_CHECK_LAUNCH(ctx);
    complement_kernel<<<grid_n(ctx, total), 256, 0, st>>>(cnt.p, total);
    SB_CHECK_LAUNCH(ctx);
    radix_sort_pairs(ctx, cnt.p, gidx.p, cnt2.p, gidx2.p, cnt.p, gidx.p, total, 0, 32);
    if (plan->K > 0) {
      hot_slots_kernel<<<(unsigned)ceil_div(plan->K, 256), 256, 0, st>>>(
          cnt2.p, gidx2.p, total, plan->K, lo, plan->hot.p, slotmap.p);
      SB_CHECK_LAUNCH(ctx);
    }
    leaf_records_kernel<<<grid_n(ctx, c.nnz), 256, 0, st>>>(
        c.ids[N - 1].p, c.vals.p, c.nnz, slotmap.p, lo.off[N - 1], ldb, (uint32_t)(N - 1),
        plan->rec.p);
    SB_CHECK_LAUNCH(ctx);
    PtrChain pc{};
    pc.N = N;
    for (int l = 0; l < N - 1; ++l) pc.ptr[l] = c.ptr[l].p;
    for (int l = N - 2; l >= 0; --l) {
      close_level_kernel<<<grid_n(ctx, c.nodes[l]), 256, 0, st>>>(
          pc, l, c.nodes[l], c.ids[l].p, slotmap.p, l >= 1 ? lo.off[l] : 0, ldb, plan->rec.p);
      SB_CHECK_LAUNCH(ctx);
    }
    for (int l = 1; l <= N - 3; ++l) {
      code_level_kernel<<<grid_n(ctx, c.nodes[l]), 256, 0, st>>>(c.ids[l].p, c.nodes[l],
                                                                  slotmap.p, lo.off[l], ldb,
                                                                  plan->cid[l].p);
      SB_CHECK_LAUNCH(ctx);
    }
  }
  plan->ready = true;
  c.plan = std::move(plan);
}

bool root_plan_begin(splatt_ctx* ctx, DevCsf& c, const uint32_t* const* coord,
                     const double* vals, int ld, RootPlanRecOut* ro) {
  if (c.nnz == 0 || !root2_eligible(ctx, c, ld)) return false;
  cudaStream_t st = ctx->stream;
  const int N = c.N;
  auto plan = std::make_unique<RootPlan>();  // from the current arena (the tree's)
  plan->ld = ld;
  plan->K = root2_hot_capacity(N, ld);
  plan->K = std::min<uint32_t>(plan->K, root2_hot_rows());
  LevelOffsets lo{};
  lo.N = N;
  uint64_t total = 0;
  for (int l = 1; l < N; ++l) { lo.off[l] = total; total += c.dims[l]; }
  lo.off[N] = total;
  for (int l = 0; l <= N; ++l) plan->off[l] = lo.off[l];
  plan->rec.alloc(c.nnz, st);
  plan->hot.alloc(std::max<uint32_t>(1, plan->K), st);
  {
    ArenaScope pooled(nullptr, false);  // released by root_plan_end, not with the arena
    plan->slotmap.alloc(total, st);
  }
  SB_CUDA(cudaMemsetAsync(plan->slotmap.p, 0xff, total * 4, st));
  CoordSet cs{};
  cs.N = N;
  for (int l = 0; l < N; ++l) cs.c[l] = coord[l];
  {
    ArenaScope tmp(current_arena(), true);
    DevBuf<uint32_t> cnt(total, st), cnt2(total, st), gidx(total, st), gidx2(total, st);
    SB_CUDA(cudaMemsetAsync(cnt.p, 0, total * 4, st));
    sampled_hist_coords_kernel<<<grid_n(ctx, ceil_div(c.nnz, kSample)), 256, 0, st>>>(
        cs, c.nnz, lo, cnt.p);
    SB_CHECK_LAUNCH(ctx);
    iota_u32_kernel<<<grid_n(ctx, total), 256, 0, st>>>(gidx.p, total);
    SB_CHECK_LAUNCH(ctx);
    complement_kernel<<<grid_n(ctx, total), 256, 0, st>>>(cnt.p, total);
    SB_CHECK_LAUNCH(ctx);
    radix_sort_pairs(ctx, cnt.p, gidx.p, cnt2.p, gidx2.p, cnt.p, gidx.p, total, 0, 32);
    if (plan->K > 0) {
      hot_slots_kernel<<<(unsigned)ceil_div(plan->K, 256), 256, 0, st>>>(
          cnt2.p, gidx2.p, total, plan->K, lo, plan->hot.p, plan->slotmap.p);
      SB_CHECK_LAUNCH(ctx);
    }
  }
  ro->rec = plan->rec.p;
  ro->slotmap = plan->slotmap.p;
  ro->off_leaf = lo.off[N - 1];
  ro->off_fiber = lo.off[N - 2];
  ro->ldb = (uint32_t)ld * 8u;
  ro->vals = vals;
  c.plan = std::move(plan);
  return true;
}

void root_plan_end(splatt_ctx* ctx, DevCsf& c) {
  RootPlan& p = *c.plan;
  cudaStream_t st = ctx->stream;
  const int N = c.N;
  const uint32_t ldb = (uint32_t)p.ld * 8u;
  // padded id arrays (one entry more: the kernel loads one node ahead without a bounds test)
  for (int l = 0; l <= N - 3; ++l) {
    p.cid[l].alloc(c.nodes[l] + 1, st);
    SB_CUDA(cudaMemsetAsync(p.cid[l].p + c.nodes[l], 0, 4, st));
    if (l == 0) {
      SB_CUDA(cudaMemcpyAsync(p.cid[0].p, c.ids[0].p, c.nodes[0] * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      code_level_kernel<<<grid_n(ctx, c.nodes[l]), 256, 0, st>>>(c.ids[l].p, c.nodes[l],
                                                                  p.slotmap.p, p.off[l], ldb,
                                                                  p.cid[l].p);
      SB_CHECK_LAUNCH(ctx);
    }
  }
  p.slotmap.release();
  p.ready = true;
}

namespace {

template <int N, int G, int U>
void launch2_t(splatt_ctx* ctx, DevCsf& c, const double* const* fac_by_mode, double* out, int ld,
               int R, int acc) {
  const RootPlan& p = *c.plan;
  r2::Args<N> a{};
  a.rec = p.rec.p;
  for (int l = 0; l < N; ++l) {
    a.cid[l] = p.cid[l].p;
    a.ids[l] = c.ids[l].p;
    a.fac[l] = (l == 0) ? nullptr : fac_by_mode[c.perm[l]];
    a.nodes[l] = (uint32_t)c.nodes[l];
  }
  a.out = out;
  a.tab = c.tab.p;
  a.hot = p.hot.p;
  a.K = p.K;
  a.nnz = (uint32_t)c.nnz;
  a.nchunks = (uint32_t)c.nchunks;
  a.chunk = (uint32_t)c.tab_chunk;
  a.ld = (uint32_t)ld;
  a.R = R;
  a.accumulate = acc & 1;
  a.conv = ctx->d_conv;
  constexpr int T = r2::Threads<N>::k;
  const size_t smem = (size_t)p.K * ld * 8 + r2::rec_smem_bytes<G, T>();
  auto kern = r2::mttkrp_root2_kernel<N, G, U>;
  // (the opt-in is cached per kernel and device: always ask for the whole budget)
  set_max_dynamic_smem((const void*)kern, r2::kSmemBudget);
  const uint64_t groups = (uint64_t)r2::Lanes<G, T>::kGroups;
  // guided units (Args::unit): big units of kRoot2Unit table chunks while more than
  // kRoot2Tail table chunks per group of the whole grid remain
  {
    const uint64_t all_groups = (uint64_t)ctx->num_sms * groups;
    const uint64_t small = std::min<uint64_t>(c.nchunks, (uint64_t)SB_ROOT2_TAIL * all_groups);
    a.unit = SB_ROOT2_UNIT;
    a.nbig = (uint32_t)((c.nchunks - small) / SB_ROOT2_UNIT);
    a.nunits = (uint32_t)(a.nbig + c.nchunks - (uint64_t)a.nbig * SB_ROOT2_UNIT);
  }
  uint64_t blocks = ceil_div(a.nunits, groups);
  if (blocks > (uint64_t)ctx->num_sms) {
    blocks = (uint64_t)ctx->num_sms;  // one CTA per SM, chunks taken dynamically
    ArenaScope own(c.arena, false);
    if (c.work.n < 1) {
      c.work.alloc(1, ctx->stream);
      SB_CUDA(cudaMemsetAsync(c.work.p, 0, sizeof(unsigned), ctx->stream));
      c.work_base = 0;
    }
    if (!c.work_seq) {
      SB_CUDA(cudaMemsetAsync(c.work.p, 0, sizeof(unsigned), ctx->stream));
      c.work_base = 0;
    }
    a.work = c.work.p;
    a.work_base = c.work_base;
    c.work_base += (unsigned)(a.nunits + blocks * groups);
  }
  kern<<<(unsigned)blocks, T, smem, ctx->stream>>>(a);
  SB_CHECK_LAUNCH(ctx);
}

#ifndef SB_ROOT2_U
#define SB_ROOT2_U 2
#endif

template <int N>
void launch2_n(splatt_ctx* ctx, DevCsf& c, const double* const* f, double* out, int ld, int R,
               int acc) {
  constexpr int U = SB_ROOT2_U;
  switch (root2_group_width(ld)) {
    case 2: return launch2_t<N, 2, U>(ctx, c, f, out, ld, R, acc);
    case 4: return launch2_t<N, 4, U>(ctx, c, f, out, ld, R, acc);
    case 8: return launch2_t<N, 8, U>(ctx, c, f, out, ld, R, acc);
    case 10: return launch2_t<N, 10, U>(ctx, c, f, out, ld, R, acc);
    case 16: return launch2_t<N, 16, U>(ctx, c, f, out, ld, R, acc);
    default: return launch2_t<N, 32, U>(ctx, c, f, out, ld, R, acc);
  }
}

}  // namespace

void mttkrp_root2_launch(splatt_ctx* ctx, DevCsf& c, const double* const* f, double* out, int ld,
                         int R, int acc) {
  if (!c.plan || c.plan->ld != ld || !c.plan->ready) fail(SPLATT_ERR_CUDA, "internal: ROOT plan missing");
  if (c.N == 3) return launch2_n<3>(ctx, c, f, out, ld, R, acc);
  if (c.N == 4) return launch2_n<4>(ctx, c, f, out, ld, R, acc);
  fail(SPLATT_ERR_UNSUPPORTED, "internal: ROOT kernel v2 for N = 3, 4 only");
}

}  // namespace sb
